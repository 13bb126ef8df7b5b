"""GPU parity: the CUDA STP (through the C ABI) against the CPU oracle on identical inputs.

Tolerance: the reference's rel_diff metric (proj/src/checks.cpp:27-34), per element and per
output array, <= 1e-12 (BASELINE.json north_star).  Inputs are generated on the device and copied
back, so both sides see bit-identical data.
"""
import zlib as _zlib

import numpy as np
import pytest

import oracle as O

TOL = 1e-12

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_12787_b200 as S
    return S


def _compare(S, oracle, n, out, ref, layout, out_stride, m=9):
    E = ref.qavg.shape[0]
    qa = out.qavg.cpu().numpy()
    if layout == S.LAYOUT_AOSOA:
        qa_c = oracle.from_aosoa(n, m, out_stride, qa)
        fa_c = np.stack([oracle.from_aosoa(n, m, out_stride, out.favg[:, d].cpu().numpy()) for d in range(3)], 1)
    else:
        qa_c = qa.reshape(E, n ** 3, out_stride)[:, :, :m].reshape(E, -1)
        fa_c = out.favg.cpu().numpy().reshape(E, 3, n ** 3, out_stride)[..., :m].reshape(E, 3, -1)
    worst = {
        "qavg": O.per_element_rel_diff(ref.qavg, qa_c),
        "favg": max(O.per_element_rel_diff(ref.favg[:, d], fa_c[:, d]) for d in range(3)),
        "face_q": max(O.per_element_rel_diff(ref.face_q[:, f], out.face_q[:, f].cpu().numpy()) for f in range(6)),
        "face_f": max(O.per_element_rel_diff(ref.face_f[:, f], out.face_f[:, f].cpu().numpy()) for f in range(6)),
    }
    return worst


@pytest.mark.parametrize("n", list(range(2, 11)))
def test_elastic_parity(stp, oracle, n):
    S = stp
    E = 37 if n <= 8 else 9  # not a multiple of the elements-per-block
    q, par = S.generate(0, 1234 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    par_h = par.cpu().numpy()
    dt = O.cfl_dt(n, par_h[:, 1].max())
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    out = plan.predict(q, dt, par=par)
    plan.status()
    qc = oracle.from_aosoa(n, 9, 9, q.cpu().numpy())
    ref = oracle.stp(n, 9, qc, dt, par=oracle.material_lmr(par_h))
    worst = _compare(S, oracle, n, out, ref, S.LAYOUT_AOSOA, 9)
    assert max(worst.values()) <= TOL, worst


@pytest.mark.parametrize("force_generic", [False, True])
@pytest.mark.parametrize("q_stride", [9, 12])
def test_order8_kernels_parity(stp, oracle, monkeypatch, force_generic, q_stride):
    """nDof 8 runs on the DMMA kernel by default; ADERSTP_FORCE_GENERIC=1 selects the generic one."""
    S = stp
    monkeypatch.setenv("ADERSTP_FORCE_GENERIC", "1" if force_generic else "0")
    n, E = 8, 301
    q, par = S.generate(0, 77, n, 1000, E, layout=S.LAYOUT_AOSOA, q_stride=q_stride)
    par_h = par.cpu().numpy()
    dt = O.cfl_dt(n, par_h[:, 1].max())
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=q_stride, par_kind=S.PAR_RHO_CP_CS)
    out = plan.predict(q, dt, par=par)
    plan.status()
    qc = oracle.from_aosoa(n, 9, q_stride, q.cpu().numpy())
    ref = oracle.stp(n, 9, qc, dt, par=oracle.material_lmr(par_h))
    worst = _compare(S, oracle, n, out, ref, S.LAYOUT_AOSOA, 9)
    assert max(worst.values()) <= TOL, worst


@pytest.mark.parametrize("n", [2, 3, 5, 6, 8, 9, 10])
def test_kernel_variants_agree(stp, oracle, monkeypatch, n):
    """Every kernel family against the oracle: the default dispatch (dmmap nDof 4-7, dmma8 nDof 8,
    bip nDof 9-10, line-pass nDof 2-3), the line-pass kernel at every order (NO_DMMA8 / NO_DMMAP /
    PASS_SLOTS=6), the bipartite kernel forced, the generic table kernel, and no L2 prefetch."""
    S = stp
    E = 19
    q, par = S.generate(0, 5 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    par_h = par.cpu().numpy()
    dt = O.cfl_dt(n, par_h[:, 1].max())
    ref = oracle.stp(n, 9, oracle.from_aosoa(n, 9, 9, q.cpu().numpy()), dt, par=oracle.material_lmr(par_h))
    keys = ("ADERSTP_NO_DMMA8", "ADERSTP_NO_DMMAP", "ADERSTP_PASS_SLOTS", "ADERSTP_FORCE_GENERIC", "ADERSTP_PREFETCH")
    variants = [{}, {"ADERSTP_NO_DMMA8": "1", "ADERSTP_NO_DMMAP": "1", "ADERSTP_PASS_SLOTS": "6"},
                {"ADERSTP_FORCE_GENERIC": "1"}, {"ADERSTP_PREFETCH": "0"}]
    if n in (9, 10):
        variants.append({"ADERSTP_PASS_SLOTS": "12"})
    for env in variants:
        for k in keys:
            if k in env:
                monkeypatch.setenv(k, env[k])
            else:
                monkeypatch.delenv(k, raising=False)
        plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
        out = plan.predict(q, dt, par=par)
        plan.status()
        worst = _compare(S, oracle, n, out, ref, S.LAYOUT_AOSOA, 9)
        assert max(worst.values()) <= TOL, (env, worst)


@pytest.mark.parametrize("n,E,qs", [(6, 19, 9), (6, 1037, 9), (6, 50, 12), (5, 19, 9), (5, 1500, 9), (5, 50, 12),
                                    (4, 19, 9), (4, 2100, 9), (4, 50, 12)])
def test_warp_per_element_kernel(stp, oracle, monkeypatch, n, E, qs):
    """The opt-in warp-per-element kernel (ADERSTP_WPE=1, csrc/stp_wpe.cu: nDof 4 / 5 / 6, persistent
    warps, several elements per warp, ragged last wave, padded input stride) against the oracle."""
    S = stp
    monkeypatch.setenv("ADERSTP_WPE", "1")
    q, par = S.generate(0, 11 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=qs)
    par_h = par.cpu().numpy()
    dt = O.cfl_dt(n, par_h[:, 1].max())
    ref = oracle.stp(n, 9, oracle.from_aosoa(n, 9, qs, q.cpu().numpy()), dt, par=oracle.material_lmr(par_h))
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=qs, par_kind=S.PAR_RHO_CP_CS)
    out = plan.predict(q, dt, par=par)
    plan.status()
    worst = _compare(S, oracle, n, out, ref, S.LAYOUT_AOSOA, 9)
    assert max(worst.values()) <= TOL, worst
    # optional outputs: qavg alone, and qavg + favg without faces, match the full call bit for bit
    o1 = plan.predict(q, dt, par=par, want_favg=False, want_faces=False)
    o2 = plan.predict(q, dt, par=par, want_faces=False)
    plan.status()
    assert torch.equal(o1.qavg, out.qavg) and torch.equal(o2.qavg, out.qavg) and torch.equal(o2.favg, out.favg)
    # non-finite input and bad material are flagged like in the default kernels
    q2 = q.clone()
    q2.view(-1)[7] = float("nan")
    plan.predict(q2, dt, par=par)
    with pytest.raises(Exception):
        plan.status()
    par2 = par.clone()
    par2[E // 2, 0] = -1.0
    plan.predict(q, dt, par=par2)
    with pytest.raises(Exception):
        plan.status()


# ---------------------------------------------------------------------------------------------
# Against the reference's own outputs (tests/golden, produced by the unmodified reference)
# ---------------------------------------------------------------------------------------------
import json as _json  # noqa: E402
import os as _os  # noqa: E402

GOLDEN = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "golden")


def _golden_cases():
    with open(_os.path.join(GOLDEN, "index.json")) as f:
        return _json.load(f)["cases"]


def _pde_for(S, case, g):
    kind = case.get("pde_kind", 0)
    args = g["args"] if "args" in g else None
    if kind == 0:
        return S.elastic_pde()
    if kind == 1:
        return S.advection_pde(args[:3], case["m"])
    if kind == 2:
        return S.ncp_advection_pde(args[:3], case["m"])
    if kind == 3:
        return S.paper_demo_pde()
    src = S.PointSourceSpec(tuple(args[:3]), int(args[3]), args[4], args[5], args[6])
    if kind == 4:
        return S.elastic_pde(source=src)
    return S.source_only_pde(case["m"], src)


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c["name"])
@pytest.mark.parametrize("layout", ["aosoa", "aos16"])
def test_matches_reference_golden(stp, oracle, case, layout):
    """GPU output vs the reference's own predict(splitck) + extrapolate_faces outputs."""
    S = stp
    g = np.load(_os.path.join(GOLDEN, case["name"] + ".npz"))
    n, m = case["n"], case["m"]
    E = g["q"].shape[0]
    pde = _pde_for(S, case, g)
    if layout == "aosoa":
        qs, lay = m, S.LAYOUT_AOSOA
        qdev = oracle.to_aosoa(n, m, qs, g["q"])
    else:  # the reference ElementTensor layout: AoS, quantity padded to 16 (layout.cpp:9-21)
        qs, lay = 16, S.LAYOUT_AOS
        qdev = np.zeros((E, n ** 3, 16))
        qdev[:, :, :m] = g["q"].reshape(E, n ** 3, m)
    q = torch.from_numpy(np.ascontiguousarray(qdev).reshape(E, -1)).cuda()
    par = torch.from_numpy(g["par_lmr"]).cuda() if "par_lmr" in g else None
    plan = S.Plan(n, pde, layout=lay, q_stride=qs, out_stride=qs, par_kind=S.PAR_LAMBDA_MU_RHO)
    out = plan.predict(q, float(g["dt"]), par=par, t_start=float(g["t_start"]))
    plan.status()
    qa = out.qavg.cpu().numpy()
    fa = out.favg.cpu().numpy()
    if layout == "aosoa":
        qa_c = oracle.from_aosoa(n, m, qs, qa)
        fa_c = np.stack([oracle.from_aosoa(n, m, qs, fa[:, d]) for d in range(3)], 1)
    else:
        qa_c = qa.reshape(E, n ** 3, 16)[:, :, :m].reshape(E, -1)
        fa_c = fa.reshape(E, 3, n ** 3, 16)[..., :m].reshape(E, 3, -1)
        # padding lanes of every output stay exactly zero (test_predictor.cpp:157-170)
        assert not np.any(qa.reshape(E, n ** 3, 16)[:, :, m:])
        assert not np.any(fa.reshape(E, 3, n ** 3, 16)[..., m:])
    assert O.per_element_rel_diff(g["qavg"], qa_c) <= TOL
    assert O.per_element_rel_diff(g["favg"].reshape(E, -1), fa_c.reshape(E, -1)) <= TOL
    assert O.per_element_rel_diff(g["face_q"].reshape(E, -1), out.face_q.cpu().numpy().reshape(E, -1)) <= TOL
    assert O.per_element_rel_diff(g["face_f"].reshape(E, -1), out.face_f.cpu().numpy().reshape(E, -1)) <= TOL


# ---------------------------------------------------------------------------------------------
# Properties and edge cases
# ---------------------------------------------------------------------------------------------
def test_zero_dynamics_exact(stp):
    """advection with v = 0: qavg == dt*q bit-exactly, favg == 0 (test_predictor.cpp:36-53)."""
    S = stp
    for n in (2, 4, 8):
        rng = np.random.default_rng(42 + n)
        qn = rng.uniform(-1, 1, (5, n ** 3 * 3))
        q = torch.from_numpy(qn).cuda()
        dt = 0.013
        plan = S.Plan(n, S.advection_pde([0.0, 0.0, 0.0], 3))
        out = plan.predict(q, dt)
        assert torch.equal(out.qavg, dt * q)
        assert not torch.any(out.favg)
        assert not torch.any(out.face_f)


def test_generator_matches_host_stream(stp, oracle):
    """The device generator reproduces the documented SplitMix64 stream bit-exactly."""
    S = stp
    for n in (3, 8):
        qd, pd = S.generate(0, 99, n, 7, 5, layout=S.LAYOUT_AOSOA, q_stride=9)
        qh, ph = oracle.generate(0, 99, n, 7, 5)
        assert np.array_equal(oracle.from_aosoa(n, 9, 9, qd.cpu().numpy()), qh)
        assert np.array_equal(pd.cpu().numpy(), ph)


def test_layout_conversion_roundtrip(stp, oracle):
    S = stp
    n, m, E = 6, 9, 7
    q, _ = S.generate(0, 3, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=12)
    aos = torch.empty(E, n ** 3 * 16, dtype=torch.float64, device="cuda")
    back = torch.empty_like(q)
    S.convert_layout(n, m, E, S.LAYOUT_AOSOA, 12, q, S.LAYOUT_AOS, 16, aos)
    S.convert_layout(n, m, E, S.LAYOUT_AOS, 16, aos, S.LAYOUT_AOSOA, 12, back)
    assert torch.equal(back, q)
    a = aos.cpu().numpy().reshape(E, n ** 3, 16)
    assert not np.any(a[:, :, m:])
    assert np.array_equal(a[:, :, :m].reshape(E, -1), oracle.from_aosoa(n, m, 12, q.cpu().numpy()))


@pytest.mark.parametrize("n", [4, 8, 10])
def test_edge_batches(stp, n):
    """0, 1 and odd element counts; deterministic (bit-identical reruns)."""
    S = stp
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=12, par_kind=S.PAR_RHO_CP_CS)
    q, par = S.generate(0, 1, n, 0, 3, layout=S.LAYOUT_AOSOA, q_stride=12)
    out0 = plan.predict(q[:0], 1e-3, par=par[:0])
    assert out0.qavg.shape[0] == 0
    a = plan.predict(q[:1], 1e-3, par=par[:1])
    b = plan.predict(q, 1e-3, par=par)
    c = plan.predict(q, 1e-3, par=par)
    plan.status()
    assert torch.equal(a.qavg[0], b.qavg[0]) and torch.equal(b.qavg, c.qavg) and torch.equal(b.face_f, c.face_f)


def test_input_checks(stp):
    """validate_stp semantics: non-finite DOFs and invalid material are reported."""
    S = stp
    for n in (4, 8, 10):
        plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=9, par_kind=S.PAR_LAMBDA_MU_RHO)
        q = torch.zeros(2, n ** 3 * 9, dtype=torch.float64, device="cuda")
        par = torch.tensor([[2.0, 1.0, 1.0], [2.0, 1.0, 1.0]], dtype=torch.float64, device="cuda")
        plan.predict(q, 0.01, par=par)
        plan.status()
        q[1, 5] = float("nan")
        plan.predict(q, 0.01, par=par)
        with pytest.raises(S.StpError) as e:
            plan.status()
        assert e.value.code == S.ADERSTP_ERR_NONFINITE
        q[1, 5] = 0.0
        par[0, 0] = -3.0  # lambda + 2 mu <= 0
        plan.predict(q, 0.01, par=par)
        with pytest.raises(S.StpError) as e:
            plan.status()
        assert e.value.code == S.ADERSTP_ERR_MATERIAL
        with pytest.raises(S.StpError):
            plan.predict(q, 0.0, par=par)  # dt <= 0


@pytest.mark.parametrize("n", [6, 8])
def test_host_path_matches_device_path(stp, n):
    S = stp
    E = 1000
    q, par = S.generate(0, 11, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=12)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=12, par_kind=S.PAR_RHO_CP_CS)
    plan.reserve_host_path(97)  # several chunks, ragged last chunk
    dev = plan.predict(q, 2e-3, par=par)
    host = plan.predict_host(q.cpu().numpy(), 2e-3, par=par.cpu().numpy())
    for name in ("qavg", "favg", "face_q", "face_f"):
        assert np.array_equal(getattr(dev, name).cpu().numpy(), getattr(host, name)), name


def test_full_size_linearity_and_sampled_parity(stp, oracle):
    """C3 at full size (131,072 elements): the STP is linear in q, so
    STP(a q1 + b q2) = a STP(q1) + b STP(q2) per element; plus oracle parity on a sample."""
    S = stp
    n, E = 8, 131072
    q1, par = S.generate(0, 21, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=12)
    q2, _ = S.generate(0, 22, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=12)
    dt = 0.5 / (3 * 6.0 * 15)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=12, par_kind=S.PAR_RHO_CP_CS)
    o1 = plan.predict(q1, dt, par=par)
    o2 = plan.predict(q2, dt, par=par)
    oc = plan.predict(0.75 * q1 - 1.25 * q2, dt, par=par)
    plan.status()
    for name in ("qavg", "face_q", "face_f"):
        want = 0.75 * getattr(o1, name) - 1.25 * getattr(o2, name)
        got = getattr(oc, name)
        err = (got - want).abs().reshape(E, -1).amax(1) / want.abs().reshape(E, -1).amax(1)
        assert float(err.max()) < 1e-12, name
    idx = torch.tensor([0, 1, 4097, 65536, E - 1], device="cuda")
    qs = q1[idx].cpu().numpy()
    ref = oracle.stp(n, 9, oracle.from_aosoa(n, 9, 12, qs), dt, par=oracle.material_lmr(par[idx].cpu().numpy()))
    got = oracle.from_aosoa(n, 9, 9, o1.qavg[idx].cpu().numpy())
    assert O.per_element_rel_diff(ref.qavg, got) <= TOL
    assert O.per_element_rel_diff(ref.face_f.reshape(5, -1), o1.face_f[idx].cpu().numpy().reshape(5, -1)) <= TOL


def test_dense_volume_operator_taylor_series(stp, oracle):
    """acceptance criterion 2: (N,m) = (4,9) elastic vs the dense V power series."""
    S = stp
    from test_oracle import _dense_volume_operator, _elastic_A, _taylor
    n = 4
    b = oracle.basis(n)
    lam, mu, rho = 2.0, 1.0, 1.0
    rng = np.random.default_rng(2024)
    qc = rng.uniform(-1, 1, n ** 3 * 9)
    dt = 0.4 / (3 * 2.0 * 7)
    want = _taylor(_dense_volume_operator(b, _elastic_A(lam, mu, rho)), qc, n, dt)
    plan = S.Plan(n, S.elastic_pde(lam, mu, rho), layout=S.LAYOUT_AOSOA)
    out = plan.predict(torch.from_numpy(oracle.to_aosoa(n, 9, 9, qc[None])).cuda(), dt)
    got = oracle.from_aosoa(n, 9, 9, out.qavg.cpu().numpy())[0]
    assert O.rel_diff(want, got) < 1e-11


@pytest.mark.parametrize("n", [3, 6, 8, 9, 10])
def test_aos_staged_path_matches_generic_and_oracle(stp, oracle, monkeypatch, n):
    """The reference layout (AoS, m_pad 16) runs straight through stp_dmma8 / stp_bip (nDof 8-10) or through
    device transposes and the tuned kernel; the generic kernel (ADERSTP_FORCE_GENERIC) on the same
    AoS buffers and the oracle agree."""
    S = stp
    E = 11
    q, par = S.generate(1, 77 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    aos = torch.empty(E, n ** 3 * 16, dtype=torch.float64, device="cuda")
    S.convert_layout(n, 9, E, S.LAYOUT_AOSOA, 9, q, S.LAYOUT_AOS, 16, aos)
    par_h = par.cpu().numpy()
    dt = O.cfl_dt(n, par_h[:, 1].max())
    ref = oracle.stp(n, 9, oracle.from_aosoa(n, 9, 9, q.cpu().numpy()), dt, par=oracle.material_lmr(par_h))
    # default (nDof 8: straight into stp_dmma8), the transposes (one chunk, three chunks with the
    # last ragged), the generic kernel on the AoS buffers
    for generic, chunk, staged in (("0", "0", "0"), ("0", "0", "1"), ("0", "4", "1"), ("1", "0", "0")):
        monkeypatch.setenv("ADERSTP_FORCE_GENERIC", generic)
        monkeypatch.setenv("ADERSTP_AOS_CHUNK", chunk)
        monkeypatch.setenv("ADERSTP_AOS_STAGED", staged)
        plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOS, q_stride=16, out_stride=16, par_kind=S.PAR_RHO_CP_CS)
        out = plan.predict(aos, dt, par=par)
        plan.status()
        worst = _compare(S, oracle, n, out, ref, S.LAYOUT_AOS, 16)
        assert max(worst.values()) <= TOL, (generic, staged, worst)
        qa = out.qavg.cpu().numpy().reshape(E, n ** 3, 16)
        assert not np.any(qa[:, :, 9:])
        if generic == "0" and chunk == "0":  # the host-buffer path takes the same device route
            host = plan.predict_host(aos.cpu().numpy(), dt, par=par_h)
            assert np.array_equal(host.qavg, out.qavg.cpu().numpy())
            assert np.array_equal(host.face_f, out.face_f.cpu().numpy())


def test_aos_plan_alone_in_a_fresh_process(stp):
    """An AoS plan must upload the device constants of the kernels its staged path uses even
    when no native-layout plan was ever created in the process."""
    import subprocess
    import sys
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle as O, paper_2003_12787_b200 as S
orc = O.Oracle()
worst = 0.0
for n in (4, 8, 10):
    E = 5
    q, par = S.generate(0, 3 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    qc = orc.from_aosoa(n, 9, 9, q.cpu().numpy())
    aos = np.zeros((E, n ** 3, 16)); aos[:, :, :9] = qc.reshape(E, n ** 3, 9)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOS, q_stride=16, out_stride=16, par_kind=S.PAR_RHO_CP_CS)
    dt = O.cfl_dt(n, float(par[:, 1].max()))
    out = plan.predict(torch.from_numpy(aos.reshape(E, -1)).cuda(), dt, par=par)
    plan.status()
    ref = orc.stp(n, 9, qc, dt, par=orc.material_lmr(par.cpu().numpy()))
    got = out.qavg.cpu().numpy().reshape(E, n ** 3, 16)[:, :, :9].reshape(E, -1)
    worst = max(worst, O.per_element_rel_diff(ref.qavg, got))
print(worst)
""" % _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TOL


@pytest.mark.parametrize("n", [6, 8, 9, 10])
def test_reference_layout_checks_and_edges(stp, oracle, n):
    """The reference (AoS, m_pad 16) layout on the tuned paths: non-finite DOFs flagged (slot 8
    of a node is the tail of a 16-byte pair), padding slots never read (NaN there is harmless),
    empty batch, and an unaligned batch (staged through the generic transposes) agreeing with the
    aligned one."""
    S = stp
    E = 6
    q, par = S.generate(0, 5 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    aos = torch.empty(E, n ** 3 * 16, dtype=torch.float64, device="cuda")
    S.convert_layout(n, 9, E, S.LAYOUT_AOSOA, 9, q, S.LAYOUT_AOS, 16, aos)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOS, q_stride=16, out_stride=16, par_kind=S.PAR_RHO_CP_CS,
                  check_inputs=True)
    dt = O.cfl_dt(n, float(par[:, 1].max()))
    assert plan.predict(aos[:0], dt, par=par[:0]).qavg.shape[0] == 0
    ref = plan.predict(aos, dt, par=par)
    plan.status()
    padded = aos.clone().view(E, n ** 3, 16)
    padded[:, :, 9:] = float("nan")  # ElementTensor padding lanes are never read
    out = plan.predict(padded.view(E, -1), dt, par=par)
    plan.status()
    assert torch.equal(out.qavg, ref.qavg) and torch.equal(out.face_f, ref.face_f)
    for slot in (0, 8):
        bad = aos.clone().view(E, n ** 3, 16)
        bad[E - 1, n ** 3 - 1, slot] = float("inf")
        plan.predict(bad.view(E, -1), dt, par=par)
        with pytest.raises(S.StpError) as e:
            plan.status()
        assert e.value.code == S.ADERSTP_ERR_NONFINITE
    # an 8-byte offset batch cannot take the 16-byte paths: generic transposes, same results
    buf = torch.empty(E * n ** 3 * 16 + 1, dtype=torch.float64, device="cuda")
    buf[1:].copy_(aos.view(-1))
    qoff = buf[1:].view(E, -1)
    o2 = S.PredictorOutput(*(torch.empty(t.numel() + 1, dtype=torch.float64, device="cuda")[1:].view(t.shape)
                             for t in (ref.qavg, ref.favg, ref.face_q, ref.face_f)))
    plan.predict(qoff, dt, par=par, out=o2)
    plan.status()
    for a, b in ((o2.qavg, ref.qavg), (o2.favg, ref.favg), (o2.face_q, ref.face_q), (o2.face_f, ref.face_f)):
        assert O.per_element_rel_diff(b.cpu().numpy().reshape(E, -1), a.cpu().numpy().reshape(E, -1)) <= TOL


@pytest.mark.parametrize("n", [4, 5, 6, 7, 8, 9, 10])
@pytest.mark.parametrize("case", ["advection_m3", "ncp_advection_m2", "demo_m6", "probed_m5", "probed_m8", "probed_m9"])
def test_table_pdes_on_tensor_cores(stp, oracle, monkeypatch, case, n):
    """Table PDEs (the user-LinearPde path) on their tuned kernels: stp_dmma8_table at nDof 8,
    stp_dmmat (zero-padded tiles) at nDof 5..7, the line-pass table kernel stp_tlp at nDof 9, 10
    (nDof 4: the generic kernel); the reference's PDEs against the oracle, random
    probed systems (flux + ncp matrices) against the unmodified reference's predict() on a
    MatrixPde with the same matrices; all against the generic table kernel on the same inputs."""
    S = stp
    E = 7
    rng = np.random.default_rng(_zlib.crc32(case.encode()) + n)
    if case == "advection_m3":
        m, pde, kind, args = 3, S.advection_pde((1.0, 0.5, 0.25), 3), O.PDE_ADVECTION, [1.0, 0.5, 0.25]
    elif case == "ncp_advection_m2":
        m, pde, kind, args = 2, S.ncp_advection_pde((1.0, 0.5, 0.25), 2), O.PDE_NCP_ADVECTION, [1.0, 0.5, 0.25]
    elif case == "demo_m6":
        m, pde, kind, args = 6, S.paper_demo_pde(), O.PDE_DEMO, []
    else:
        m = int(case[-1])
        A, B = [], []
        for _ in range(3):
            a, b = np.zeros((m, m)), np.zeros((m, m))
            for r in range(m):  # two flux and one ncp nonzero per row
                a[r, rng.choice(m, 2, replace=False)] = rng.uniform(-1, 1, 2)
                b[r, rng.integers(m)] = rng.uniform(-0.5, 0.5)
            A.append(a)
            B.append(b)
        pde, kind, args = S.linear_pde(A, B), None, None
    qn = rng.uniform(-1, 1, (E, n ** 3 * m))
    q = torch.from_numpy(oracle.to_aosoa(n, m, m, qn)).cuda()
    dt = 2e-3
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=m, out_stride=m)
    out = plan.predict(q, dt)
    plan.status()
    if kind is not None:
        ref = oracle.stp(n, m, qn, dt, pde_kind=kind, args=args)
    else:  # the reference itself on a user LinearPde defined by the same matrices (MatrixPde)
        if not O.reference_available():
            pytest.skip("oracle/_ref not built")
        ref = O.Reference().stp_matrix(n, m, qn, dt, A, B)
    worst = _compare(S, oracle, n, out, ref, S.LAYOUT_AOSOA, m, m=m)
    assert max(worst.values()) <= TOL, worst
    monkeypatch.setenv("ADERSTP_FORCE_GENERIC", "1")
    gplan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=m, out_stride=m)
    gen = gplan.predict(q, dt)
    gplan.status()
    for x, y in ((out.qavg, gen.qavg), (out.favg, gen.favg), (out.face_q, gen.face_q), (out.face_f, gen.face_f)):
        assert O.per_element_rel_diff(y.cpu().numpy().reshape(E, -1), x.cpu().numpy().reshape(E, -1)) <= TOL


@pytest.mark.parametrize("n", [8, 9, 10])
@pytest.mark.parametrize("case", ["advection_m3", "demo_m6"])
def test_table_pdes_reference_layout_nDof8(stp, oracle, case, n):
    """The reference layout (AoS, m_pad = 8 for m <= 8, layout.cpp:9-21) of a table PDE at nDof 8
    goes through the device transposes to stp_dmma8_table (nDof 9, 10: stp_tlp, the padded AoSoA
    staging with out_stride 8); it agrees with the oracle and the padding slots stay zero."""
    S = stp
    E = 5
    m, pde, kind, args = ((3, S.advection_pde((1.0, 0.5, 0.25), 3), O.PDE_ADVECTION, [1.0, 0.5, 0.25])
                          if case == "advection_m3" else (6, S.paper_demo_pde(), O.PDE_DEMO, []))
    rng = np.random.default_rng(_zlib.crc32(case.encode()) + 1)
    qn = rng.uniform(-1, 1, (E, n ** 3 * m))
    aos = np.zeros((E, n ** 3, 8))
    aos[:, :, :m] = qn.reshape(E, n ** 3, m)
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOS, q_stride=8, out_stride=8)
    out = plan.predict(torch.from_numpy(aos.reshape(E, -1)).cuda(), 2e-3)
    plan.status()
    ref = oracle.stp(n, m, qn, 2e-3, pde_kind=kind, args=args)
    worst = _compare(S, oracle, n, out, ref, S.LAYOUT_AOS, 8, m=m)
    assert max(worst.values()) <= TOL, worst
    assert not np.any(out.qavg.cpu().numpy().reshape(E, n ** 3, 8)[:, :, m:])


@pytest.mark.parametrize("n", [9, 10])
def test_table_pde_line_pass_edges(stp, oracle, monkeypatch, n):
    """stp_tlp (table PDEs at nDof 9, 10) on padded AoSoA strides (q_stride, out_stride > m: the
    output padding slots are written as zeros), a single-quantity system (32 face groups per warp),
    an empty batch and a non-finite input, against the generic table kernel and the oracle."""
    S = stp
    E = 3
    rng = np.random.default_rng(11 + n)
    for m, pde, kind, args, qs, os_ in ((3, S.advection_pde((1.0, 0.5, 0.25), 3), O.PDE_ADVECTION, [1.0, 0.5, 0.25], 5, 4),
                                        (1, S.advection_pde((0.3, -0.7, 0.2), 1), O.PDE_ADVECTION, [0.3, -0.7, 0.2], 1, 1)):
        qn = rng.uniform(-1, 1, (E, n ** 3 * m))
        q = torch.from_numpy(oracle.to_aosoa(n, m, qs, qn)).cuda()
        plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=qs, out_stride=os_)
        out = plan.predict(q, 2e-3)
        plan.status()
        ref = oracle.stp(n, m, qn, 2e-3, pde_kind=kind, args=args)
        worst = _compare(S, oracle, n, out, ref, S.LAYOUT_AOSOA, os_, m=m)
        assert max(worst.values()) <= TOL, (m, worst)
        if os_ > m:  # padding slots of qavg / favg are exact zeros
            qa = out.qavg.cpu().numpy().reshape(E, n, n, os_, n)
            fa = out.favg.cpu().numpy().reshape(E, 3, n, n, os_, n)
            assert not np.any(qa[:, :, :, m:, :]) and not np.any(fa[:, :, :, :, m:, :])
        monkeypatch.setenv("ADERSTP_FORCE_GENERIC", "1")
        gplan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=qs, out_stride=os_)
        gen = gplan.predict(q, 2e-3)
        gplan.status()
        monkeypatch.delenv("ADERSTP_FORCE_GENERIC")
        for x, y in ((out.qavg, gen.qavg), (out.favg, gen.favg), (out.face_q, gen.face_q), (out.face_f, gen.face_f)):
            assert O.per_element_rel_diff(y.cpu().numpy().reshape(E, -1), x.cpu().numpy().reshape(E, -1)) <= TOL
        empty = plan.predict(q[:0], 2e-3)
        plan.status()
        assert empty.qavg.shape[0] == 0
        cplan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=qs, out_stride=os_, check_inputs=True)
        pad = q.clone()  # a NaN in a padding slot (s >= m) is never read: no flag
        if qs > m:
            pad[E - 1, ((n * n - 1) * qs + m) * n] = float("nan")
        cplan.predict(pad, 2e-3)
        cplan.status()
        bad = q.clone()  # quantity 0 of the last node of the last element
        bad[E - 1, ((n * n - 1) * qs) * n + n - 1] = float("nan")
        cplan.predict(bad, 2e-3)
        with pytest.raises(S.StpError) as err:
            cplan.status()
        assert err.value.code == S.ADERSTP_ERR_NONFINITE
