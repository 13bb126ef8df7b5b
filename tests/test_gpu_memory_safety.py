"""Memory-safety evidence for every kernel family without compute-sanitizer (closed on this GPU
pool: runs under it left GPUs needing a reset).

* Out-of-bounds WRITES: every output array lives inside a larger allocation whose guard bands
  before and after hold a canary bit pattern; after the launch the canaries must be intact, and
  so must the padding lanes the kernels must not touch.
* Out-of-bounds READS: the batch is a slice of a larger tensor whose neighbouring elements (and
  the padding slots of q, and the neighbouring material rows) are NaN; any read outside the
  element's own data would poison its outputs (checked against the oracle, and by the kernels'
  own non-finite check).
* Shared-memory races: a race shows up as run-to-run differences; each family is re-run with
  the batch at a different offset inside the poisoned tensor and under a CUDA graph replay, and
  the results must be bit-identical.
"""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CANARY = np.frombuffer(np.uint64(0x7FF4DEADBEEF0001).tobytes(), dtype=np.float64)[0]  # a quiet-NaN payload
GUARD = 4096  # doubles on each side


@pytest.fixture(scope="module")
def stp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_12787_b200 as S
    return S


def _guarded(shape):
    """A tensor of `shape` in the middle of a canary-filled buffer; returns (view, buffer)."""
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), float(CANARY), dtype=torch.float64, device="cuda")
    return buf[GUARD:GUARD + n].view(shape), buf


def _canaries_intact(buf, n):
    b = buf.cpu().numpy().view(np.uint64)
    want = np.uint64(0x7FF4DEADBEEF0001)
    return bool(np.all(b[:GUARD] == want) and np.all(b[GUARD + n:] == want))


FAMILIES = [  # (name, nDof, env, q layout, q stride)
    ("dmma8", 8, {}, "aosoa", 12),
    ("dmma8_aos", 8, {}, "aos", 16),
    ("dmmap4", 4, {}, "aosoa", 12),
    ("dmmap6", 6, {}, "aosoa", 9),
    ("dmmap7_aos", 7, {}, "aos", 16),
    ("bip9", 9, {}, "aosoa", 12),
    ("bip10", 10, {}, "aosoa", 9),
    ("bip10_aos", 10, {}, "aos", 16),
    ("pass3", 3, {}, "aosoa", 12),
    ("pass8", 8, {"ADERSTP_NO_DMMA8": "1"}, "aosoa", 9),
    ("generic5", 5, {"ADERSTP_FORCE_GENERIC": "1"}, "aosoa", 12),
    ("staged3_aos", 3, {}, "aos", 16),
]


@pytest.mark.parametrize("name,n,env,lay,qs", FAMILIES, ids=[f[0] for f in FAMILIES])
def test_guard_bands_and_poisoned_neighbours(stp, oracle, monkeypatch, name, n, env, lay, qs):
    S = stp
    for k in ("ADERSTP_NO_DMMA8", "ADERSTP_NO_DMMAP", "ADERSTP_FORCE_GENERIC", "ADERSTP_PASS_SLOTS"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    E, off = 7, 3
    layout = S.LAYOUT_AOS if lay == "aos" else S.LAYOUT_AOSOA
    ostride = 16 if lay == "aos" else 9
    q9, par = S.generate(0, 100 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    # poisoned input tensor: NaN everywhere except the batch's real entries
    big = torch.full((E + 2 * off, n ** 3 * qs), float("nan"), dtype=torch.float64, device="cuda")
    if lay == "aos":
        tmp = torch.empty(E, n ** 3 * 16, dtype=torch.float64, device="cuda")
        S.convert_layout(n, 9, E, S.LAYOUT_AOSOA, 9, q9, S.LAYOUT_AOS, 16, tmp)
        view = big[off:off + E].view(E, n ** 3, 16)
        view[:, :, :9] = tmp.view(E, n ** 3, 16)[:, :, :9]  # padding slots stay NaN
    else:
        view = big[off:off + E].view(E, n, n, qs, n)
        view[:, :, :, :9, :] = q9.view(E, n, n, 9, n)      # padding slots stay NaN
    pbig = torch.full((E + 2 * off, 3), float("nan"), dtype=torch.float64, device="cuda")
    pbig[off:off + E] = par
    q = big[off:off + E]
    p = pbig[off:off + E]
    plan = S.Plan(n, S.elastic_pde(), layout=layout, q_stride=qs, out_stride=ostride, par_kind=S.PAR_RHO_CP_CS,
                  check_inputs=True)
    shapes = [(E, n ** 3 * ostride), (E, 3, n ** 3 * ostride), (E, 6, n * n * 9), (E, 6, n * n * 9)]
    views, bufs = zip(*[_guarded(s) for s in shapes])
    out = S.PredictorOutput(*views)
    dt = O.cfl_dt(n, float(par[:, 1].max()))
    plan.predict(q, dt, par=p, out=out)
    plan.status()  # raises if any NaN (a neighbour or a padding slot) was read as data
    torch.cuda.synchronize()
    for s, b in zip(shapes, bufs):
        assert _canaries_intact(b, int(np.prod(s))), (name, s)
    ref = oracle.stp(n, 9, oracle.from_aosoa(n, 9, 9, q9.cpu().numpy()), dt, par=oracle.material_lmr(par.cpu().numpy()))
    if lay == "aos":
        qa = out.qavg.cpu().numpy().reshape(E, n ** 3, 16)
        assert not np.any(qa[:, :, 9:])  # output padding lanes written as zeros, nothing else
        got = qa[:, :, :9].reshape(E, -1)
    else:
        got = oracle.from_aosoa(n, 9, 9, out.qavg.cpu().numpy())
    assert O.per_element_rel_diff(ref.qavg, got) <= 1e-12
    assert O.per_element_rel_diff(ref.face_f.reshape(E, -1), out.face_f.cpu().numpy().reshape(E, -1)) <= 1e-12
    # race check by repetition: another offset, eager and graph-replayed, bit-identical outputs
    q2 = torch.full_like(big, float("nan"))
    q2[2 * off - 1:2 * off - 1 + E] = q
    p2 = torch.full_like(pbig, float("nan"))
    p2[2 * off - 1:2 * off - 1 + E] = p
    o2 = plan.alloc_output(E)
    g = torch.cuda.CUDAGraph()
    plan.predict(q2[2 * off - 1:2 * off - 1 + E], dt, par=p2[2 * off - 1:2 * off - 1 + E], out=o2)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        plan.predict(q2[2 * off - 1:2 * off - 1 + E], dt, par=p2[2 * off - 1:2 * off - 1 + E], out=o2)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        for a, b in ((o2.qavg, out.qavg), (o2.favg, out.favg), (o2.face_q, out.face_q), (o2.face_f, out.face_f)):
            assert torch.equal(a, b), name
    plan.status()


@pytest.mark.parametrize("n", [4, 8, 10])
def test_time_loop_guard_bands(stp, n):
    """The fused time step (predictor writing u in place + the surface corrector) on a guarded
    mesh state: nothing outside the e^3 elements is touched."""
    S = stp
    e = 3
    E = e ** 3
    q, par = S.generate(0, 9, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    u, buf = _guarded((E, n ** 3 * 9))
    u.copy_(q * 1e-3)
    pg, pbuf = _guarded((E, 3))
    pg.copy_(par)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    ok, steps, _ = plan.run_simulation(u, e, 1e-3, par=pg, cfl=0.35)
    torch.cuda.synchronize()
    assert ok and steps >= 1
    assert _canaries_intact(buf, E * n ** 3 * 9) and _canaries_intact(pbuf, E * 3)
    assert bool(torch.isfinite(u).all())


def _dense_pde(S, m, seed):
    rng = np.random.default_rng(seed)
    A = [rng.uniform(-1, 1, (m, m)) / m for _ in range(3)]
    B = [rng.uniform(-0.5, 0.5, (m, m)) / m for _ in range(3)]
    return S.linear_pde(A, B), A, B


USER_FAMILIES = [  # (name, nDof, pde, m, q stride, out stride): the user-LinearPde kernels
    ("tlp9_adv", 9, "advection", 8, 10, 8),
    ("tlp10_demo", 10, "demo", 6, 6, 7),
    ("dmmat6_adv", 6, "advection", 3, 3, 3),
    ("dmma8_table_demo", 8, "demo", 6, 6, 6),
    ("general6_dense12", 6, "dense", 12, 12, 12),
    ("generic4_adv", 4, "advection", 3, 4, 4),
]


@pytest.mark.parametrize("name,n,kind,m,qs,os_", USER_FAMILIES, ids=[f[0] for f in USER_FAMILIES])
def test_user_pde_kernels_guard_bands_and_poisoned_neighbours(stp, oracle, name, n, kind, m, qs, os_):
    """The user-LinearPde kernels (line-pass table kernel, DMMA table kernels, general, generic):
    guard bands around every output, NaN neighbours and NaN padding slots in the input, results
    against the oracle / the reference, bit-identical on another offset under a graph replay."""
    S = stp
    E, off = 5, 2
    if kind == "advection":
        pde, ref_kw = S.advection_pde((1.0, 0.5, 0.25), m), dict(pde_kind=O.PDE_ADVECTION, args=[1.0, 0.5, 0.25])
    elif kind == "demo":
        pde, ref_kw = S.paper_demo_pde(), dict(pde_kind=O.PDE_DEMO, args=[])
    else:
        pde, A, B = _dense_pde(S, m, 3)
        ref_kw = None
    rng = np.random.default_rng(len(name) + n)
    qn = rng.uniform(-1, 1, (E, n ** 3 * m))
    big = torch.full((E + 2 * off, n ** 3 * qs), float("nan"), dtype=torch.float64, device="cuda")
    big[off:off + E] = torch.from_numpy(oracle.to_aosoa(n, m, qs, qn)).cuda()
    big.view(E + 2 * off, n, n, qs, n)[:, :, :, m:, :] = float("nan")  # padding slots stay NaN
    q = big[off:off + E]
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=qs, out_stride=os_, check_inputs=True)
    shapes = [(E, n ** 3 * os_), (E, 3, n ** 3 * os_), (E, 6, n * n * m), (E, 6, n * n * m)]
    views, bufs = zip(*[_guarded(s) for s in shapes])
    out = S.PredictorOutput(*views)
    dt = 2e-3
    plan.predict(q, dt, out=out)
    plan.status()  # raises if a NaN neighbour or padding slot was read as data
    torch.cuda.synchronize()
    for s, b in zip(shapes, bufs):
        assert _canaries_intact(b, int(np.prod(s))), (name, s)
    if ref_kw is not None:
        ref = oracle.stp(n, m, qn, dt, **ref_kw)
    else:
        if not O.reference_available():
            pytest.skip("oracle/_ref not built")
        ref = O.Reference().stp_matrix(n, m, qn, dt, A, B)
    got = oracle.from_aosoa(n, m, os_, out.qavg.cpu().numpy())
    assert O.per_element_rel_diff(ref.qavg, got) <= 1e-12
    assert O.per_element_rel_diff(ref.face_f.reshape(E, -1), out.face_f.cpu().numpy().reshape(E, -1)) <= 1e-12
    if os_ > m:
        assert not np.any(out.qavg.cpu().numpy().reshape(E, n, n, os_, n)[:, :, :, m:, :])
    q2 = torch.full_like(big, float("nan"))
    q2[2 * off - 1:2 * off - 1 + E] = q
    o2 = plan.alloc_output(E)
    plan.predict(q2[2 * off - 1:2 * off - 1 + E], dt, out=o2)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.predict(q2[2 * off - 1:2 * off - 1 + E], dt, out=o2)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        for a, b in ((o2.qavg, out.qavg), (o2.favg, out.favg), (o2.face_q, out.face_q), (o2.face_f, out.face_f)):
            assert torch.equal(a, b), name
    plan.status()
