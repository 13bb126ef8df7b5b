"""The BASELINE.json configs at their full sizes, through the same calls bench.py times.

* the device input generator for every distribution the configs use (C1/C3/C5 U[-1,1], C4 Box-
  Muller N(0,1), C2 random-phase sinusoids on the 32^3 periodic grid) against the host stream of
  the oracle;
* C2 (nDof 6, 32,768 elements) and C4 (nDof 10, 65,536 elements) at full size: oracle parity on
  sampled elements including the first and the last;
* C5 (nDof 8, 1,048,576 elements) through bench.py's chunked launch loop (8 launches of 131,072,
  output buffers reused): oracle parity on the elements either side of every chunk boundary.

Tolerance: the reference's rel_diff per element and output array (proj/src/checks.cpp:27-34),
<= 1e-12 (BASELINE.json north_star).
"""
import os
import sys

import numpy as np
import pytest

import oracle as O

TOL = 1e-12
SEED = 20031278  # bench.py SEED
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def stp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_12787_b200 as S
    return S


@pytest.fixture(scope="module")
def bench():
    sys.path.insert(0, ROOT)
    import bench as B
    return B


def _check_outputs(S, oracle, n, q_rows, par_rows, dt, out_rows, q_stride):
    """oracle STP of the sampled rows vs the GPU's outputs of the same rows."""
    k = q_rows.shape[0]
    ref = oracle.stp(n, 9, oracle.from_aosoa(n, 9, q_stride, q_rows), dt, par=oracle.material_lmr(par_rows))
    qavg, favg, face_q, face_f = out_rows
    worst = {"qavg": O.per_element_rel_diff(ref.qavg, oracle.from_aosoa(n, 9, 9, qavg)),
             "favg": max(O.per_element_rel_diff(ref.favg[:, d], oracle.from_aosoa(n, 9, 9, favg[:, d]))
                         for d in range(3)),
             "face_q": O.per_element_rel_diff(ref.face_q.reshape(k, -1), face_q.reshape(k, -1)),
             "face_f": O.per_element_rel_diff(ref.face_f.reshape(k, -1), face_f.reshape(k, -1))}
    assert max(worst.values()) <= TOL, worst
    return worst


@pytest.mark.parametrize("dist,n,e0,grid", [(0, 8, 1048570, 1), (1, 10, 65530, 1), (1, 9, 3, 1),
                                            (2, 6, 0, 32), (2, 6, 32767 - 5, 32)])
def test_generator_all_distributions(stp, oracle, dist, n, e0, grid):
    """Device generator vs the oracle's host generator: the SplitMix64 draws and the material are
    bit-identical; the transcendental distributions (Box-Muller log/cos, sinusoids) agree to the
    last ulps (CUDA's and glibc's log/sin/cos may round differently).  The parity tests never
    depend on this: they copy the device-generated inputs to the oracle."""
    S = stp
    E = 6
    qd, pd = S.generate(dist, SEED, n, e0, E, grid=grid, layout=S.LAYOUT_AOSOA, q_stride=9)
    qh, ph = oracle.generate(dist, SEED, n, e0, E, grid=grid)
    qd = oracle.from_aosoa(n, 9, 9, qd.cpu().numpy())
    assert np.array_equal(pd.cpu().numpy(), ph)
    if dist == 0:
        assert np.array_equal(qd, qh)
    else:
        # Box-Muller: a few ulps; sinusoids: the phase argument (up to ~40 rad) carries the
        # rounding of both sides' sin/range reduction, ~1e-15 absolute per unit of argument
        err = np.max(np.abs(qd - qh)) / np.max(np.abs(qh))
        assert err <= (4e-15 if dist == 1 else 2e-14), err


def test_generator_distribution_properties(stp):
    """Size-independent checks of the configs' inputs: C4's N(0,1) has mean 0 and variance 1;
    C2's sinusoids are periodic on the 32^3 grid (the left face of element ex = 0 continues the
    right face of ex = 31 exactly as the Lagrange extrapolation of a smooth function would) and
    bounded by the sum of the three amplitudes (<= 3)."""
    S = stp
    q, _ = S.generate(1, SEED, 10, 0, 4096, layout=S.LAYOUT_AOSOA, q_stride=9)
    x = q.view(-1)
    assert abs(float(x.mean())) < 3e-3 and abs(float(x.var()) - 1.0) < 3e-3
    q2, _ = S.generate(2, SEED, 6, 0, 32768, grid=32, layout=S.LAYOUT_AOSOA, q_stride=9)
    assert float(q2.abs().max()) <= 3.0
    # every element's field is a smooth periodic function: the x-extrapolations of neighbours
    # across the periodic boundary agree to the interpolation error of a degree-5 polynomial
    b = S.make_basis(6)
    v = q2.view(32, 32, 32, 6, 6, 9, 6).cpu().numpy()  # [ez][ey][ex][k3][k2][s][k1]
    right = np.einsum("zyxabsk,k->zyxabs", v[:, :, 31:32], b.face_right)
    left = np.einsum("zyxabsk,k->zyxabs", v[:, :, 0:1], b.face_left)
    assert np.max(np.abs(right - left)) < 1e-4


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_full_size_config_parity(stp, oracle, bench, name):
    """C2 and C4 as bench.py runs them (same generator call, plan and dt), oracle parity on the
    first, last and 8 interior elements."""
    S, B = stp, bench
    cfg = B.CONFIGS[name]
    n, E = cfg["n"], cfg["elems"]
    grid = round(E ** (1.0 / 3.0)) if cfg["dist"] == 2 else 1
    q, par = S.generate(cfg["dist"], B.SEED, n, 0, E, grid=grid, layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"])
    plan = B.make_plan(S, cfg)
    dt = B.config_dt(n)
    out = plan.predict(q, dt, par=par)
    plan.status()
    rng = np.random.default_rng(E)
    idx = torch.tensor(sorted({0, E - 1, *rng.integers(1, E - 1, 8).tolist()}), device="cuda")
    _check_outputs(S, oracle, n, q[idx].cpu().numpy(), par[idx].cpu().numpy(), dt,
                   (out.qavg[idx].cpu().numpy(), out.favg[idx].cpu().numpy(),
                    out.face_q[idx].cpu().numpy(), out.face_f[idx].cpu().numpy()), cfg["q_stride"])


@pytest.mark.parametrize("n,E", [(4, 8192), (4, 40000), (5, 32768), (5, 40001)])
def test_ndof4_large_batch_dispatch_parity(stp, oracle, monkeypatch, n, E):
    """nDof 4 from 8,192 and nDof 5 from 32,768 elements on run on the warp-per-element kernel
    (csrc/stp_wpe.cu, kWpeMinElems4 / 5; persistent warps walking several elements each, ragged
    last rounds): oracle parity on the first, last and 30 interior elements, and agreement with the
    padded-DMMA kernel (ADERSTP_WPE=0) on every element."""
    S = stp
    monkeypatch.delenv("ADERSTP_WPE", raising=False)
    q, par = S.generate(0, SEED, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    dt = O.cfl_dt(n, 6.0)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    out = plan.predict(q, dt, par=par)
    plan.status()
    rng = np.random.default_rng(E)
    idx = torch.tensor(sorted({0, E - 1, *rng.integers(1, E - 1, 30).tolist()}), device="cuda")
    _check_outputs(S, oracle, n, q[idx].cpu().numpy(), par[idx].cpu().numpy(), dt,
                   (out.qavg[idx].cpu().numpy(), out.favg[idx].cpu().numpy(),
                    out.face_q[idx].cpu().numpy(), out.face_f[idx].cpu().numpy()), 9)
    again = plan.predict(q, dt, par=par)  # deterministic: a rerun is bit-identical (SURVEY 8(b) determinism)
    plan.status()
    assert all(torch.equal(x, y) for x, y in ((out.qavg, again.qavg), (out.favg, again.favg),
                                              (out.face_q, again.face_q), (out.face_f, again.face_f)))
    monkeypatch.setenv("ADERSTP_WPE", "0")
    plan0 = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    out0 = plan0.predict(q, dt, par=par)
    plan0.status()
    for a, b in ((out.qavg, out0.qavg), (out.favg, out0.favg), (out.face_q, out0.face_q), (out.face_f, out0.face_f)):
        a2, b2 = a.reshape(E, -1), b.reshape(E, -1)
        scale = torch.maximum(b2.abs().amax(dim=1), torch.tensor(1e-300, device="cuda", dtype=torch.float64))
        assert float(((a2 - b2).abs().amax(dim=1) / scale).max()) <= TOL


@pytest.mark.parametrize("name", ["c5", "c5n6"])
def test_c5_chunked_launch_loop_parity(stp, oracle, bench, name):
    """C5 through bench.py's own loop: the rank's shard of 1,048,576 elements resident in HBM,
    streamed through fixed-size launches with reused output buffers; elements on both sides of
    every chunk boundary (and the first / last) against the oracle, and each sampled element's
    inputs against the host generator at its global index."""
    S, B = stp, bench
    cfg = B.CONFIGS[name]
    n = cfg["n"]
    sh = B.shard_of(cfg, 1, 0)
    chunk = cfg["chunk"]
    q, par = S.generate(cfg["dist"], B.SEED, n, sh.start, sh.count, layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"])
    plan = B.make_plan(S, cfg)
    dt = B.config_dt(n)
    out = plan.alloc_output(chunk)
    checked = 0
    for s0, c in B.chunks(sh, chunk):
        off = s0 - sh.start
        o = S.PredictorOutput(out.qavg[:c], out.favg[:c], out.face_q[:c], out.face_f[:c])
        plan.predict(q[off:off + c], dt, par=par[off:off + c], out=o)
        plan.status()
        local = [0, 1, c - 1]  # first elements after the previous boundary, last before the next
        g = torch.tensor(local, device="cuda")
        q_rows = q[off:off + c][g].cpu().numpy()
        qh, ph = oracle.generate(cfg["dist"], B.SEED, n, s0 + c - 1, 1)
        assert np.array_equal(oracle.from_aosoa(n, 9, cfg["q_stride"], q_rows[2:3]), qh)
        _check_outputs(S, oracle, n, q_rows, par[off:off + c][g].cpu().numpy(), dt,
                       (o.qavg[g].cpu().numpy(), o.favg[g].cpu().numpy(), o.face_q[g].cpu().numpy(),
                        o.face_f[g].cpu().numpy()), cfg["q_stride"])
        checked += len(local)
    assert checked == 3 * (sh.count // chunk)
    del q, par, out
    torch.cuda.empty_cache()
