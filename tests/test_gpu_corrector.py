"""GPU corrector step and time loop against the reference.

* aderstp_correct_batch vs ader::corrector_step (proj/src/solver.cpp:257-311) on identical
  predictor outputs, every PDE kind the GPU corrector supports;
* aderstp_run_simulation vs ader::run_simulation (:313-359) over several steps;
* the reference's own end-to-end pins (proj/tests/test_solver.cpp), run on the GPU: zero dynamics
  (bit-exact), free-stream preservation over 100 steps, mass conservation, one advection period,
  the elastic P-wave phase, instability reported.

Tolerances: rel_diff (proj/src/checks.cpp:27-34) per element <= 1e-12 for one corrector step
(on the increments u_new - u_old), <= 1e-11 after ten full time steps; the pins use the
reference tests' own bounds.
"""
import math

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

KVEL = (1.0, 0.5, 0.25)  # test_solver.cpp:22


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_12787_b200 as pkg
    return pkg


# ---- mesh helpers (ader::Mesh, proj/src/solver.cpp:17-91), canonical [c][k3][k2][k1][s] --------
def node_coords(S, n, e, L=1.0):
    b = S.make_basis(n)
    h = L / e
    iz, iy, ix, k3, k2, k1 = np.meshgrid(*(np.arange(e),) * 3, *(np.arange(n),) * 3, indexing="ij")
    x = (ix + b.nodes[k1]) * h
    y = (iy + b.nodes[k2]) * h
    z = (iz + b.nodes[k3]) * h
    w = b.weights[k1] * b.weights[k2] * b.weights[k3] * h ** 3
    shape = (e ** 3, n ** 3)
    return x.reshape(shape), y.reshape(shape), z.reshape(shape), w.reshape(shape)


def set_initial(S, n, e, m, f, L=1.0, t=0.0):
    x, y, z, _ = node_coords(S, n, e, L)
    q = np.zeros(x.shape + (m,))
    for s in range(m):
        q[..., s] = f(x, y, z, t, s)
    return q.reshape(e ** 3, -1)


def to_dev(oracle, n, m, qc):
    return torch.from_numpy(oracle.to_aosoa(n, m, m, qc)).cuda()


def from_dev(oracle, n, m, u):
    return oracle.from_aosoa(n, m, m, u.cpu().numpy())


def integral(S, n, e, m, qc, s, L=1.0):
    _, _, _, w = node_coords(S, n, e, L)
    return float(np.sum(w * qc.reshape(e ** 3, n ** 3, m)[..., s]))


def l2_error(S, n, e, m, qc, exact, t, L=1.0):
    ref = set_initial(S, n, e, m, exact, L, t)
    _, _, _, w = node_coords(S, n, e, L)
    d = (qc - ref).reshape(e ** 3, n ** 3, m)
    return math.sqrt(float(np.sum(w[..., None] * d * d)))


def pde_cases(S):
    return {
        "elastic": (S.elastic_pde(2.0, 1.0, 1.0), O.PDE_ELASTIC, 9, None, [2.0, 1.0, 1.0]),
        "advection": (S.advection_pde(KVEL, 2), O.PDE_ADVECTION, 2, list(KVEL), None),
        "ncp_advection": (S.ncp_advection_pde(KVEL, 3), O.PDE_NCP_ADVECTION, 3, list(KVEL), None),
        "demo": (S.paper_demo_pde(), O.PDE_DEMO, 6, None, None),
    }


# ---- one corrector step ----------------------------------------------------------------------
@pytest.mark.parametrize("case", ["elastic", "advection", "ncp_advection", "demo"])
@pytest.mark.parametrize("n", [3, 4, 8])
def test_corrector_step_matches_reference(S, oracle, reference, case, n):
    pde, kind, m, args, par = pde_cases(S)[case]
    e, L = 3, 1.5
    E = e ** 3
    rng = np.random.default_rng(100 + n)
    u0 = rng.standard_normal((E, n ** 3 * m))
    qavg = rng.standard_normal((E, n ** 3 * m))
    face_q = rng.standard_normal((E, 6, n * n * m))
    face_f = rng.standard_normal((E, 6, n * n * m))
    dt = 1e-2
    ref_u, ok = reference.corrector_step(n, m, e, L, u0, qavg, face_q, face_f, dt, par=par,
                                         pde_kind=kind, args=args)
    assert ok
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA)
    u = to_dev(oracle, n, m, u0)
    out = S.PredictorOutput(to_dev(oracle, n, m, qavg), None, torch.from_numpy(face_q).cuda(),
                            torch.from_numpy(face_f).cuda())
    plan.correct(u, e, out, domain_len=L)
    plan.status()
    got = from_dev(oracle, n, m, u)
    worst = O.per_element_rel_diff(ref_u - u0, got - u0)
    assert worst <= 1e-12, worst


def test_corrector_elastic_per_face_wavespeed(S, oracle):
    """Per-element material: smax of a face = max(cp) of its two elements; an explicit
    max_wavespeed overrides it.  With uniform material both coincide."""
    n, m, e = 4, 9, 2
    E = e ** 3
    rng = np.random.default_rng(7)
    u0 = rng.standard_normal((E, n ** 3 * m))
    qavg, fq, ff = (rng.standard_normal(s) for s in ((E, n ** 3 * m), (E, 6, n * n * m), (E, 6, n * n * m)))
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    par = torch.tensor([[2.5, 5.0, 3.0]] * E, dtype=torch.float64, device="cuda")
    outs = S.PredictorOutput(to_dev(oracle, n, m, qavg), None, torch.from_numpy(fq).cuda(), torch.from_numpy(ff).cuda())
    u1 = to_dev(oracle, n, m, u0)
    plan.correct(u1, e, outs, par=par)
    u2 = to_dev(oracle, n, m, u0)
    plan.correct(u2, e, outs, par=par, max_wavespeed=5.0)
    plan.status()
    d = O.rel_diff((u2 - to_dev(oracle, n, m, u0)).cpu().numpy(), (u1 - to_dev(oracle, n, m, u0)).cpu().numpy())
    assert d <= 1e-14, d


# ---- the time loop ---------------------------------------------------------------------------
@pytest.mark.parametrize("case,n,e", [("elastic", 4, 2), ("elastic", 5, 2), ("elastic", 6, 2), ("elastic", 7, 2),
                                      ("elastic", 8, 2), ("elastic", 9, 2), ("elastic", 10, 2), ("elastic", 8, 3),
                                      ("advection", 5, 3), ("demo", 3, 2), ("advection", 9, 2), ("demo", 10, 2),
                                      ("ncp_advection", 10, 2)])
def test_run_simulation_matches_reference(S, oracle, reference, case, n, e):
    pde, kind, m, args, par = pde_cases(S)[case]
    init = lambda x, y, z, t, s: np.sin(2 * np.pi * x + s) + 0.3 * np.cos(2 * np.pi * (y - z) + 0.2 * s)  # noqa: E731
    q0 = set_initial(S, n, e, m, init)
    smax = reference.max_wavespeed(kind, m, par=par, args=args)
    h = 1.0 / e
    dt = 0.35 * h / (3.0 * smax * (2 * n - 1))
    t_end = 10 * dt
    ref_u, stable, steps, t_final = reference.run_simulation(n, m, e, 1.0, q0, 0.35, t_end, par=par,
                                                            pde_kind=kind, args=args)
    assert stable and steps == 10
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA)
    u = to_dev(oracle, n, m, q0)
    ok, our_steps, our_t = plan.run_simulation(u, e, t_end, cfl=0.35)
    assert ok and our_steps == steps and abs(our_t - t_final) <= 1e-15
    worst = O.per_element_rel_diff(ref_u, from_dev(oracle, n, m, u))
    assert worst <= 1e-11, worst


def test_zero_dynamics_leaves_mesh_unchanged(S, oracle):
    """test_solver.cpp:76-89: advection with v = 0, bit-exact."""
    n, m, e = 3, 2, 2
    rng = np.random.default_rng(1)
    q0 = rng.uniform(-1, 1, (e ** 3, n ** 3 * m))
    plan = S.Plan(n, S.advection_pde((0.0, 0.0, 0.0), m), layout=S.LAYOUT_AOSOA)
    u = to_dev(oracle, n, m, q0)
    ok, steps, _ = plan.run_simulation(u, e, 0.1)
    assert ok and steps >= 1
    assert np.array_equal(from_dev(oracle, n, m, u), q0)


def test_free_stream_preservation_100_steps(S, oracle):
    """test_solver.cpp:91-110."""
    n, m, e = 4, 2, 3
    q0 = set_initial(S, n, e, m, lambda x, y, z, t, s: np.full_like(x, 0.75 if s == 0 else -2.0))
    pde = S.advection_pde(KVEL, m)
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA)
    dt = S.stable_dt(n, pde.max_wavespeed(), cfl=0.35, h=1.0 / e)
    u = to_dev(oracle, n, m, q0)
    ok, steps, _ = plan.run_simulation(u, e, 100 * dt)
    assert ok and steps >= 100
    got = from_dev(oracle, n, m, u).reshape(-1, m)
    assert np.abs(got[:, 0] - 0.75).max() < 1e-13
    assert np.abs(got[:, 1] + 2.0).max() < 1e-13


def test_mass_conservation_periodic_advection(S, oracle):
    """test_solver.cpp:112-140: per-step drift < 1e-12."""
    n, m, e = 3, 1, 3
    q0 = set_initial(S, n, e, m, lambda x, y, z, t, s: 1.0 + 0.5 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * (y + z)))
    pde = S.advection_pde(KVEL, m)
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA)
    dt = S.stable_dt(n, pde.max_wavespeed(), cfl=0.35, h=1.0 / e)
    u = to_dev(oracle, n, m, q0)
    mass0 = prev = integral(S, n, e, m, q0, 0)
    for _ in range(25):
        ok, steps, _ = plan.run_simulation(u, e, dt)
        assert ok and steps == 1
        mass = integral(S, n, e, m, from_dev(oracle, n, m, u), 0)
        assert abs(mass - prev) < 1e-12
        prev = mass
    assert abs(prev - mass0) < 1e-12 * 25


def test_one_advection_period(S, oracle):
    """test_solver.cpp:142-158: l2 error after one period in (0, 5e-3)."""
    n, m, e = 4, 1, 3
    exact = lambda x, y, z, t, s: np.sin(2 * np.pi * (x - t))  # noqa: E731
    plan = S.Plan(n, S.advection_pde((1.0, 0.0, 0.0), m), layout=S.LAYOUT_AOSOA)
    u = to_dev(oracle, n, m, set_initial(S, n, e, m, exact))
    ok, steps, t_final = plan.run_simulation(u, e, 1.0)
    assert ok and abs(t_final - 1.0) < 1e-12
    err = l2_error(S, n, e, m, from_dev(oracle, n, m, u), exact, 1.0)
    assert 0.0 < err < 5e-3, err


def test_elastic_p_wave_phase(S, oracle):
    """test_solver.cpp:185-231: a right-going P wave travels at cp within 1 % phase error."""
    lam, mu, rho = 2.0, 1.0, 1.0
    cp = math.sqrt((lam + 2 * mu) / rho)
    n, m, e = 4, 9, 9

    def exact(x, y, z, t, s):
        g = np.sin(2 * np.pi * (x - cp * t))
        return {6: g, 0: -cp * rho * g, 1: -(lam / cp) * g, 2: -(lam / cp) * g}.get(s, 0 * g)

    plan = S.Plan(n, S.elastic_pde(lam, mu, rho), layout=S.LAYOUT_AOSOA)
    u = to_dev(oracle, n, m, set_initial(S, n, e, m, exact))
    t_end = 0.125
    ok, _, _ = plan.run_simulation(u, e, t_end)
    assert ok
    qc = from_dev(oracle, n, m, u).reshape(e ** 3, n ** 3, m)
    x, _, _, w = node_coords(S, n, e)
    vel = qc[..., 6]
    c_re = float(np.sum(w * vel * np.cos(2 * np.pi * x)))
    c_im = float(np.sum(w * vel * np.sin(2 * np.pi * x)))
    shift = math.atan2(-c_re, c_im) / (2 * np.pi)
    want = cp * t_end
    err = math.fmod(abs(shift - want), 1.0)
    err = min(err, 1.0 - err)
    assert err < 0.01 * want, err


def test_instability_is_reported(S, oracle):
    """test_solver.cpp:233-247: an absurd CFL on near-overflow data is flagged, not returned as NaN."""
    n, m, e = 5, 1, 3
    plan = S.Plan(n, S.advection_pde((1.0, 0.0, 0.0), m), layout=S.LAYOUT_AOSOA)
    u = to_dev(oracle, n, m, set_initial(S, n, e, m, lambda x, y, z, t, s: 1e300 * np.sin(2 * np.pi * x)))
    ok, _, _ = plan.run_simulation(u, e, 10.0, cfl=40.0)
    assert not ok


def test_source_only_run_simulation_accumulates_the_source_integral(S, oracle, reference):
    """A source-only PDE (no flux): run_simulation is pure accumulation of the projected source
    integrals (correct_cell, solver.cpp:206-216), matching ader::run_simulation."""
    src = S.PointSourceSpec((0.5, 0.5, 0.5), 0, 1.0, 0.1, 0.05)
    n, m, e = 4, 2, 2
    plan = S.Plan(n, S.source_only_pde(m, src), layout=S.LAYOUT_AOSOA)
    u = torch.zeros(e ** 3, plan.q_size, dtype=torch.float64, device="cuda")
    ok, steps, t = plan.run_simulation(u, e, 0.1)  # max_wavespeed() = 0: one step of dt = t_end
    ref_u, ok2, steps2, _ = reference.run_simulation(n, m, e, 1.0, np.zeros((e ** 3, n ** 3 * m)), 0.35, 0.1,
                                                     pde_kind=O.PDE_SOURCE_ONLY, args=src.args())
    assert ok and ok2 and steps == steps2 > 0
    assert O.per_element_rel_diff(ref_u, from_dev(oracle, n, m, u)) <= 1e-11


# ---- the slab decomposition of the multi-GPU time loop (one slab per thread on one GPU) --------
class _ThreadSync:
    """sync(flag) -> max over the slab threads; doubles as the barrier (host side only: no kernel
    waits on another slab)."""

    def __init__(self, parties):
        import threading
        self.flags = [0] * parties
        self.barrier = threading.Barrier(parties)
        self.local = threading.local()

    def bind(self, idx):
        def sync(flag):
            self.flags[idx] = int(flag)
            self.barrier.wait()
            out = max(self.flags)
            self.barrier.wait()
            return out
        return sync


@pytest.mark.parametrize("n,e,slabs", [(4, 6, 2), (4, 6, 3), (5, 4, 2), (8, 4, 2), (9, 3, 3), (10, 3, 3)])
def test_slab_decomposition_matches_single_gpu(S, n, e, slabs):
    """aderstp_run_simulation_slab on `slabs` z-slabs, each corrector reading its neighbours'
    faces through halo pointers, reproduces the single-GPU run_simulation."""
    import threading
    from paper_2003_12787_b200.shard import slab_partition
    E = e ** 3
    q, par = S.generate(0, 99 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    p = par.cpu().numpy()
    mu = p[:, 0] * p[:, 2] * p[:, 2]
    lam = p[:, 0] * p[:, 1] * p[:, 1] - 2.0 * mu
    cp_max = float(np.sqrt((lam + 2.0 * mu) / p[:, 0]).max())
    dt = 0.35 * (1.0 / e) / (3.0 * cp_max * (2 * n - 1))
    t_end = 3.5 * dt
    u_ref = q.clone()
    ok, steps_ref, _ = plan.run_simulation(u_ref, e, t_end, par=par, cfl=0.35)
    assert ok and steps_ref == 4
    parts = [slab_partition(e, slabs, r) for r in range(slabs)]
    us, pars, fqs, ffs = [], [], [], []
    for z0, nz in parts:
        a, b = z0 * e * e, (z0 + nz) * e * e
        us.append(q[a:b].clone())
        pars.append(par[a:b].contiguous())
        fqs.append(torch.empty(b - a, 6, plan.face_size, dtype=torch.float64, device="cuda"))
        ffs.append(torch.empty_like(fqs[-1]))
    halo = lambda r: (fqs[r], ffs[r], pars[r], parts[r][0])  # noqa: E731
    sync = _ThreadSync(slabs)
    results = [None] * slabs
    torch.cuda.synchronize()

    def work(r):
        stream = torch.cuda.Stream()
        results[r] = plan.run_simulation_slab(us[r], e, parts[r], fqs[r], ffs[r], t_end, cp_max,
                                              lo=halo((r - 1) % slabs), hi=halo((r + 1) % slabs), par=pars[r],
                                              cfl=0.35, sync=sync.bind(r), stream=stream)

    threads = [threading.Thread(target=work, args=(r,)) for r in range(slabs)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    torch.cuda.synchronize()
    assert all(r is not None and r[0] and r[1] == steps_ref for r in results), results
    got = torch.cat(us).cpu().numpy()
    worst = O.per_element_rel_diff(u_ref.cpu().numpy(), got)
    assert worst <= 1e-12, worst


def test_long_run_matches_reference(S, oracle, reference):
    """100 full time steps (elastic nDof 5 on a 3^3 mesh, smooth data): the GPU time loop stays
    on the reference's trajectory (no drift beyond rounding)."""
    n, m, e = 5, 9, 3
    pde, kind, _, args, par = pde_cases(S)["elastic"]
    init = lambda x, y, z, t, s: np.sin(2 * np.pi * (x + 2 * y) + s) * np.cos(2 * np.pi * z)  # noqa: E731
    q0 = set_initial(S, n, e, m, init)
    smax = reference.max_wavespeed(kind, m, par=par)
    dt = 0.35 * (1.0 / e) / (3.0 * smax * (2 * n - 1))
    t_end = 100 * dt
    ref_u, stable, steps, _ = reference.run_simulation(n, m, e, 1.0, q0, 0.35, t_end, par=par, pde_kind=kind)
    assert stable and steps == 100
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA)
    u = to_dev(oracle, n, m, q0)
    ok, our_steps, _ = plan.run_simulation(u, e, t_end)
    assert ok and our_steps == steps
    worst = O.per_element_rel_diff(ref_u, from_dev(oracle, n, m, u))
    assert worst <= 1e-10, worst


def test_plan_trim_returns_pooled_scratch(S, oracle):
    """The time loop's face buffers stay pooled between calls (no re-mapping per call) until
    Plan.trim(); the loop runs the same before and after a trim."""
    n, e = 4, 3
    q, par = S.generate(0, 3, n, 0, e ** 3, layout=S.LAYOUT_AOSOA, q_stride=9)
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    u1, u2 = (q * 1e-3).clone(), (q * 1e-3).clone()
    assert plan.run_simulation(u1, e, 2e-3, par=par)[0]
    plan.trim()
    assert plan.run_simulation(u2, e, 2e-3, par=par)[0]
    plan.trim()
    assert torch.equal(u1, u2)
