"""The general user-LinearPde path (stp_general.cu) and point sources in the GPU corrector /
time loop, against the unmodified reference.

* predictor: dense flux + ncp systems (m = 12 at nDof 6 and 8, m = 21 -- the paper's application
  size, proj PAPER.md:676 -- at nDof 4, 8 and 10, the last on the global-scratch path; at nDof 8
  m = 4 .. 21 on the tensor-core kernel stp_gdense, every k-step count 1..6), both layouts, against predict() + extrapolate_faces of a reference LinearPde subclass with the same
  matrices (oracle/ref_shim.cpp MatrixPde); the reference's own PDEs forced onto the general
  kernel (ADERSTP_GENERAL=1) against the oracle; built-in kinds beyond the table kernels
  (advection with m = 20); a LinearPde with a point source;
* corrector / time loop: corrector_step with a point source (elastic, source-only, general)
  against ader::corrector_step, and run_simulation with an elastic point source and with a dense
  general system against ader::run_simulation.

Tolerance: rel_diff per element and output array <= 1e-12 for the predictor, <= 1e-12 on the
corrector increments, <= 1e-11 after several time steps (as tests/test_gpu_corrector.py).
"""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2003_12787_b200 as pkg
    return pkg


def dense_system(m, seed, ncp=True, scale=1.0):
    rng = np.random.default_rng(seed)
    A = [rng.uniform(-1, 1, (m, m)) * scale / m ** 0.5 for _ in range(3)]
    B = [rng.uniform(-0.5, 0.5, (m, m)) * scale / m ** 0.5 for _ in range(3)] if ncp else None
    return A, B


def compare(S, oracle, n, m, out, ref, layout, stride):
    E = ref.qavg.shape[0]
    if layout == S.LAYOUT_AOSOA:
        qa = oracle.from_aosoa(n, m, stride, out.qavg.cpu().numpy())
        fa = np.stack([oracle.from_aosoa(n, m, stride, out.favg[:, d].cpu().numpy()) for d in range(3)], 1)
    else:
        qa = out.qavg.cpu().numpy().reshape(E, n ** 3, stride)[:, :, :m].reshape(E, -1)
        fa = out.favg.cpu().numpy().reshape(E, 3, n ** 3, stride)[..., :m].reshape(E, 3, -1)
        assert not np.any(out.qavg.cpu().numpy().reshape(E, n ** 3, stride)[:, :, m:])
    worst = {"qavg": O.per_element_rel_diff(ref.qavg, qa),
             "favg": O.per_element_rel_diff(ref.favg.reshape(E, -1), fa.reshape(E, -1)),
             "face_q": O.per_element_rel_diff(ref.face_q.reshape(E, -1), out.face_q.cpu().numpy().reshape(E, -1)),
             "face_f": O.per_element_rel_diff(ref.face_f.reshape(E, -1), out.face_f.cpu().numpy().reshape(E, -1))}
    return worst


def run_gpu(S, oracle, n, m, pde, qn, dt, layout, stride, t_start=0.0):
    E = qn.shape[0]
    if layout == S.LAYOUT_AOSOA:
        q = torch.from_numpy(oracle.to_aosoa(n, m, stride, qn)).cuda()
    else:
        a = np.zeros((E, n ** 3, stride))
        a[:, :, :m] = qn.reshape(E, n ** 3, m)
        q = torch.from_numpy(a.reshape(E, -1)).cuda()
    plan = S.Plan(n, pde, layout=layout, q_stride=stride, out_stride=stride)
    out = plan.predict(q, dt, t_start=t_start)
    plan.status()
    return out


@pytest.mark.parametrize("m,n,layout", [(12, 6, "aosoa"), (12, 8, "aosoa"), (12, 8, "aos"), (21, 4, "aosoa"),
                                        (21, 8, "aos"), (21, 8, "aosoa"), (21, 10, "aosoa"), (5, 3, "aosoa"),
                                        (7, 8, "aosoa"), (9, 8, "aos"), (16, 8, "aosoa"), (17, 8, "aosoa"),
                                        (20, 8, "aos")])
def test_dense_system_matches_reference(S, oracle, reference, m, n, layout):
    A, B = dense_system(m, 1000 * m + n)
    E = 3 if n >= 10 else 5
    rng = np.random.default_rng(m + n)
    qn = rng.uniform(-1, 1, (E, n ** 3 * m))
    dt = 0.3 / (3 * 2.0 * (2 * n - 1))
    lay = S.LAYOUT_AOS if layout == "aos" else S.LAYOUT_AOSOA
    stride = (m + 7) // 8 * 8 if layout == "aos" else m
    out = run_gpu(S, oracle, n, m, S.linear_pde(A, B), qn, dt, lay, stride)
    reference.set_matrix_pde(A, B)
    ref = reference.stp(n, m, qn, dt, pde_kind=O.PDE_MATRIX, threads=4)
    worst = compare(S, oracle, n, m, out, ref, lay, stride)
    assert max(worst.values()) <= TOL, worst


@pytest.mark.parametrize("m,layout", [(21, "aosoa"), (13, "aos"), (6, "aosoa")])
def test_dense_tensor_core_kernel_matches_general_kernel(S, oracle, monkeypatch, m, layout):
    """nDof 8 dense systems run on stp_gdense (DMMA GEMMs); ADERSTP_NO_GDENSE=1 keeps them on the
    scalar general kernel.  Both against each other on 37 elements (several CTA waves' worth of
    element offsets), plus the padding slots of the AoS rows."""
    n = 8
    A, B = dense_system(m, 4242 + m)
    E = 37
    rng = np.random.default_rng(m)
    qn = rng.standard_normal((E, n ** 3 * m))
    lay = S.LAYOUT_AOS if layout == "aos" else S.LAYOUT_AOSOA
    stride = (m + 7) // 8 * 8 if layout == "aos" else m
    dt = 0.3 / (3 * 2.0 * (2 * n - 1))
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("ADERSTP_NO_GDENSE", flag)
        outs.append(run_gpu(S, oracle, n, m, S.linear_pde(A, B), qn, dt, lay, stride))
    for name in ("qavg", "favg", "face_q", "face_f"):
        a, b = (getattr(o, name).cpu().numpy().reshape(E, -1) for o in outs)
        assert O.per_element_rel_diff(b, a) <= TOL, name


@pytest.mark.parametrize("case", ["advection", "ncp_advection", "demo", "source_only", "elastic_matrix"])
@pytest.mark.parametrize("n", [2, 5, 8, 10])
def test_reference_pdes_on_the_general_kernel(S, oracle, monkeypatch, case, n):
    """ADERSTP_GENERAL=1 routes the reference's own PDEs (normally the table kernels) through
    the general kernel: it must reproduce the oracle."""
    monkeypatch.setenv("ADERSTP_GENERAL", "1")
    v = [1.0, 0.5, 0.25]
    src = S.PointSourceSpec((0.3, 0.6, 0.45), 1, 2.0, 0.01, 0.5)
    if case == "advection":
        m, pde, kind, args = 3, S.advection_pde(v, 3), O.PDE_ADVECTION, v
    elif case == "ncp_advection":
        m, pde, kind, args = 2, S.ncp_advection_pde(v, 2), O.PDE_NCP_ADVECTION, v
    elif case == "demo":
        m, pde, kind, args = 6, S.paper_demo_pde(), O.PDE_DEMO, None
    elif case == "source_only":
        m, pde, kind, args = 4, S.source_only_pde(4, src), O.PDE_SOURCE_ONLY, src.args()
    else:  # the elastic system (uniform material) as its probed matrices
        m, kind, args = 9, O.PDE_ELASTIC, None
        lam, mu, rho = 2.0, 1.0, 1.5
        A = []
        idx_in = [[6, 7, 8], [6, 7, 8], [6, 7, 8], [7, 6, 0], [8, 0, 6], [0, 8, 7], [0, 3, 4], [3, 1, 5], [4, 5, 2]]
        coef = [[0, 1, 1], [1, 0, 1], [1, 1, 0], [2, 2, 4], [2, 4, 2], [4, 2, 2], [3, 3, 3], [3, 3, 3], [3, 3, 3]]
        c4 = [lam + 2 * mu, lam, mu, 1.0 / rho, 0.0]
        for d in range(3):
            a = np.zeros((9, 9))
            for s in range(9):
                a[s, idx_in[s][d]] = c4[coef[s][d]]
            A.append(a)
        pde = S.linear_pde(A)
    E = 4
    rng = np.random.default_rng(n * 7 + m)
    qn = rng.uniform(-1, 1, (E, n ** 3 * m))
    dt, t0 = 2e-3, 0.004
    out = run_gpu(S, oracle, n, m, pde, qn, dt, S.LAYOUT_AOSOA, m, t_start=t0)
    par = np.array([[2.0, 1.0, 1.5]] * E) if kind == O.PDE_ELASTIC else None
    ref = oracle.stp(n, m, qn, dt, par=par, pde_kind=kind, args=args, t_start=t0)
    worst = compare(S, oracle, n, m, out, ref, S.LAYOUT_AOSOA, m)
    assert max(worst.values()) <= TOL, worst


def test_builtin_kind_beyond_table_size(S, oracle):
    """advection_pde(v, m) with m = 20 > 16: the general kernel, against the oracle."""
    n, m, E = 5, 20, 3
    v = [1.0, -0.5, 0.25]
    rng = np.random.default_rng(20)
    qn = rng.uniform(-1, 1, (E, n ** 3 * m))
    out = run_gpu(S, oracle, n, m, S.advection_pde(v, m), qn, 3e-3, S.LAYOUT_AOSOA, m)
    ref = oracle.stp(n, m, qn, 3e-3, pde_kind=O.PDE_ADVECTION, args=v)
    worst = compare(S, oracle, n, m, out, ref, S.LAYOUT_AOSOA, m)
    assert max(worst.values()) <= TOL, worst


@pytest.mark.parametrize("n", [3, 6])
def test_linear_pde_with_point_source(S, oracle, reference, n):
    m = 7
    A, B = dense_system(m, 77 + n)
    src = S.PointSourceSpec((0.2, 0.7, 0.55), 4, 1.5, 0.003, 0.02)
    E = 4
    rng = np.random.default_rng(n)
    qn = rng.uniform(-1, 1, (E, n ** 3 * m))
    dt, t0 = 4e-3, 0.001
    out = run_gpu(S, oracle, n, m, S.linear_pde(A, B, source=src), qn, dt, S.LAYOUT_AOSOA, m, t_start=t0)
    reference.set_matrix_pde(A, B, src.args())
    ref = reference.stp(n, m, qn, dt, pde_kind=O.PDE_MATRIX, t_start=t0, threads=2)
    worst = compare(S, oracle, n, m, out, ref, S.LAYOUT_AOSOA, m)
    assert max(worst.values()) <= TOL, worst


def test_default_max_wavespeed_is_the_characteristic_speed(S):
    """Probed systems: max_d max|eig(A_d + B_d)| (advection: max |v_d|), or the user's value."""
    v = [1.0, -0.5, 0.25]
    A = [-v[d] * np.eye(3) for d in range(3)]
    assert abs(S.linear_pde(A).max_wavespeed() - 1.0) < 1e-14
    assert S.linear_pde(A, max_wavespeed=3.5).max_wavespeed() == 3.5


# ---- corrector and time loop with point sources and general systems --------------------------
def to_dev(oracle, n, m, qc):
    return torch.from_numpy(oracle.to_aosoa(n, m, m, qc)).cuda()


def from_dev(oracle, n, m, u):
    return oracle.from_aosoa(n, m, m, u.cpu().numpy())


@pytest.mark.parametrize("case,n", [("elastic_source", 4), ("elastic_source", 8), ("source_only", 3),
                                    ("matrix_source", 5), ("matrix_dense", 4)])
def test_corrector_step_with_sources_and_general_systems(S, oracle, reference, case, n):
    e, L = 2, 1.5
    E = e ** 3
    src = S.PointSourceSpec((0.25, 0.5, 0.75), 7, 3.0, 0.01, 0.05)
    if case == "elastic_source":
        m, pde, kind, args, par = 9, S.elastic_pde(2.0, 1.0, 1.0, source=src), O.PDE_ELASTIC_SOURCE, src.args(), [2.0, 1.0, 1.0]
        smax = None
    elif case == "source_only":
        src = S.PointSourceSpec((0.25, 0.5, 0.75), 1, 3.0, 0.01, 0.05)
        m, pde, kind, args, par, smax = 3, S.source_only_pde(3, src), O.PDE_SOURCE_ONLY, src.args(), None, 0.0
    else:
        m = 8 if case == "matrix_source" else 12
        A, B = dense_system(m, 5 + m)
        s = S.PointSourceSpec((0.25, 0.5, 0.75), 2, 3.0, 0.01, 0.05) if case == "matrix_source" else None
        pde = S.linear_pde(A, B, source=s, max_wavespeed=1.7)
        reference.set_matrix_pde(A, B, None if s is None else s.args(), 1.7)
        kind, args, par, smax = O.PDE_MATRIX, None, None, 1.7
    rng = np.random.default_rng(100 + n)
    u0 = rng.standard_normal((E, n ** 3 * m))
    qavg = rng.standard_normal((E, n ** 3 * m))
    face_q = rng.standard_normal((E, 6, n * n * m))
    face_f = rng.standard_normal((E, 6, n * n * m))
    dt, t = 1e-2, 0.02
    ref_u, ok = reference.corrector_step(n, m, e, L, u0, qavg, face_q, face_f, dt, par=par, pde_kind=kind,
                                         args=args, t=t)
    assert ok
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA)
    u = to_dev(oracle, n, m, u0)
    out = S.PredictorOutput(to_dev(oracle, n, m, qavg), None, torch.from_numpy(face_q).cuda(),
                            torch.from_numpy(face_f).cuda())
    plan.correct(u, e, out, domain_len=L, max_wavespeed=smax, dt=dt, t=t)
    plan.status()
    worst = O.per_element_rel_diff(ref_u - u0, from_dev(oracle, n, m, u) - u0)
    assert worst <= TOL, worst
    if pde.has_source:
        with pytest.raises(S.StpError):
            plan.correct(u, e, out, domain_len=L, max_wavespeed=smax)  # dt is required with a source


@pytest.mark.parametrize("case,n,e", [("elastic_source", 4, 2), ("elastic_source", 6, 2), ("elastic_source", 8, 3),
                                      ("matrix_dense", 4, 2), ("matrix_source", 3, 2), ("matrix_m21", 3, 2),
                                      ("matrix_m21", 8, 2)])
def test_run_simulation_with_sources_and_general_systems(S, oracle, reference, case, n, e):
    """Several full time steps (predictor on the scaled PDE + corrector) against
    ader::run_simulation."""
    L, cfl = 1.0, 0.35
    E = e ** 3
    if case == "elastic_source":
        src = S.PointSourceSpec((0.4, 0.5, 0.6), 8, 5.0, 0.0, 0.05)
        m, pde, kind, args, par = 9, S.elastic_pde(2.0, 1.0, 1.0, source=src), O.PDE_ELASTIC_SOURCE, src.args(), [2.0, 1.0, 1.0]
        smax = reference.max_wavespeed(O.PDE_ELASTIC, 9, par=par)
        gpu_smax = None
    else:
        m = {"matrix_dense": 6, "matrix_source": 5, "matrix_m21": 21}[case]
        A, B = dense_system(m, 31 + m)
        s = S.PointSourceSpec((0.4, 0.5, 0.6), 1, 5.0, 0.0, 0.05) if case == "matrix_source" else None
        smax = S.linear_pde(A, B).max_wavespeed()
        pde = S.linear_pde(A, B, source=s, max_wavespeed=smax)
        reference.set_matrix_pde(A, B, None if s is None else s.args(), smax)
        kind, args, par, gpu_smax = O.PDE_MATRIX, None, None, smax
    rng = np.random.default_rng(3 + n)
    u0 = rng.standard_normal((E, n ** 3 * m))
    t_end = 4 * cfl * (L / e) / (3.0 * smax * (2 * n - 1))
    ref_u, ok, steps, _ = reference.run_simulation(n, m, e, L, u0, cfl, t_end, par=par, pde_kind=kind, args=args)
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA)
    u = to_dev(oracle, n, m, u0)
    ok2, steps2, _ = plan.run_simulation(u, e, t_end, cfl=cfl, domain_len=L, max_wavespeed=gpu_smax)
    assert ok and ok2 and steps == steps2 == 4
    worst = O.per_element_rel_diff(ref_u, from_dev(oracle, n, m, u))
    assert worst <= 1e-11, worst
