"""CPU tests: pin the oracle (our C restatement) against the reference.

* golden vectors produced by the unmodified reference (tests/golden/, make_golden.py);
* known-answer tests from the reference's own suites (SplitMix64 seed-0 sequence,
  Gauss-Legendre closed forms, zero dynamics, dense volume-operator Taylor series,
  superposition, face extrapolation);
* live comparison with oracle/_ref when it is built.
"""
import glob
import json
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-12  # parity tolerance used throughout (BASELINE.json north_star)


def _cases():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_oracle_matches_reference_golden(oracle, case):
    g = np.load(os.path.join(GOLDEN, case["name"] + ".npz"))
    n, m = case["n"], case["m"]
    kind = case.get("pde_kind", O.PDE_ELASTIC)
    par = g["par_lmr"] if "par_lmr" in g else None
    args = g["args"] if "args" in g else None
    out = oracle.stp(n, m, g["q"], float(g["dt"]), par=par, pde_kind=kind, args=args,
                     t_start=float(g["t_start"]), threads=1)
    for name in ("qavg", "favg", "face_q", "face_f"):
        ref = g[name]
        got = getattr(out, name)
        assert O.per_element_rel_diff(ref, got) <= TOL, name


def test_splitmix_known_sequence(oracle):
    # proj/tests/test_harness.cpp:32-37
    assert oracle.splitmix(0, 3) == [16294208416658607535, 7960286522194355700, 487617019471545679]
    g = np.load(os.path.join(GOLDEN, "splitmix.npz"))
    assert oracle.splitmix(0, 16) == [int(x) for x in g["seed0"]]
    assert oracle.splitmix(12345, 64) == [int(x) for x in g["seed12345"]]


def test_gauss_legendre_closed_forms(oracle):
    # proj/tests/test_basis.cpp:12-37
    b1 = oracle.basis(1)
    assert abs(b1["nodes"][0] - 0.5) < 1e-15 and abs(b1["weights"][0] - 1.0) < 1e-15
    b2 = oracle.basis(2)
    s3 = np.sqrt(3.0)
    assert abs(b2["nodes"][0] - (3 - s3) / 6) < 1e-15 and abs(b2["nodes"][1] - (3 + s3) / 6) < 1e-15
    assert np.all(np.abs(b2["weights"] - 0.5) < 1e-15)
    b3 = oracle.basis(3)
    assert abs(b3["nodes"][1] - 0.5) < 1e-15
    assert np.allclose(b3["weights"], [5 / 18, 8 / 18, 5 / 18], atol=1e-15, rtol=0)
    for n in range(1, 11):
        b = oracle.basis(n)
        assert abs(b["weights"].sum() - 1.0) < 1e-14
        for p in range(2 * n):
            assert abs(np.dot(b["weights"], b["nodes"] ** p) - 1.0 / (p + 1)) < 1e-14
        # derivative exact for monomials up to degree n-1, rows annihilate constants
        for p in range(n):
            assert np.max(np.abs(b["d"] @ b["nodes"] ** p - (p * b["nodes"] ** (p - 1) if p else 0))) < 1e-11
        assert np.max(np.abs(b["d"].sum(axis=1))) < 1e-12


def test_basis_matches_reference_golden(oracle):
    g = np.load(os.path.join(GOLDEN, "basis.npz"))
    for n in range(1, 11):
        b = oracle.basis(n)
        for k in ("nodes", "weights", "d", "face_left", "face_right"):
            assert O.rel_diff(g[f"{k}_{n}"].reshape(b[k].shape), b[k]) < 1e-14, (n, k)


def test_zero_dynamics_exact(oracle):
    # proj/tests/test_predictor.cpp:36-53: qavg == dt*q exactly, favg == 0
    rng = np.random.default_rng(42)
    for n in (1, 4):
        q = rng.uniform(-1, 1, size=(3, n ** 3 * 3))
        dt = 0.013
        out = oracle.stp(n, 3, q, dt, pde_kind=O.PDE_ADVECTION, args=[0, 0, 0])
        assert np.array_equal(out.qavg, dt * q)
        assert not np.any(out.favg)


def _dense_volume_operator(basis, A, B=None):
    """V = sum_d (D_d kron A_d) + (D_d kron B_d) over the canonical (k3,k2,k1,s) ordering:
    the operator the CK recursion iterates (proj/src/predictor_common.cpp:243-259)."""
    n = basis["d"].shape[0]
    eye = np.eye(n)
    dx = np.kron(eye, np.kron(eye, basis["d"]))
    dy = np.kron(eye, np.kron(basis["d"], eye))
    dz = np.kron(basis["d"], np.kron(eye, eye))
    V = 0
    for d, Dd in enumerate((dx, dy, dz)):
        M = A[d] + (0 if B is None else B[d])
        V = V + np.kron(Dd, M)
    return V


def _elastic_A(lam, mu, rho):
    A = np.zeros((3, 9, 9))
    L, ir = lam + 2 * mu, 1.0 / rho
    A[0][[0, 1, 2], 6] = [L, lam, lam]; A[0][3, 7] = mu; A[0][4, 8] = mu
    A[0][6, 0] = ir; A[0][7, 3] = ir; A[0][8, 4] = ir
    A[1][[0, 1, 2], 7] = [lam, L, lam]; A[1][3, 6] = mu; A[1][5, 8] = mu
    A[1][6, 3] = ir; A[1][7, 1] = ir; A[1][8, 5] = ir
    A[2][[0, 1, 2], 8] = [lam, lam, L]; A[2][4, 6] = mu; A[2][5, 7] = mu
    A[2][6, 4] = ir; A[2][7, 5] = ir; A[2][8, 2] = ir
    return A


def _taylor(V, q, n, dt):
    # proj/tests/support/oracles.hpp:84-100
    it, acc, c = q.copy(), np.zeros_like(q), dt
    for o in range(n):
        acc += c * it
        it = V @ it
        c *= dt / (o + 2)
    return acc


def test_dense_volume_operator_taylor_series(oracle):
    # acceptance criterion 2 (proj/tests/acceptance.cpp:92-126): (N,m) = (3,6) demo, (4,9) elastic
    rng = np.random.default_rng(2024)
    b3 = oracle.basis(3)
    Ad = np.zeros((3, 6, 6))
    rows = [[(0, (0, 3, 4)), (1, (1, 3, 5)), (2, (2, 4, 5))],
            [(1, (1, 4, 5)), (2, (2, 4, 3)), (0, (0, 5, 3))],
            [(2, (2, 5, 3)), (0, (0, 5, 4)), (1, (1, 3, 4))]]
    for d in range(3):
        for out, ins in rows[d]:
            Ad[d][out, list(ins)] = -1.0
    q = rng.uniform(-1, 1, 27 * 6)
    dt = 0.4 / (3 * 3.0 * 5)
    got = oracle.stp(3, 6, q[None], dt, pde_kind=O.PDE_DEMO).qavg[0]
    want = _taylor(_dense_volume_operator(b3, Ad), q, 3, dt)
    assert O.rel_diff(want, got) < 1e-11

    b4 = oracle.basis(4)
    lam, mu, rho = 2.0, 1.0, 1.0
    q = rng.uniform(-1, 1, 64 * 9)
    dt = 0.4 / (3 * 2.0 * 7)
    got = oracle.stp(4, 9, q[None], dt, par=np.array([[lam, mu, rho]])).qavg[0]
    want = _taylor(_dense_volume_operator(b4, _elastic_A(lam, mu, rho)), q, 4, dt)
    assert O.rel_diff(want, got) < 1e-11


def test_superposition(oracle):
    # proj/tests/test_predictor.cpp:172-197
    rng = np.random.default_rng(321)
    n, m = 4, 6
    q1, q2 = rng.uniform(-1, 1, (2, 1, n ** 3 * m))
    a, b = 0.75, -1.25
    dt = 0.4 / (3 * 3.0 * 7)
    o1, o2, oc = (oracle.stp(n, m, x, dt, pde_kind=O.PDE_DEMO) for x in (q1, q2, a * q1 + b * q2))
    assert O.rel_diff(a * o1.qavg + b * o2.qavg, oc.qavg) < 1e-12


def test_face_extrapolation_constant(oracle):
    # proj/tests/test_predictor.cpp:247-258: constant qavg -> the constant on every face.  With
    # zero dynamics qavg = dt*q, so a constant q gives dt*q on every face.
    n, m = 4, 3
    q = np.tile(1.0 + np.arange(m), n ** 3)[None]
    out = oracle.stp(n, m, q, 1.0, pde_kind=O.PDE_ADVECTION, args=[0, 0, 0])
    want = np.tile(1.0 + np.arange(m), n * n)
    for f in range(6):
        assert np.max(np.abs(out.face_q[0, f] - want)) < 1e-13


def test_layout_roundtrip_bit_exact(oracle):
    rng = np.random.default_rng(5)
    for n, m, qs in ((4, 9, 9), (8, 9, 12), (5, 6, 16)):
        q = rng.uniform(-1, 1, (3, n ** 3 * m))
        x = oracle.to_aosoa(n, m, qs, q)
        assert np.array_equal(oracle.from_aosoa(n, m, qs, x), q)
        x = x.reshape(3, n, n, qs, n)
        assert not np.any(x[:, :, :, m:, :])  # padding slots are zero


def test_generator_documented_stream(oracle):
    # element e's U[-1,1] values are draws e*K .. e*K+9n^3-1 of one SplitMix64(seed) stream,
    # K = 9n^3 + 3, followed by (rho, cp, cs)
    n, seed = 3, 99
    q, par = oracle.generate(0, seed, n, 5, 2)
    K = 9 * n ** 3 + 3
    raw = oracle.splitmix(seed, 2 * K, start=5 * K)
    sym = [2.0 * ((x >> 11) * 2.0 ** -53) - 1.0 for x in raw]
    assert np.array_equal(q[0], np.array(sym[:9 * n ** 3]))
    assert np.array_equal(q[1], np.array(sym[K:K + 9 * n ** 3]))
    u = [(x >> 11) * 2.0 ** -53 for x in raw[9 * n ** 3:K]]
    assert par[0, 0] == 2.0 + 1.0 * u[0] and par[0, 1] == 4.0 + 2.0 * u[1] and par[0, 2] == 2.0 + 1.5 * u[2]
    assert np.all((par[:, 0] >= 2) & (par[:, 0] < 3) & (par[:, 1] >= 4) & (par[:, 1] < 6))


def test_validation_rejects_like_reference(oracle):
    q = np.zeros((1, 27 * 9))
    with pytest.raises(ValueError):
        oracle.stp(3, 9, q, 0.0, par=np.array([[2.0, 1.0, 1.0]]))  # dt <= 0
    bad = q.copy()
    bad[0, 5] = np.nan
    with pytest.raises(ValueError):
        oracle.stp(3, 9, bad, 0.01, par=np.array([[2.0, 1.0, 1.0]]))  # non-finite input
    with pytest.raises(ValueError):
        oracle.stp(3, 9, q, 0.01, par=np.array([[-3.0, 1.0, 1.0]]))  # lambda + 2 mu <= 0


def test_oracle_matches_live_reference(oracle, reference):
    rng = np.random.default_rng(11)
    for n in (3, 6, 9):
        q, rcc = oracle.generate(0, 500 + n, n, 0, 3)
        lmr = oracle.material_lmr(rcc)
        dt = O.cfl_dt(n, rcc[:, 1].max())
        a = oracle.stp(n, 9, q, dt, par=lmr)
        for variant in ("generic", "log", "splitck", "aosoa"):
            b = reference.stp(n, 9, q, dt, par=lmr, variant=variant, threads=2)
            for name in ("qavg", "favg", "face_q", "face_f"):
                assert O.per_element_rel_diff(getattr(b, name), getattr(a, name)) <= TOL, (n, variant, name)
    del rng


def test_golden_files_present():
    assert len(glob.glob(os.path.join(GOLDEN, "elastic_n*.npz"))) == 9


@pytest.mark.parametrize("kind,m,n,args,par", [
    (O.PDE_ELASTIC, 9, 3, None, [2.0, 1.0, 1.3]),
    (O.PDE_ELASTIC, 9, 5, None, [1.5, 0.7, 2.0]),
    (O.PDE_ADVECTION, 2, 4, [1.0, 0.5, 0.25], None),
    (O.PDE_NCP_ADVECTION, 3, 3, [0.3, -1.0, 0.5], None),
    (O.PDE_DEMO, 6, 2, None, None),
])
def test_corrector_restatement_matches_reference(oracle, reference, kind, m, n, args, par):
    """orc_corrector_step pinned against the reference's own corrector_step (solver.cpp:257-311)."""
    e, L = 3, 2.0
    E = e ** 3
    rng = np.random.default_rng(n + m)
    u0 = rng.standard_normal((E, n ** 3 * m))
    qavg = rng.standard_normal((E, n ** 3 * m))
    fq = rng.standard_normal((E, 6, n * n * m))
    ff = rng.standard_normal((E, 6, n * n * m))
    smax = reference.max_wavespeed(kind, m, par=par, args=args)
    ref_u, ok = reference.corrector_step(n, m, e, L, u0, qavg, fq, ff, 0.01, par=par, pde_kind=kind, args=args)
    got, ok2 = oracle.corrector_step(n, m, e, L, u0, qavg, fq, ff, smax, par=par, pde_kind=kind, args=args)
    assert ok and ok2
    assert O.per_element_rel_diff(ref_u - u0, got - u0) <= 1e-13


def _demo_matrices():
    """The paper demo system (proj/include/ader/pde.hpp:68-73) as matrices: x-flux rows
    F0 = -(Q0+Q3+Q4), F1 = -(Q1+Q3+Q5), F2 = -(Q2+Q4+Q5), y/z by the rotation (0 1 2)(3 4 5)."""
    rot = [0, 1, 2, 3, 4, 5]
    A = []
    for _ in range(3):
        a = np.zeros((6, 6))
        for r, cols in ((0, (0, 3, 4)), (1, (1, 3, 5)), (2, (2, 4, 5))):
            for c in cols:
                a[rot[r], rot[c]] = -1.0
        A.append(a)
        rot = [rot[1], rot[2], rot[0], rot[4], rot[5], rot[3]]
    return A


def test_matrix_pde_shim_matches_builtin_pdes(oracle, reference):
    """The shim's MatrixPde (a user LinearPde defined by A_d, B_d) reproduces the reference's own
    advection / ncp-advection / demo systems given as their probed matrices: this pins the
    matrix-PDE oracle used for the GPU's arbitrary probed systems."""
    v = [1.0, 0.5, 0.25]
    rng = np.random.default_rng(7)
    n = 4
    for kind, m, A, B, args in (
            (O.PDE_ADVECTION, 3, [-v[d] * np.eye(3) for d in range(3)], None, v),
            (O.PDE_NCP_ADVECTION, 2, [np.zeros((2, 2))] * 3, [-v[d] * np.eye(2) for d in range(3)], v)):
        q = rng.uniform(-1, 1, (3, n ** 3 * m))
        want = reference.stp(n, m, q, 2e-3, pde_kind=kind, args=args, threads=2)
        got = reference.stp_matrix(n, m, q, 2e-3, A, B, threads=2)
        for name in ("qavg", "favg", "face_q", "face_f"):
            assert O.per_element_rel_diff(getattr(want, name), getattr(got, name)) <= 1e-14, (kind, name)
    q = rng.uniform(-1, 1, (3, n ** 3 * 6))
    want = reference.stp(n, 6, q, 2e-3, pde_kind=O.PDE_DEMO, threads=2)
    got = reference.stp_matrix(n, 6, q, 2e-3, _demo_matrices(), threads=2)
    for name in ("qavg", "favg", "face_q", "face_f"):
        assert O.per_element_rel_diff(getattr(want, name), getattr(got, name)) <= 1e-14, name
    # and the C restatement agrees with the matrix form of the demo system
    c = oracle.stp(n, 6, q, 2e-3, pde_kind=O.PDE_DEMO)
    assert O.per_element_rel_diff(c.face_f, got.face_f) <= TOL
