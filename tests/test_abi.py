"""CPU tests of the C-ABI library: it loads, exports every symbol include/aderstp.h declares,
and its host-side helpers (basis, FLOP/byte model, argument validation) behave -- no GPU compute."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "aderstp.h")


@pytest.fixture(scope="module")
def S():
    import paper_2003_12787_b200 as pkg
    return pkg


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(aderstp_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(S):
    names = declared_functions()
    assert len(names) >= 14
    lib = ctypes.CDLL(S.library_path)
    for name in names:
        assert hasattr(lib, name), name
    dyn = subprocess.run(["nm", "-D", "--defined-only", S.library_path], capture_output=True, text=True).stdout
    for name in names:
        assert re.search(rf"\bT {name}\b", dyn), name


def test_library_is_sm100a(S):
    out = subprocess.run(["cuobjdump", "--list-elf", S.library_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version(S):
    assert S.lib.aderstp_abi_version() == 2


def test_basis_matches_oracle_and_reference_golden(S, oracle):
    g = np.load(os.path.join(ROOT, "tests", "golden", "basis.npz"))
    for n in range(1, 11):
        b = S.make_basis(n)
        o = oracle.basis(n)
        for k in ("nodes", "weights", "d", "face_left", "face_right"):
            ours = getattr(b, k)
            assert O.rel_diff(o[k], ours) < 1e-14, (n, k)
            assert O.rel_diff(g[f"{k}_{n}"].reshape(ours.shape), ours) < 1e-14, (n, k)
        assert np.array_equal(b.d_t, b.d.T)


@pytest.mark.parametrize("n,flops,nbytes", [(4, 71424, 36888), (6, 482112, 108888),
                                            (8, 1935360, 239640), (10, 5760000, 446424)])
def test_algorithmic_counts(S, n, flops, nbytes):
    # SURVEY.md 8(d) / BASELINE.md 2
    assert S.flop_count(n, 9) == flops
    assert S.byte_count(n, 9) == nbytes
    assert S.byte_count(n, 9, with_favg=False) == 8 * 9 * (2 * n ** 3 + 12 * n * n) + 24


def test_supported_orders(S):
    assert [n for n in range(1, 13) if S.lib.aderstp_supported_order(n)] == list(range(2, 11))


def test_plan_validation_before_any_device_work(S):
    with pytest.raises(S.StpError) as e:
        S.Plan(11, S.elastic_pde())
    assert e.value.code == S.ADERSTP_ERR_UNSUPPORTED
    with pytest.raises(S.StpError) as e:
        S.Plan(4, S.LinearPde(0, 8, []))  # elastic kind with m != 9
    assert e.value.code == S.ADERSTP_ERR_INVALID_ARG
    with pytest.raises(S.StpError) as e:
        S.Plan(4, S.elastic_pde(), q_stride=5)
    assert e.value.code == S.ADERSTP_ERR_INVALID_ARG
    with pytest.raises(S.StpError):
        S.elastic_pde(-3.0, 1.0, 1.0)  # lambda + 2 mu <= 0 (proj/src/pde.cpp:175)
    with pytest.raises(S.StpError):
        S.elastic_pde(2.0, 1.0, 1.0, source=S.PointSourceSpec(component=1))  # pde.cpp:333-334


def test_null_and_negative_arguments_are_rejected(S):
    lib = S.lib
    assert lib.aderstp_predict_batch(None, 1, None, None, 0.1, 0.0, None, None, None, None, None) == 1
    assert lib.aderstp_convert_layout(4, 9, 1, 7, 9, None, 0, 9, None, None) == 1
    assert lib.aderstp_generate(9, 0, 4, 0, 1, 1, 0, 9, None, None, None) == 1
    assert b"unknown distribution" in lib.aderstp_last_error()


def test_stable_dt_matches_reference_formula(S):
    # proj/src/solver.cpp:170-174
    assert S.stable_dt(8, 6.0, cfl=0.5) == 0.5 / (3.0 * 6.0 * 15.0)
    assert S.stable_dt(4, 0.0) == float("inf")


def test_corrector_entry_points_validate_arguments(S):
    """aderstp_correct_batch / aderstp_run_simulation reject bad arguments before any device work."""
    L = S.lib
    mesh = S.stp._Mesh(2, 1.0)
    rc = L.aderstp_correct_batch(None, ctypes.byref(mesh), None, None, None, None, None, 1.0, 0.0, 0.0, None)
    assert rc == S.ADERSTP_ERR_INVALID_ARG
    steps, t_final = ctypes.c_int64(7), ctypes.c_double(7.0)
    rc = L.aderstp_run_simulation(None, ctypes.byref(mesh), None, None, 0.35, 1.0, 1.0,
                                  ctypes.byref(steps), ctypes.byref(t_final), None)
    assert rc == S.ADERSTP_ERR_INVALID_ARG and steps.value == 0 and t_final.value == 0.0
    assert b"null" in L.aderstp_last_error()
