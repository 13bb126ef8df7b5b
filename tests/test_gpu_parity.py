"""GPU parity: the CUDA STP (through the C ABI) against the CPU oracle on identical inputs.

Tolerance: the reference's rel_diff metric (proj/src/checks.cpp:27-34), per element and per
output array, <= 1e-12 (BASELINE.json north_star).  Inputs are generated on the device and copied
back, so both sides see bit-identical data.
"""
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


@pytest.mark.parametrize("n", [2, 3, 5, 8, 9])
def test_kernel_variants_agree(stp, oracle, monkeypatch, n):
    """Every kernel family (DMMA nDof 8, line-pass, generic table) against the oracle."""
    S = stp
    E = 19
    q, par = S.generate(0, 5 + n, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    par_h = par.cpu().numpy()
    dt = O.cfl_dt(n, par_h[:, 1].max())
    ref = oracle.stp(n, 9, oracle.from_aosoa(n, 9, 9, q.cpu().numpy()), dt, par=oracle.material_lmr(par_h))
    for env in ({"ADERSTP_NO_DMMA8": "1"}, {"ADERSTP_FORCE_GENERIC": "1"}, {"ADERSTP_DMMA8_DB": "1"}):
        for k in ("ADERSTP_NO_DMMA8", "ADERSTP_FORCE_GENERIC", "ADERSTP_DMMA8_DB"):
            monkeypatch.setenv(k, env.get(k, "0"))
        plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
        out = plan.predict(q, dt, par=par)
        plan.status()
        worst = _compare(S, oracle, n, out, ref, S.LAYOUT_AOSOA, 9)
        assert max(worst.values()) <= TOL, (env, worst)
