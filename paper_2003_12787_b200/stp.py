"""Python host mirror of the reference predictor interface over the C ABI (include/aderstp.h).

Reference interface mirrored (paths under /root/reference/proj):

* ``make_basis(n)``                     <- ``ader::make_basis``  (include/ader/basis.hpp:37)
* ``elastic_pde`` / ``advection_pde`` / ``ncp_advection_pde`` / ``paper_demo_pde`` /
  ``source_only_pde``                   <- the LinearPde factories (include/ader/pde.hpp:62-84)
* ``PredictorOutput``                   <- ``ader::PredictorOutput`` (include/ader/predictor.hpp:22-29)
* ``predict(q, pde, dt, ...)``          <- ``ader::predict`` + ``ader::extrapolate_faces``
                                           (include/ader/predictor.hpp:118-125), batched over
                                           the leading element axis
* ``stable_dt``                         <- ``ader::stable_dt`` (src/solver.cpp:170-174)
* ``flop_count`` / ``byte_count``       <- ``ader::flop_count`` (predictor.hpp:86), algorithmic

Errors raise ``StpError`` (a ``ValueError``, the analogue of the reference's
``std::invalid_argument``).  Every compute call goes through ``libaderstp.so``; there is no CPU
fallback and importing this module fails loudly if the library is missing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.environ.get("ADERSTP_LIB") or os.path.join(_HERE, "libaderstp.so")

ADERSTP_OK = 0
ADERSTP_ERR_INVALID_ARG = 1
ADERSTP_ERR_UNSUPPORTED = 2
ADERSTP_ERR_NONFINITE = 3
ADERSTP_ERR_MATERIAL = 4
ADERSTP_ERR_CUDA = 5

PDE_ELASTIC, PDE_ADVECTION, PDE_NCP_ADVECTION, PDE_DEMO, PDE_ELASTIC_SOURCE, PDE_SOURCE_ONLY, PDE_LINEAR = range(7)
PAR_LAMBDA_MU_RHO, PAR_RHO_CP_CS = 0, 1
LAYOUT_AOSOA, LAYOUT_AOS = 0, 1


class StpError(ValueError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[aderstp {code}] {msg}")
        self.code = code


class _Config(ctypes.Structure):
    _fields_ = [
        ("order", ctypes.c_int),
        ("quantities", ctypes.c_int),
        ("pde_kind", ctypes.c_int),
        ("layout", ctypes.c_int),
        ("q_stride", ctypes.c_int),
        ("out_stride", ctypes.c_int),
        ("par_kind", ctypes.c_int),
        ("check_inputs", ctypes.c_int),
        ("pde_args", ctypes.c_double * 8),
        ("linear", ctypes.POINTER(ctypes.c_double) * 6),
    ]


_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64


class _Mesh(ctypes.Structure):
    _fields_ = [("elements_per_dim", ctypes.c_int), ("domain_len", ctypes.c_double)]


class _Slab(ctypes.Structure):
    _fields_ = [("z0", ctypes.c_int), ("nz", ctypes.c_int)]


class _Halo(ctypes.Structure):
    _fields_ = [("face_q", ctypes.c_void_p), ("face_f", ctypes.c_void_p), ("par", ctypes.c_void_p),
                ("z_base", ctypes.c_int)]


_SyncFn = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int)


def _load():
    if not os.path.exists(library_path):
        raise ImportError(
            f"{library_path} is missing: build it with `make -C paper_2003_12787_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(library_path)
    L.aderstp_plan_create.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(_vp)]
    L.aderstp_plan_destroy.argtypes = [_vp]
    L.aderstp_plan_destroy.restype = None
    L.aderstp_predict_batch.argtypes = [_vp, _i64, _vp, _vp, ctypes.c_double, ctypes.c_double,
                                        _vp, _vp, _vp, _vp, _vp]
    L.aderstp_predict_batch_host.argtypes = [_vp, _i64, _dp, _dp, ctypes.c_double, ctypes.c_double,
                                             _dp, _dp, _dp, _dp]
    L.aderstp_plan_reserve_host_path.argtypes = [_vp, _i64]
    L.aderstp_plan_status.argtypes = [_vp, _vp]
    L.aderstp_plan_trim.argtypes = [_vp]
    L.aderstp_convert_layout.argtypes = [ctypes.c_int, ctypes.c_int, _i64, ctypes.c_int, ctypes.c_int,
                                         _vp, ctypes.c_int, ctypes.c_int, _vp, _vp]
    L.aderstp_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, _i64, _i64, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]
    L.aderstp_correct_batch.argtypes = [_vp, ctypes.POINTER(_Mesh), _vp, _vp, _vp, _vp, _vp, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, _vp]
    L.aderstp_run_simulation.argtypes = [_vp, ctypes.POINTER(_Mesh), _vp, _vp, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.POINTER(_i64), _dp, _vp]
    L.aderstp_correct_slab.argtypes = [_vp, ctypes.POINTER(_Mesh), ctypes.POINTER(_Slab), _vp, _vp, _vp, _vp, _vp,
                                       ctypes.POINTER(_Halo), ctypes.POINTER(_Halo), ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, _vp]
    L.aderstp_run_simulation_slab.argtypes = [_vp, ctypes.POINTER(_Mesh), ctypes.POINTER(_Slab), _vp, _vp, _vp, _vp,
                                              ctypes.POINTER(_Halo), ctypes.POINTER(_Halo), ctypes.c_double,
                                              ctypes.c_double, ctypes.c_double, _SyncFn, _vp,
                                              ctypes.POINTER(_i64), _dp, _vp]
    L.aderstp_device_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(_vp)]
    L.aderstp_device_free.argtypes = [_vp]
    L.aderstp_ipc_handle.argtypes = [_vp, ctypes.c_char_p]
    L.aderstp_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(_vp)]
    L.aderstp_ipc_close.argtypes = [_vp]
    L.aderstp_basis.argtypes = [ctypes.c_int, _dp, _dp, _dp, _dp, _dp]
    L.aderstp_flop_count.restype = ctypes.c_double
    L.aderstp_flop_count.argtypes = [ctypes.c_int, ctypes.c_int]
    L.aderstp_byte_count.restype = ctypes.c_double
    L.aderstp_byte_count.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.aderstp_supported_order.argtypes = [ctypes.c_int]
    L.aderstp_last_error.restype = ctypes.c_char_p
    L.aderstp_abi_version.restype = ctypes.c_int
    return L


lib = _load()


def _check(rc: int):
    if rc != ADERSTP_OK:
        raise StpError(rc, lib.aderstp_last_error().decode())


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


# ----------------------------------------------------------------------------- basis --------
@dataclass
class BasisOperators:
    """Nodal operators on [0,1] (include/ader/basis.hpp:18-27)."""
    n: int
    nodes: np.ndarray
    weights: np.ndarray
    inv_weights: np.ndarray
    d: np.ndarray
    d_t: np.ndarray
    face_left: np.ndarray
    face_right: np.ndarray


def make_basis(n: int) -> BasisOperators:
    nodes, w, fl, fr = (np.zeros(n) for _ in range(4))
    d = np.zeros(n * n)
    _check(lib.aderstp_basis(n, _np_ptr(nodes), _np_ptr(w), _np_ptr(d), _np_ptr(fl), _np_ptr(fr)))
    d = d.reshape(n, n)
    return BasisOperators(n, nodes, w, 1.0 / w, d, d.T.copy(), fl, fr)


def flop_count(order: int, quantities: int = 9) -> float:
    return lib.aderstp_flop_count(order, quantities)


def byte_count(order: int, quantities: int = 9, with_favg: bool = True) -> float:
    return lib.aderstp_byte_count(order, quantities, int(with_favg))


def stable_dt(order: int, max_wavespeed: float, cfl: float = 0.35, h: float = 1.0) -> float:
    """dt = cfl*h/(3*smax*(2N-1)) (src/solver.cpp:170-174); BASELINE uses cfl = 0.5."""
    if max_wavespeed <= 0.0:
        return float("inf")
    return cfl * h / (3.0 * max_wavespeed * (2.0 * order - 1.0))


# ------------------------------------------------------------------------------- PDEs -------
@dataclass
class PointSourceSpec:
    """include/ader/pde.hpp:47-56."""
    position: tuple = (0.5, 0.5, 0.5)
    component: int = 0
    amplitude: float = 1.0
    center: float = 0.0
    width: float = 1.0

    def args(self):
        return [*self.position, float(self.component), self.amplitude, self.center, self.width]


@dataclass
class LinearPde:
    kind: int
    quantities: int
    args: list = field(default_factory=list)
    linear: list | None = None  # [A_x, A_y, A_z, B_x, B_y, B_z] (m x m) for PDE_LINEAR
    wavespeed: float | None = None  # PDE_LINEAR: the user's max_wavespeed() (pde.hpp:41)

    @property
    def has_source(self) -> bool:
        return self.kind in (PDE_ELASTIC_SOURCE, PDE_SOURCE_ONLY) or (
            self.kind == PDE_LINEAR and len(self.args) >= 8 and self.args[7] != 0.0)

    def max_wavespeed(self) -> float:
        if self.kind == PDE_LINEAR:
            if self.wavespeed is not None:
                return float(self.wavespeed)
            # the characteristic speeds of q_t = sum_d (A_d + B_d) d_d q: the largest |eigenvalue|
            # over the three directions
            m = self.quantities
            best = 0.0
            for d in range(3):
                c = np.zeros((m, m))
                for mat in (self.linear[d], self.linear[3 + d]):
                    if mat is not None:
                        c = c + np.asarray(mat, dtype=np.float64)
                best = max(best, float(np.max(np.abs(np.linalg.eigvals(c)))) if m else 0.0)
            return best
        if self.kind in (PDE_ADVECTION, PDE_NCP_ADVECTION):
            return max(abs(v) for v in self.args[:3])
        if self.kind == PDE_DEMO:
            return 3.0
        if self.kind == PDE_SOURCE_ONLY:
            return 0.0
        raise NotImplementedError


@dataclass
class ElasticPde(LinearPde):
    """Elastic system (src/pde.cpp:171-284); material either uniform (lam, mu, rho as in the
    reference's constructor) or per element through the ``par`` argument of predict()."""
    lam: float | None = None
    mu: float | None = None
    rho: float | None = None

    def max_wavespeed(self) -> float:
        return float(np.sqrt((self.lam + 2.0 * self.mu) / self.rho))


AdvectionPde = NcpAdvectionPde = DemoPde = SourceOnlyPde = LinearPde


def elastic_pde(lam=None, mu=None, rho=None, source: PointSourceSpec | None = None) -> ElasticPde:
    if lam is not None and (not (rho > 0.0) or mu < 0.0 or not (lam + 2.0 * mu > 0.0)):
        raise StpError(ADERSTP_ERR_MATERIAL, "elastic_pde: need rho > 0, mu >= 0, lambda + 2mu > 0")
    if source is not None:
        if not 6 <= source.component <= 8:
            raise StpError(ADERSTP_ERR_INVALID_ARG,
                           "elastic_pde: source must act on a velocity component (6..8)")
        return ElasticPde(PDE_ELASTIC_SOURCE, 9, source.args(), lam=lam, mu=mu, rho=rho)
    return ElasticPde(PDE_ELASTIC, 9, [], lam=lam, mu=mu, rho=rho)


def advection_pde(velocity, m: int) -> LinearPde:
    return LinearPde(PDE_ADVECTION, m, list(map(float, velocity)))


def ncp_advection_pde(velocity, m: int) -> LinearPde:
    return LinearPde(PDE_NCP_ADVECTION, m, list(map(float, velocity)))


def paper_demo_pde() -> LinearPde:
    return LinearPde(PDE_DEMO, 6, [])


def source_only_pde(m: int, source: PointSourceSpec) -> LinearPde:
    return LinearPde(PDE_SOURCE_ONLY, m, source.args())


def linear_pde(flux_jacobians, ncp_matrices=None, source: PointSourceSpec | None = None,
               max_wavespeed: float | None = None) -> LinearPde:
    """Any constant-coefficient system given by A_d (F_d(q) = A_d q) and B_d, any m up to 64,
    dense or sparse, optionally with one Gaussian point source.  This is the probed form of an
    arbitrary reference LinearPde (tests/test_pde.cpp:14-24 probes it the same way: F_d(e_r) is
    column r of A_d); max_wavespeed is the user's max_wavespeed() (default: the largest
    characteristic speed, max_d max |eig(A_d + B_d)|)."""
    A = [np.ascontiguousarray(a, dtype=np.float64) for a in flux_jacobians]
    B = [None] * 3 if ncp_matrices is None else [np.ascontiguousarray(b, dtype=np.float64) for b in ncp_matrices]
    m = A[0].shape[0]
    args = []
    if source is not None:
        if not 0 <= source.component < m:
            raise StpError(ADERSTP_ERR_INVALID_ARG, "point source: component out of range")
        args = source.args() + [1.0]  # pde_args[7] != 0: the LinearPde carries this source
    return LinearPde(PDE_LINEAR, m, args, A + B, max_wavespeed)


# ----------------------------------------------------------------------------- outputs ------
@dataclass
class PredictorOutput:
    """Batched include/ader/predictor.hpp:22-29: qavg [E, ...], favg [E, 3, ...],
    face_q / face_f [E, 6, n*n*m] (faces -x,+x,-y,+y,-z,+z, quantity fastest)."""
    qavg: object
    favg: object
    face_q: object
    face_f: object


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class Plan:
    """One compiled configuration (order, PDE, layout).  Mirrors SolverConfig + BasisOperators
    + LinearPde of the reference; immutable; device constants only."""

    def __init__(self, order: int, pde: LinearPde, layout: int = LAYOUT_AOSOA, q_stride: int | None = None,
                 out_stride: int | None = None, par_kind: int = PAR_LAMBDA_MU_RHO, check_inputs: bool = True):
        self.order = order
        self.pde = pde
        self.m = pde.quantities
        self.layout = layout
        self.q_stride = q_stride or self.m
        self.out_stride = out_stride or self.m
        self.par_kind = par_kind
        cfg = _Config()
        cfg.order = order
        cfg.quantities = self.m
        cfg.pde_kind = pde.kind
        cfg.layout = layout
        cfg.q_stride = self.q_stride
        cfg.out_stride = self.out_stride
        cfg.par_kind = par_kind
        cfg.check_inputs = int(check_inputs)
        for i, v in enumerate(pde.args[:8]):
            cfg.pde_args[i] = v
        self._keep = []
        if pde.linear is not None:
            for i, mat in enumerate(pde.linear):
                if mat is not None:
                    self._keep.append(mat)
                    cfg.linear[i] = mat.ctypes.data_as(_dp)
        handle = _vp()
        _check(lib.aderstp_plan_create(ctypes.byref(cfg), ctypes.byref(handle)))
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.aderstp_plan_destroy(h)
            self._h = None

    # sizes (doubles per element)
    @property
    def q_size(self):
        return self.order ** 3 * self.q_stride

    @property
    def out_size(self):
        return self.order ** 3 * self.out_stride

    @property
    def face_size(self):
        return self.order * self.order * self.m

    def _uniform_par(self, n_elem, like):
        pde = self.pde
        if pde.lam is None:
            raise StpError(ADERSTP_ERR_INVALID_ARG, "elastic: pass per-element par or a uniform material")
        import torch
        row = ([pde.lam, pde.mu, pde.rho] if self.par_kind == PAR_LAMBDA_MU_RHO else
               [pde.rho, float(np.sqrt((pde.lam + 2 * pde.mu) / pde.rho)), float(np.sqrt(pde.mu / pde.rho))])
        if isinstance(like, np.ndarray):
            return np.tile(np.array(row), (n_elem, 1))
        return torch.tensor(row, dtype=torch.float64, device=like.device).repeat(n_elem, 1)

    def alloc_output(self, n_elem: int, device="cuda", want_favg=True, want_faces=True) -> PredictorOutput:
        import torch
        z = lambda *s: torch.empty(*s, dtype=torch.float64, device=device)  # noqa: E731
        return PredictorOutput(z(n_elem, self.out_size), z(n_elem, 3, self.out_size) if want_favg else None,
                               z(n_elem, 6, self.face_size) if want_faces else None,
                               z(n_elem, 6, self.face_size) if want_faces else None)

    def predict(self, q, dt: float, par=None, t_start: float = 0.0, out: PredictorOutput | None = None,
                stream=None, want_favg=True, want_faces=True) -> PredictorOutput:
        """Device path: q and par are CUDA float64 tensors (leading axis = element)."""
        import torch
        if not (isinstance(q, torch.Tensor) and q.is_cuda and q.dtype == torch.float64 and q.is_contiguous()):
            raise StpError(ADERSTP_ERR_INVALID_ARG, "predict: q must be a contiguous CUDA float64 tensor")
        n_elem = q.shape[0]
        if q.numel() != n_elem * self.q_size:
            raise StpError(ADERSTP_ERR_INVALID_ARG, "stp: input tensor shape does not match the plan")
        if self.pde.kind in (PDE_ELASTIC, PDE_ELASTIC_SOURCE) and par is None:
            par = self._uniform_par(n_elem, q)
        if par is not None and (par.dtype != torch.float64 or not par.is_contiguous() or par.numel() != 3 * n_elem):
            raise StpError(ADERSTP_ERR_INVALID_ARG, "stp: par must be a contiguous float64 [E, 3] tensor")
        if out is None:
            out = self.alloc_output(n_elem, q.device, want_favg, want_faces)
        ptr = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _check(lib.aderstp_predict_batch(self._h, n_elem, ptr(q), ptr(par), dt, t_start, ptr(out.qavg),
                                         ptr(out.favg), ptr(out.face_q), ptr(out.face_f), _stream_handle(stream)))
        return out

    # ---- GPU corrector and time loop (proj/src/solver.cpp) ---------------------------------
    def correct(self, u, elements_per_dim: int, out: PredictorOutput, par=None, domain_len: float = 1.0,
                max_wavespeed: float | None = None, stream=None, dt: float | None = None, t: float = 0.0):
        """corrector_step(mesh, outs, pde, ops, dt, t) (solver.cpp:257-311) in place on the device
        mesh state u [e^3, q_size] from this step's predictor outputs (computed on the 1/h-scaled
        PDE).  max_wavespeed: the PDE's unscaled max_wavespeed(); None = the PDE's own (elastic:
        per face from the material).  dt, t: the step (they enter through a point source only)."""
        import torch
        E = elements_per_dim ** 3
        if not (isinstance(u, torch.Tensor) and u.is_cuda and u.dtype == torch.float64 and u.is_contiguous()
                and u.numel() == E * self.q_size):
            raise StpError(ADERSTP_ERR_INVALID_ARG, "correct: u must be a contiguous CUDA float64 [e^3, q_size] tensor")
        if self.pde.kind in (PDE_ELASTIC, PDE_ELASTIC_SOURCE) and par is None:
            par = self._uniform_par(E, u)
        smax = self._smax(max_wavespeed)
        mesh = _Mesh(elements_per_dim, domain_len)
        ptr = lambda x: None if x is None else ctypes.c_void_p(x.data_ptr())  # noqa: E731
        _check(lib.aderstp_correct_batch(self._h, ctypes.byref(mesh), ptr(u), ptr(par), ptr(out.qavg),
                                         ptr(out.face_q), ptr(out.face_f), smax, self._step_dt(dt), float(t),
                                         _stream_handle(stream)))

    def _step_dt(self, dt):
        if dt is None:
            if self.pde.has_source:
                raise StpError(ADERSTP_ERR_INVALID_ARG, "corrector_step: a point-source PDE needs the step's dt")
            return 0.0
        return float(dt)

    def _smax(self, max_wavespeed):
        if max_wavespeed is not None:
            return float(max_wavespeed)
        if self.pde.kind in (PDE_ELASTIC, PDE_ELASTIC_SOURCE):
            return -1.0
        return float(self.pde.max_wavespeed())

    def run_simulation(self, u, elements_per_dim: int, t_end: float, par=None, cfl: float = 0.35,
                       domain_len: float = 1.0, max_wavespeed: float | None = None, stream=None):
        """run_simulation (solver.cpp:313-359) on the device mesh state u (in place).  Returns
        (stable, steps, t_final) like RunResult; raises on argument / CUDA errors."""
        import torch
        E = elements_per_dim ** 3
        if not (isinstance(u, torch.Tensor) and u.is_cuda and u.dtype == torch.float64 and u.is_contiguous()
                and u.numel() == E * self.q_size):
            raise StpError(ADERSTP_ERR_INVALID_ARG, "run_simulation: u must be a contiguous CUDA float64 tensor")
        if self.pde.kind in (PDE_ELASTIC, PDE_ELASTIC_SOURCE) and par is None:
            par = self._uniform_par(E, u)
        smax = self._smax(max_wavespeed)
        mesh = _Mesh(elements_per_dim, domain_len)
        steps, t_final = _i64(0), ctypes.c_double(0.0)
        ptr = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
        rc = lib.aderstp_run_simulation(self._h, ctypes.byref(mesh), ptr(u), ptr(par), cfl, t_end, smax,
                                        ctypes.byref(steps), ctypes.byref(t_final), _stream_handle(stream))
        if rc not in (ADERSTP_OK, ADERSTP_ERR_NONFINITE):
            _check(rc)
        return rc == ADERSTP_OK, steps.value, t_final.value

    # ---- the time loop on a z-slab of the mesh (one rank of a multi-GPU run) -----------------
    @staticmethod
    def _halo(h):
        """h = (face_q, face_f, par, z_base): device pointers (ints) or tensors."""
        if h is None:
            return None
        ptr = lambda t: None if t is None else (t if isinstance(t, int) else t.data_ptr())  # noqa: E731
        return _Halo(ptr(h[0]), ptr(h[1]), ptr(h[2]), int(h[3]))

    def correct_slab(self, u, elements_per_dim: int, slab, out: PredictorOutput, lo=None, hi=None, par=None,
                     domain_len: float = 1.0, max_wavespeed: float | None = None, stream=None,
                     dt: float | None = None, t: float = 0.0):
        """corrector_step on the layers [z0, z0 + nz) (slab = (z0, nz)); z-neighbours outside the
        slab come from the halos lo / hi = (face_q, face_f, par, z_base) of the adjacent slabs."""
        mesh, sl = _Mesh(elements_per_dim, domain_len), _Slab(*slab)
        hl, hh = self._halo(lo), self._halo(hi)
        ptr = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _check(lib.aderstp_correct_slab(self._h, ctypes.byref(mesh), ctypes.byref(sl), ptr(u), ptr(par),
                                        ptr(out.qavg), ptr(out.face_q), ptr(out.face_f),
                                        ctypes.byref(hl) if hl else None, ctypes.byref(hh) if hh else None,
                                        self._smax(max_wavespeed), self._step_dt(dt), float(t),
                                        _stream_handle(stream)))

    def run_simulation_slab(self, u, elements_per_dim: int, slab, face_q, face_f, t_end: float,
                            max_wavespeed: float, lo=None, hi=None, par=None, cfl: float = 0.35,
                            domain_len: float = 1.0, sync=None, stream=None):
        """aderstp_run_simulation_slab: this rank's slab (z0, nz); face_q / face_f its predictor
        output buffers (tensors or device pointers) shared with the neighbours; sync(flag) -> max
        over ranks (shard.make_rank_sync()).  Returns (stable, steps, t_final)."""
        mesh, sl = _Mesh(elements_per_dim, domain_len), _Slab(*slab)
        hl, hh = self._halo(lo), self._halo(hi)
        cb = _SyncFn(lambda ctx, flag: int(sync(int(flag)))) if sync is not None else _SyncFn(0)
        steps, t_final = _i64(0), ctypes.c_double(0.0)
        vp = lambda t: None if t is None else ctypes.c_void_p(t if isinstance(t, int) else t.data_ptr())  # noqa: E731
        rc = lib.aderstp_run_simulation_slab(self._h, ctypes.byref(mesh), ctypes.byref(sl), vp(u), vp(par), vp(face_q),
                                             vp(face_f), ctypes.byref(hl) if hl else None,
                                             ctypes.byref(hh) if hh else None, cfl, t_end, float(max_wavespeed),
                                             cb, None, ctypes.byref(steps), ctypes.byref(t_final),
                                             _stream_handle(stream))
        if rc not in (ADERSTP_OK, ADERSTP_ERR_NONFINITE):
            _check(rc)
        return rc == ADERSTP_OK, steps.value, t_final.value

    def trim(self):
        """Return the plan's pooled device scratch (AoS staging, time-loop buffers) to the device."""
        _check(lib.aderstp_plan_trim(self._h))

    def status(self, stream=None):
        """Synchronise and raise on flagged inputs (validate_stp's non-finite / material checks)."""
        _check(lib.aderstp_plan_status(self._h, _stream_handle(stream)))

    def predict_host(self, q: np.ndarray, dt: float, par: np.ndarray | None = None, t_start: float = 0.0,
                     out: PredictorOutput | None = None, want_favg=True, want_faces=True) -> PredictorOutput:
        """Host path (aderstp_predict_batch_host): numpy in, numpy out, copies pipelined."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        n_elem = q.shape[0]
        if q.size != n_elem * self.q_size:
            raise StpError(ADERSTP_ERR_INVALID_ARG, "stp: input tensor shape does not match the plan")
        if self.pde.kind in (PDE_ELASTIC, PDE_ELASTIC_SOURCE):
            par = self._uniform_par(n_elem, q) if par is None else np.ascontiguousarray(par, dtype=np.float64)
        if out is None:
            out = PredictorOutput(np.empty((n_elem, self.out_size)),
                                  np.empty((n_elem, 3, self.out_size)) if want_favg else None,
                                  np.empty((n_elem, 6, self.face_size)) if want_faces else None,
                                  np.empty((n_elem, 6, self.face_size)) if want_faces else None)
        _check(lib.aderstp_predict_batch_host(self._h, n_elem, _np_ptr(q), _np_ptr(par), dt, t_start,
                                              _np_ptr(out.qavg), _np_ptr(out.favg), _np_ptr(out.face_q),
                                              _np_ptr(out.face_f)))
        return out

    def reserve_host_path(self, chunk_elems: int):
        _check(lib.aderstp_plan_reserve_host_path(self._h, chunk_elems))


_plan_cache: dict = {}


def predict(q, pde: LinearPde, dt: float, order: int | None = None, par=None, t_start: float = 0.0,
            layout: int = LAYOUT_AOSOA, q_stride=None, out_stride=None, stream=None) -> PredictorOutput:
    """Batched ader::predict + extrapolate_faces on CUDA tensors (plan cached per config)."""
    if order is None:
        per = q.shape[1] if q.dim() == 2 else int(np.prod(q.shape[1:]))
        order = round((per / (q_stride or pde.quantities)) ** (1.0 / 3.0))
    key = (order, pde.kind, pde.quantities, tuple(pde.args), layout, q_stride, out_stride,
           None if pde.linear is None else tuple(id(x) for x in pde.linear))
    plan = _plan_cache.get(key)
    if plan is None:
        plan = _plan_cache[key] = Plan(order, pde, layout, q_stride, out_stride)
    return plan.predict(q, dt, par=par, t_start=t_start, stream=stream)


def generate(dist: int, seed: int, order: int, e0: int, n_elem: int, grid: int = 1, layout: int = LAYOUT_AOSOA,
             q_stride: int = 9, q=None, par=None, stream=None):
    """Seeded synthetic elastic inputs on the device; returns (q, par)."""
    import torch
    if q is None:
        q = torch.empty(n_elem, order ** 3 * q_stride, dtype=torch.float64, device="cuda")
    if par is None:
        par = torch.empty(n_elem, 3, dtype=torch.float64, device="cuda")
    _check(lib.aderstp_generate(dist, seed, order, e0, n_elem, grid, layout, q_stride,
                                ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(par.data_ptr()),
                                _stream_handle(stream)))
    return q, par


def convert_layout(order, quantities, n_elem, src_layout, src_stride, src, dst_layout, dst_stride, dst,
                   stream=None):
    """AoS <-> AoSoA on the device (src/layout.cpp:168-194)."""
    _check(lib.aderstp_convert_layout(order, quantities, n_elem, src_layout, src_stride,
                                      ctypes.c_void_p(src.data_ptr()), dst_layout, dst_stride,
                                      ctypes.c_void_p(dst.data_ptr()), _stream_handle(stream)))
    return dst


# ---- shareable device buffers and CUDA IPC (multi-GPU time loop) --------------------------------
def device_alloc(nbytes: int) -> int:
    p = _vp()
    _check(lib.aderstp_device_alloc(nbytes, ctypes.byref(p)))
    return p.value


def device_free(ptr: int):
    _check(lib.aderstp_device_free(ctypes.c_void_p(ptr)))


def ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(lib.aderstp_ipc_handle(ctypes.c_void_p(ptr), buf))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    p = _vp()
    _check(lib.aderstp_ipc_open(handle, ctypes.byref(p)))
    return p.value


def ipc_close(ptr: int):
    _check(lib.aderstp_ipc_close(ctypes.c_void_p(ptr)))
