"""TEST INFRASTRUCTURE ONLY -- CPU checkers for the STP hot path.

Two checkers live here; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only as the checker
or the timed CPU baseline -- never as part of the product path:

* ``Oracle``: ctypes binding of ``oracle/libstp_oracle.so``, our plain-C restatement of the
  reference's SplitCK predictor (``stp_oracle.c``; each function cites the reference file:line
  it restates).
* ``Reference``: ctypes binding of ``oracle/_ref/libader_ref_v{3,4}.so``, the UNMODIFIED
  reference C++ sources (``/root/reference/proj/src``) compiled by ``oracle/Makefile`` plus our
  batch shim ``ref_shim.cpp``.  Built here (where the reference is mounted) and shipped to the
  GPU box as a prebuilt file.

Canonical batch layout for both: q/qavg ``[e][k3][k2][k1][s]``, favg ``[e][3][...]``,
faces ``[e][6][a][b][s]``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
REFERENCE_SRC = "/root/reference/proj"

PDE_ELASTIC, PDE_ADVECTION, PDE_NCP_ADVECTION, PDE_DEMO, PDE_ELASTIC_SOURCE, PDE_SOURCE_ONLY, PDE_MATRIX = range(7)
VARIANTS = {"generic": 0, "log": 1, "splitck": 2, "aosoa": 3}

_dp = ctypes.POINTER(ctypes.c_double)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


def build(with_reference: bool | None = None) -> None:
    """Compile the C restatement (always) and the reference library (when the reference
    sources are mounted, i.e. in the build container, not on the GPU box)."""
    targets = ["all"]
    if with_reference is None:
        with_reference = os.path.isdir(REFERENCE_SRC)
    if with_reference:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


@dataclass
class Outputs:
    qavg: np.ndarray
    favg: np.ndarray | None
    face_q: np.ndarray | None
    face_f: np.ndarray | None
    seconds: float = 0.0


def _alloc(n, m, n_elem, want_favg=True, want_faces=True):
    vol = n ** 3 * m
    face = n * n * m
    return (np.zeros((n_elem, vol)),
            np.zeros((n_elem, 3, vol)) if want_favg else None,
            np.zeros((n_elem, 6, face)) if want_faces else None,
            np.zeros((n_elem, 6, face)) if want_faces else None)


class Oracle:
    """Our C restatement of the reference hot path (stp_oracle.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "libstp_oracle.so")
        if not os.path.exists(path):
            build(with_reference=False)
        lib = ctypes.CDLL(path)
        lib.orc_make_basis.argtypes = [ctypes.c_int] + [_dp] * 5
        lib.orc_splitmix64_at.restype = ctypes.c_uint64
        lib.orc_splitmix64_at.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.orc_generate.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_long,
                                     ctypes.c_long, ctypes.c_int, _dp, _dp]
        lib.orc_material_lmr.argtypes = [ctypes.c_long, _dp, _dp]
        lib.orc_stp_batch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_long, _dp, _dp, _dp,
                                      ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp, _dp, _dp,
                                      _dp, ctypes.c_int]
        lib.orc_corrector_step.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                           _dp, _dp, ctypes.c_double, _dp, _dp, _dp, _dp]
        lib.orc_canonical_to_aosoa.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long, _dp, _dp]
        lib.orc_aosoa_to_canonical.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long, _dp, _dp]
        self.lib = lib

    def basis(self, n):
        nodes, w, fl, fr = (np.zeros(n) for _ in range(4))
        d = np.zeros(n * n)
        if self.lib.orc_make_basis(n, _ptr(nodes), _ptr(w), _ptr(d), _ptr(fl), _ptr(fr)) != 0:
            raise ValueError("order out of range")
        return dict(nodes=nodes, weights=w, d=d.reshape(n, n), face_left=fl, face_right=fr)

    def splitmix(self, seed, count, start=0):
        return [self.lib.orc_splitmix64_at(seed, start + k) for k in range(count)]

    def generate(self, dist, seed, n, e0, count, grid=1):
        q = np.zeros((count, n ** 3 * 9))
        par = np.zeros((count, 3))
        self.lib.orc_generate(dist, seed, n, e0, count, grid, _ptr(q), _ptr(par))
        return q, par

    def material_lmr(self, par_rcc):
        par_rcc = np.ascontiguousarray(par_rcc, dtype=np.float64)
        out = np.zeros_like(par_rcc)
        self.lib.orc_material_lmr(par_rcc.shape[0], _ptr(par_rcc), _ptr(out))
        return out

    def stp(self, n, m, q, dt, par=None, pde_kind=PDE_ELASTIC, args=None, t_start=0.0,
            threads=None, want_favg=True, want_faces=True) -> Outputs:
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, n ** 3 * m)
        n_elem = q.shape[0]
        par_a = None if par is None else np.ascontiguousarray(par, dtype=np.float64).reshape(-1, 3)
        args_a = np.zeros(8) if args is None else np.ascontiguousarray(args, dtype=np.float64)
        qavg, favg, fq, ff = _alloc(n, m, n_elem, want_favg, want_faces)
        threads = threads or min(os.cpu_count() or 1, 16)
        rc = self.lib.orc_stp_batch(n, m, n_elem, _ptr(q), _ptr(par_a), _ptr(args_a), pde_kind, dt,
                                    t_start, _ptr(qavg), _ptr(favg), _ptr(fq), _ptr(ff), threads)
        if rc != 0:
            raise ValueError("oracle: invalid arguments (validate_stp semantics)")
        return Outputs(qavg, favg, fq, ff)

    def corrector_step(self, n, m, e, domain_len, u, qavg, face_q, face_f, max_wavespeed, par=None,
                       pde_kind=PDE_ELASTIC, args=None):
        """orc_corrector_step (restates proj/src/solver.cpp:184-311); returns (u, finite)."""
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        par_a = None if par is None else np.ascontiguousarray(par, dtype=np.float64).reshape(3)
        args_a = np.zeros(8) if args is None else np.ascontiguousarray(args, dtype=np.float64)
        rc = self.lib.orc_corrector_step(n, m, e, domain_len, pde_kind, _ptr(par_a), _ptr(args_a), max_wavespeed,
                                         _ptr(u), _ptr(np.ascontiguousarray(qavg, dtype=np.float64)),
                                         _ptr(np.ascontiguousarray(face_q, dtype=np.float64)),
                                         _ptr(np.ascontiguousarray(face_f, dtype=np.float64)))
        if rc == -1:
            raise ValueError("oracle: invalid corrector arguments")
        return u, rc == 0

    def to_aosoa(self, n, m, qs, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        n_elem = q.size // (n ** 3 * m)
        out = np.zeros((n_elem, n * n * qs * n))
        self.lib.orc_canonical_to_aosoa(n, m, qs, n_elem, _ptr(q), _ptr(out))
        return out

    def from_aosoa(self, n, m, qs, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        n_elem = x.size // (n * n * qs * n)
        out = np.zeros((n_elem, n ** 3 * m))
        self.lib.orc_aosoa_to_canonical(n, m, qs, n_elem, _ptr(x), _ptr(out))
        return out


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return " avx512f" in f.read()
    except OSError:
        return False


def reference_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libader_ref_v3.so"))


class Reference:
    """The unmodified reference library (oracle/_ref), driven through its own predict()."""

    def __init__(self):
        isa = "v4" if _cpu_has_avx512() else "v3"
        path = os.path.join(REF_DIR, f"libader_ref_{isa}.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        lib = ctypes.CDLL(path)
        lib.ref_stp_batch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long, _dp, _dp,
                                      _dp, ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp, _dp,
                                      _dp, _dp, ctypes.c_int, _dp]
        lib.ref_set_matrix_pde.argtypes = [ctypes.c_int, _dp, _dp, _dp, ctypes.c_double]
        lib.ref_stp_batch_matrix.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long, _dp, _dp, _dp,
                                             ctypes.c_double, _dp, _dp, _dp, _dp, ctypes.c_int, _dp]
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_make_basis.argtypes = [ctypes.c_int] + [_dp] * 5
        lib.ref_splitmix64.argtypes = [ctypes.c_uint64, ctypes.c_long, ctypes.POINTER(ctypes.c_uint64)]
        lib.ref_flop_count.restype = ctypes.c_uint64
        lib.ref_flop_count.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.ref_volume_operator.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp]
        _i = ctypes.c_int
        lib.ref_corrector_step.argtypes = [_i, _i, _i, ctypes.c_double, _i, _dp, _dp, ctypes.c_double,
                                           ctypes.c_double, _dp, _dp, _dp, _dp, _i]
        lib.ref_run_simulation.argtypes = [_i, _i, _i, ctypes.c_double, _i, _dp, _dp, ctypes.c_double,
                                           ctypes.c_double, _i, _dp, _i, ctypes.POINTER(_i), ctypes.POINTER(_i),
                                           _dp]
        lib.ref_max_wavespeed.restype = ctypes.c_double
        lib.ref_max_wavespeed.argtypes = [_i, _i, _dp, _dp]
        self.lib = lib
        self.isa = isa
        self.path = path

    def basis(self, n):
        nodes, w, fl, fr = (np.zeros(n) for _ in range(4))
        d = np.zeros(n * n)
        if self.lib.ref_make_basis(n, _ptr(nodes), _ptr(w), _ptr(d), _ptr(fl), _ptr(fr)) != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return dict(nodes=nodes, weights=w, d=d.reshape(n, n), face_left=fl, face_right=fr)

    def splitmix(self, seed, count):
        out = (ctypes.c_uint64 * count)()
        self.lib.ref_splitmix64(seed, count, out)
        return list(out)

    def volume_operator(self, n, m, pde_kind, par=None, args=None):
        out = np.zeros((n ** 3 * m) ** 2)
        par_a = None if par is None else np.ascontiguousarray(par, dtype=np.float64)
        args_a = np.zeros(8) if args is None else np.ascontiguousarray(args, dtype=np.float64)
        if self.lib.ref_volume_operator(n, m, pde_kind, _ptr(par_a), _ptr(args_a), _ptr(out)) != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return out.reshape(n ** 3 * m, n ** 3 * m)

    def stp(self, n, m, q, dt, par=None, pde_kind=PDE_ELASTIC, args=None, t_start=0.0,
            variant="splitck", threads=None, want_favg=True, want_faces=True) -> Outputs:
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, n ** 3 * m)
        n_elem = q.shape[0]
        par_a = None if par is None else np.ascontiguousarray(par, dtype=np.float64).reshape(-1, 3)
        args_a = np.zeros(8) if args is None else np.ascontiguousarray(args, dtype=np.float64)
        qavg, favg, fq, ff = _alloc(n, m, n_elem, want_favg, want_faces)
        secs = ctypes.c_double(0.0)
        threads = threads or (os.cpu_count() or 1)
        rc = self.lib.ref_stp_batch(VARIANTS[variant], n, m, n_elem, _ptr(q), _ptr(par_a), _ptr(args_a),
                                    pde_kind, dt, t_start, _ptr(qavg), _ptr(favg), _ptr(fq), _ptr(ff),
                                    threads, ctypes.byref(secs))
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return Outputs(qavg, favg, fq, ff, secs.value)


    def set_matrix_pde(self, A, B=None, source=None, max_wavespeed=1.0):
        """Make pde kind PDE_MATRIX (6) a user LinearPde with flux A_d, ncp B_d, optional point
        source (7 doubles: position, component, amplitude, center, width; the reference's own
        Gaussian) and the given max_wavespeed(), for stp / corrector_step / run_simulation."""
        a = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.float64) for x in A]))
        b = None if B is None else np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.float64) for x in B]))
        src = None if source is None else np.ascontiguousarray(source, dtype=np.float64)[:7].copy()
        if self.lib.ref_set_matrix_pde(a.shape[1], _ptr(a), _ptr(b), _ptr(src), float(max_wavespeed)) != 0:
            raise ValueError(self.lib.ref_last_error().decode())

    def stp_matrix(self, n, m, q, dt, A, B=None, variant="splitck", threads=None) -> Outputs:
        """The reference predict() + extrapolate_faces for a user LinearPde given by its
        matrices A_d (F_d(q) = A_d q) and B_d (ncp), via the shim's MatrixPde."""
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, n ** 3 * m)
        a = np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.float64) for x in A]))
        b = None if B is None else np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.float64) for x in B]))
        qavg, favg, fq, ff = _alloc(n, m, q.shape[0])
        secs = ctypes.c_double(0.0)
        rc = self.lib.ref_stp_batch_matrix(VARIANTS[variant], n, m, q.shape[0], _ptr(q), _ptr(a), _ptr(b), dt,
                                           _ptr(qavg), _ptr(favg), _ptr(fq), _ptr(ff),
                                           threads or (os.cpu_count() or 1), ctypes.byref(secs))
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return Outputs(qavg, favg, fq, ff, secs.value)

    # ---- corrector / time loop (proj/src/solver.cpp); mesh state canonical [c][k3][k2][k1][s] ----
    def corrector_step(self, n, m, e, domain_len, u, qavg, face_q, face_f, dt, par=None,
                       pde_kind=PDE_ELASTIC, args=None, t=0.0, workers=None):
        """ader::corrector_step with ONE shared PDE (par = (lambda, mu, rho)); returns (u, ok)."""
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        qavg = np.ascontiguousarray(qavg, dtype=np.float64)
        face_q = np.ascontiguousarray(face_q, dtype=np.float64)
        face_f = np.ascontiguousarray(face_f, dtype=np.float64)
        par_a = None if par is None else np.ascontiguousarray(par, dtype=np.float64).reshape(3)
        args_a = np.zeros(8) if args is None else np.ascontiguousarray(args, dtype=np.float64)
        rc = self.lib.ref_corrector_step(n, m, e, domain_len, pde_kind, _ptr(par_a), _ptr(args_a), dt, t,
                                         _ptr(u), _ptr(qavg), _ptr(face_q), _ptr(face_f),
                                         workers or (os.cpu_count() or 1))
        if rc == -1:
            raise ValueError(self.lib.ref_last_error().decode())
        return u, rc == 0

    def run_simulation(self, n, m, e, domain_len, u, cfl, t_end, par=None, pde_kind=PDE_ELASTIC,
                       args=None, variant="splitck", workers=None):
        """ader::run_simulation; returns (u, stable, steps, t_final)."""
        u = np.ascontiguousarray(u, dtype=np.float64).copy()
        par_a = None if par is None else np.ascontiguousarray(par, dtype=np.float64).reshape(3)
        args_a = np.zeros(8) if args is None else np.ascontiguousarray(args, dtype=np.float64)
        stable, steps, t_final = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_double(0.0)
        rc = self.lib.ref_run_simulation(n, m, e, domain_len, pde_kind, _ptr(par_a), _ptr(args_a), cfl,
                                         t_end, VARIANTS[variant], _ptr(u), workers or (os.cpu_count() or 1),
                                         ctypes.byref(stable), ctypes.byref(steps), ctypes.byref(t_final))
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return u, bool(stable.value), steps.value, t_final.value

    def max_wavespeed(self, pde_kind, m, par=None, args=None):
        par_a = None if par is None else np.ascontiguousarray(par, dtype=np.float64).reshape(3)
        args_a = np.zeros(8) if args is None else np.ascontiguousarray(args, dtype=np.float64)
        return self.lib.ref_max_wavespeed(pde_kind, m, _ptr(par_a), _ptr(args_a))


def rel_diff(a, b) -> float:
    """The reference's parity metric: max|a-b| / max|a| (proj/src/checks.cpp:27-34)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(a))) if a.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b))) / scale if a.size else 0.0


def per_element_rel_diff(a, b) -> float:
    """Worst per-element rel_diff over a batch shaped [e, ...]."""
    a = np.asarray(a).reshape(a.shape[0], -1)
    b = np.asarray(b).reshape(b.shape[0], -1)
    scale = np.maximum(np.max(np.abs(a), axis=1), 1e-300)
    return float(np.max(np.max(np.abs(a - b), axis=1) / scale)) if a.size else 0.0


def cfl_dt(n: int, cp_max: float, cfl: float = 0.5, h: float = 1.0) -> float:
    """stable_dt (proj/src/solver.cpp:170-174) with BASELINE's CFL 0.5."""
    return cfl * h / (3.0 * cp_max * (2.0 * n - 1.0))
