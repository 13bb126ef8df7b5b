// The user-LinearPde path for systems the term-table kernels cannot take: any number of
// quantities (1..ADERSTP_MAX_QUANTITIES), dense or sparse flux / ncp matrices, an optional
// Gaussian point source, every order 2..10 and both layouts.
//
// The reference accepts any constant-coefficient LinearPde (proj/include/ader/pde.hpp:21-46) and
// runs its SplitCK recursion (proj/src/stp_splitck.cpp:13-81) on it:
//   p_0 = q,  Qbar = dt q,  p_o = sum_d D_d F_d(p_(o-1)) + B_d (D_d p_(o-1)) + P S^(o-1)(t0),
//   Qbar += c_o p_o (c_o = c_(o-1) dt / (o+1)),  favg_d = F_d(Qbar),  faces of Qbar / favg.
// For constant coefficients D_d F_d(p) + B_d D_d p = C_d (D_d p) with C_d = A_d + B_d, so a CK
// step is "derivatives first, then one pointwise matrix":
//   phase z: D_z p_j for every quantity j, one z-line per task (N loads, N outputs), into the
//            buffer that will hold p_o (the z workspace of a plane is dead once its p_o is known);
//   then per k3 plane -- phase xy: D_x p_j and D_y p_j of the plane, one line per task;
//            phase 2: t_s = sum_d sum_(j in row s of C_d) C_d[s][j] (D_d p_j) (+ the point
//            source) = p_o of the plane, staged and copied over the plane's z workspace while the
//            next plane's lines run; Qbar += c_o t_s is kept in the caller's qavg buffer (the
//            thread that owns an entry owns it in every step: no race, L2-resident).
// The matrices live in device memory as per-(s, d) row lists (CSR), read warp-uniformly.  The
// iterate pair (p_(o-1), p_o) and the plane workspace sit in shared memory when they fit
// (2 m N^3 + 3 m N^2 doubles, 6 m N^2 for N < 6); larger systems (e.g. m = 21 at nDof 10) use a
// per-element slice of a plan-owned global scratch instead -- correct for every size, slower.
#include <cmath>
#include <cstdint>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"

namespace aderstp {

namespace {

// threads per element: 512 from nDof 8 on (one CTA per SM at most of these sizes; measured m = 8
// nDof 10 +30 %, m = 21 nDof 8 +14 %), 256 below (nDof 4 -20 % with 512)
template <int N>
constexpr int gen_threads() { return N >= 8 ? 512 : 256; }
constexpr int kSB = 8;  // targets per task of the dense phase 2 (the padded dense rows cover them)

struct GenParams {
  double d[kMaxOrder * kMaxOrder];   // d[k*N + l]
  double phi[2][kMaxOrder];
  double cf[kMaxOrder];              // c_1 .. c_(N-1) in the reference's operation sequence
  double src_amp[kMaxOrder];         // S^(o)(t0) x source scale, o = 0..N-2
  double src_proj[3][kMaxOrder];     // phi_d(x_src)[k] / w[k]
  int src_comp;                      // < 0: no source
  int m, q_stride, out_stride, layout, check;
  double scale;                      // ScaledPde gradient scale (1 outside the time loop)
  const int* t_ptr;                  // C_d rows: entries [t_ptr[3s+d], t_ptr[3s+d+1])
  const int* t_col;                  // source quantity j of the entry
  const double* t_val;
  int t_nnz, csr_smem;               // csr_smem: stage the C rows in shared memory
  const double* t_dense;             // dense C: [d][j][s < m_pad] (null: rows only)
  int dense, m_pad;                  // dense: phase 2 by target blocks from the dense C in smem
  const int* f_ptr;                  // A_d rows (favg, face_f)
  const int* f_col;
  const double* f_val;
  double* scratch;                   // global scratch (2 m N^3 per element) or null: shared memory
  int vol_mode;                      // corrector volume term: u += scale * L(qavg), nothing else
};

template <int N>
__device__ __forceinline__ long long lidx(int layout, int stride, int s, int k3, int k2, int k1) {
  return layout == ADERSTP_LAYOUT_AOSOA ? (((long long)k3 * N + k2) * stride + s) * N + k1
                                        : (((long long)k3 * N + k2) * N + k1) * stride + s;
}

// GS: the iterate pair in the plan's global scratch (large m N^3) instead of shared memory -- a
// compile-time choice, so that the shared-memory instance addresses it with LDS / STS (a pointer
// that may point to either space makes every access a generic LD / ST)
template <int N, bool GS>
__global__ void __launch_bounds__(gen_threads<N>()) stp_general_kernel(GenParams kp, BatchArgs a, unsigned int* status) {
  constexpr int kGenThreads = gen_threads<N>();
  extern __shared__ __align__(16) double smg[];
  constexpr int N2 = N * N, N3 = N * N * N;
  const int m = kp.m;
  const long long e = blockIdx.x;
  const int tid = threadIdx.x;
  double* Ds = smg;                         // D, N x N
  // plane workspace: 3 m N^2 (CK step); for N < 6 also the face staging (6 m N^2), for N >= 6 the
  // faces are staged in the dead iterate buffer instead (m N^3 >= 6 m N^2)
  double* W = smg + N2 + (N2 & 1);
  double* P;                                // p_(o-1)
  if constexpr (GS) {
    P = kp.scratch + e * (2ll * m * N3);
  } else {
    P = W + (N >= 6 ? 3 : 6) * m * N2;
  }
  double* R = P + (long long)m * N3;        // p_o; the final Qbar in the epilogue
  unsigned int flags = 0;
  for (int i = tid; i < N2; i += kGenThreads) Ds[i] = kp.d[i];
  // the CK step's coefficient rows, staged once per element next to the buffers when they fit
  // (warp-uniform broadcast reads instead of dependent L1 round trips)
  double* csr_v = nullptr;  // the CSR rows staged in shared memory (csr_smem)
  int* csr_c = nullptr;
  int* csr_p = nullptr;
  double* Cd = nullptr;  // dense C staged in shared memory (dense mode)
  if (kp.dense) {
    Cd = (GS ? W + (N >= 6 ? 3 : 6) * m * N2 : R + (long long)m * N3);
    Cd += (reinterpret_cast<uintptr_t>(Cd) & 15) ? 1 : 0;  // 16-byte aligned for LDS.128 (pointer arithmetic
                                                           // keeps the shared address space)
    for (int i = tid; i < 3 * m * kp.m_pad; i += kGenThreads) Cd[i] = kp.t_dense[i];
  } else if (kp.csr_smem) {
    double* sv = (GS ? W + (N >= 6 ? 3 : 6) * m * N2 : R + (long long)m * N3);
    int* so = reinterpret_cast<int*>(sv + kp.t_nnz);
    int* sp = so + kp.t_nnz;
    for (int i = tid; i < kp.t_nnz; i += kGenThreads) {
      sv[i] = kp.t_val[i];
      so[i] = kp.t_col[i];
    }
    for (int i = tid; i <= 3 * m; i += kGenThreads) sp[i] = kp.t_ptr[i];
    csr_v = sv;
    csr_c = so;
    csr_p = sp;
  }

  // ---- stage p_0 = q (canonical [s][k3][k2][k1]) and Qbar = dt q into the output --------
  const double* qe = a.q + e * (long long)N3 * kp.q_stride;
  double* qa = kp.vol_mode ? nullptr : a.qavg + e * (long long)N3 * kp.out_stride;
  const double* src0 = kp.vol_mode ? a.vol_r + e * (long long)N3 * kp.out_stride : qe;
  const int s_stride = kp.vol_mode ? kp.out_stride : kp.q_stride;
  for (int i = tid; i < m * N3; i += kGenThreads) {
    const int s = i / N3, node = i - s * N3;
    const int k3 = node / N2, k2 = (node / N) % N, k1 = node % N;
    const double v = src0[lidx<N>(kp.layout, s_stride, s, k3, k2, k1)];
    if (kp.check && !isfinite(v)) flags |= 1u;
    P[i] = v;
    if (qa) qa[lidx<N>(kp.layout, kp.out_stride, s, k3, k2, k1)] = a.dt * v;
  }
  __syncthreads();

  const int steps = kp.vol_mode ? 1 : N - 1;
  double* Wx = W;                    // D_x p_j on the current plane   [j][k2][k1]
  double* Wy = W + m * N2;           // D_y p_j on the current plane
  double* Wt = W + 2 * m * N2;       // p_o of the current plane, staged until its copy into R
#pragma unroll 1
  for (int o = 1; o <= steps; ++o) {
    // phase z (all planes at once): R[j][k3][k2][k1] = (D_z p_j), one z-line per task -- N
    // loads and N outputs (R doubles as the z workspace until each plane's p_o replaces it)
    for (int i = tid; i < m * N2; i += kGenThreads) {
      const int j = i / N2, node = i - j * N2;
      const double* col = P + (long long)j * N3 + node;
      double c[N];
#pragma unroll
      for (int l = 0; l < N; ++l) c[l] = col[l * N2];
      double* out = R + (long long)j * N3 + node;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) acc = fma(Ds[k * N + l], c[l], acc);
        out[k * N2] = acc;
      }
    }
#pragma unroll 1
    for (int k3 = 0; k3 <= N; ++k3) {
      // phase xy of plane k3 (x lines (j, k2), y lines (j, k1): N loads, N outputs each), and
      // the copy of plane k3-1's p_o from Wt into R (its z workspace is no longer read)
      if (k3 < N)
        for (int i = tid; i < 2 * m * N; i += kGenThreads) {
          const int dj = i / N, r = i - dj * N;
          const int d = dj / m, j = dj - d * m;
          const double* pj = P + (long long)j * N3 + k3 * N2;
          double c[N];
          if (d == 0) {
#pragma unroll
            for (int l = 0; l < N; ++l) c[l] = pj[r * N + l];
          } else {
#pragma unroll
            for (int l = 0; l < N; ++l) c[l] = pj[l * N + r];
          }
          double* out = (d == 0 ? Wx + j * N2 + r * N : Wy + j * N2 + r);
          const int ostride = d == 0 ? 1 : N;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double acc = 0.0;
#pragma unroll
            for (int l = 0; l < N; ++l) acc = fma(Ds[k * N + l], c[l], acc);
            out[k * ostride] = acc;
          }
        }
      if (k3 > 0 && !kp.vol_mode)
        for (int i = tid; i < m * N2; i += kGenThreads) {
          const int j = i / N2, node = i - j * N2;
          R[(long long)j * N3 + (k3 - 1) * N2 + node] = Wt[i];
        }
      __syncthreads();
      if (k3 == N) break;
      // phase 2: t_s = sum_d C_d[s][.] (D_d p)[.] (+ source); Qbar += c_o p_o; p_o -> Wt
      const double* Wz = R + k3 * N2;
      if (kp.dense) {  // dense C: a task = (node, block of kSB targets), each D_d p_j loaded once
        const int nb = (m + kSB - 1) / kSB;
        for (int i = tid; i < nb * N2; i += kGenThreads) {
          const int sb = i / N2, node = i - sb * N2;
          const int k2 = node / N, k1 = node - k2 * N, s0 = sb * kSB;
          double acc[kSB];
#pragma unroll
          for (int q = 0; q < kSB; ++q) acc[q] = 0.0;
#pragma unroll 1
          for (int d = 0; d < 3; ++d) {
            const double* base = d == 0 ? Wx + node : d == 1 ? Wy + node : Wz + node;
            const int js = d == 2 ? N3 : N2;
            const double* cr = Cd + (long long)d * m * kp.m_pad + s0;
#pragma unroll 2
            for (int j = 0; j < m; ++j) {
              const double w = base[j * js];
              const double* c = cr + j * kp.m_pad;
#pragma unroll
              for (int q = 0; q < kSB; q += 2) {
                const double2 cc = *reinterpret_cast<const double2*>(c + q);
                acc[q] = fma(cc.x, w, acc[q]);
                acc[q + 1] = fma(cc.y, w, acc[q + 1]);
              }
            }
          }
#pragma unroll
          for (int q = 0; q < kSB; ++q) {
            const int s = s0 + q;
            if (s >= m) break;
            double t = acc[q] * kp.scale;
            if (kp.vol_mode) {
              double* u = a.u_next + e * (long long)N3 * kp.q_stride + lidx<N>(kp.layout, kp.q_stride, s, k3, k2, k1);
              const double nv = *u + t;
              if (!isfinite(nv)) flags |= 1u;
              *u = nv;
              continue;
            }
            if (s == kp.src_comp)
              t = fma(kp.src_proj[2][k3] * (kp.src_proj[1][k2] * kp.src_proj[0][k1]), kp.src_amp[o - 1], t);
            double* ac = qa + lidx<N>(kp.layout, kp.out_stride, s, k3, k2, k1);
            const double nq = fma(kp.cf[o], t, *ac);
            *ac = nq;
            Wt[s * N2 + node] = o == N - 1 ? nq : t;
          }
        }
        __syncthreads();
        continue;
      }
      for (int i = tid; i < m * N2; i += kGenThreads) {
        const int s = i / N2, node = i - s * N2;
        const int k2 = node / N, k1 = node - k2 * N;
        double t0 = 0.0, t1 = 0.0;
        // the CSR rows from shared memory (staged) or from the global tables: two code paths, so
        // that each addresses its own space (LDS / LDG instead of generic loads)
        auto rows = [&](const double* rv, const int* rc, const int* rp) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const double* base = d == 0 ? Wx + node : d == 1 ? Wy + node : Wz + node;
            const int js = d == 2 ? N3 : N2;
            const int end = rp[3 * s + d + 1];
            int k = rp[3 * s + d];
            for (; k + 1 < end; k += 2) {
              t0 = fma(rv[k], base[rc[k] * js], t0);
              t1 = fma(rv[k + 1], base[rc[k + 1] * js], t1);
            }
            if (k < end) t0 = fma(rv[k], base[rc[k] * js], t0);
          }
        };
        if (kp.csr_smem)
          rows(csr_v, csr_c, csr_p);
        else
          rows(kp.t_val, kp.t_col, kp.t_ptr);
        double t = (t0 + t1) * kp.scale;
        if (kp.vol_mode) {  // corrector: u += V(qavg)
          double* u = a.u_next + e * (long long)N3 * kp.q_stride + lidx<N>(kp.layout, kp.q_stride, s, k3, k2, k1);
          const double nv = *u + t;
          if (!isfinite(nv)) flags |= 1u;
          *u = nv;
          continue;
        }
        if (s == kp.src_comp)  // P S^(o-1)(t0) (proj/src/predictor_common.cpp:271-283)
          t = fma(kp.src_proj[2][k3] * (kp.src_proj[1][k2] * kp.src_proj[0][k1]), kp.src_amp[o - 1], t);
        double* acc = qa + lidx<N>(kp.layout, kp.out_stride, s, k3, k2, k1);
        const double nq = fma(kp.cf[o], t, *acc);
        *acc = nq;
        Wt[i] = o == N - 1 ? nq : t;  // the last step leaves Qbar
      }
      __syncthreads();
    }
    double* sw = P;
    P = R;
    R = sw;
  }
  if (kp.vol_mode) {
    if (kp.check && flags) atomicOr(status, flags);
    return;
  }
  const double* Q = P;  // Qbar [s][k3][k2][k1]
  double* F = N >= 6 ? R : W;  // face_q staging

  // ---- favg_d = A_d Qbar (the reference's F_d(Qbar), stp_splitck.cpp:72-78) -----------------
  if (a.favg) {
    double* fo = a.favg + e * 3ll * N3 * kp.out_stride;
    for (int i = tid; i < 3 * m * N3; i += kGenThreads) {
      const int ds = i / N3, node = i - ds * N3;
      const int d = ds / m, s = ds - d * m;
      double f = 0.0;
      const int b = kp.f_ptr[3 * s + d], end = kp.f_ptr[3 * s + d + 1];
      for (int k = b; k < end; ++k) f = fma(kp.f_val[k], Q[(long long)kp.f_col[k] * N3 + node], f);
      const int k3 = node / N2, k2 = (node / N) % N, k1 = node % N;
      fo[d * (long long)N3 * kp.out_stride + lidx<N>(kp.layout, kp.out_stride, s, k3, k2, k1)] = f * kp.scale;
    }
    // padding lanes of the output rows are written as zeros (like the reference's PredictorOutput)
    if (kp.out_stride > m)
      for (int i = tid; i < 3 * N3 * (kp.out_stride - m); i += kGenThreads) {
        const int per = N3 * (kp.out_stride - m), d = i / per, r = i - d * per;
        const int node = r / (kp.out_stride - m), s = m + r % (kp.out_stride - m);
        fo[d * (long long)N3 * kp.out_stride + lidx<N>(kp.layout, kp.out_stride, s, node / N2, (node / N) % N, node % N)] = 0.0;
      }
  }
  if (kp.out_stride > m)
    for (int i = tid; i < N3 * (kp.out_stride - m); i += kGenThreads) {
      const int node = i / (kp.out_stride - m), s = m + i % (kp.out_stride - m);
      qa[lidx<N>(kp.layout, kp.out_stride, s, node / N2, (node / N) % N, node % N)] = 0.0;
    }

  // ---- faces (predictor_common.cpp:311-341): face_q of Qbar into W, face_f = A_d face_q -----
  const int FACE = N2 * m;
  if (a.face_q || a.face_f) {
    for (int i = tid; i < 6 * FACE; i += kGenThreads) {
      const int f = i / FACE, r = i - f * FACE, ab = r / m, s = r - ab * m;
      const int ia = ab / N, ib = ab - ia * N, d = f >> 1;
      const double* ph = kp.phi[f & 1];
      const double* qs = Q + (long long)s * N3;
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const int node = d == 0 ? (ia * N + ib) * N + j : d == 1 ? (ia * N + j) * N + ib : (j * N + ia) * N + ib;
        v = fma(ph[j], qs[node], v);
      }
      F[i] = v;
      if (a.face_q) a.face_q[e * 6ll * FACE + i] = v;
    }
    __syncthreads();
    if (a.face_f)
      for (int i = tid; i < 6 * FACE; i += kGenThreads) {
        const int f = i / FACE, r = i - f * FACE, ab = r / m, s = r - ab * m, d = f >> 1;
        double v = 0.0;
        const int b = kp.f_ptr[3 * s + d], end = kp.f_ptr[3 * s + d + 1];
        for (int k = b; k < end; ++k) v = fma(kp.f_val[k], F[f * FACE + ab * m + kp.f_col[k]], v);
        a.face_f[e * 6ll * FACE + i] = v * kp.scale;  // the flux of the (scaled) PDE
      }
  }
  if (kp.check && flags) atomicOr(status, flags);
}

template <int N>
size_t general_smem(int m, bool scratch) {
  const size_t n2 = N * N, n3 = n2 * N;
  return sizeof(double) * (n2 + (n2 & 1) + (N >= 6 ? 3 : 6) * (size_t)m * n2 + (scratch ? 0 : 2 * (size_t)m * n3));
}

template <int N>
cudaError_t launch_general_n(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  GenParams kp;
  for (int i = 0; i < N * N; ++i) kp.d[i] = p.basis.d[i];
  for (int j = 0; j < N; ++j) {
    kp.phi[0][j] = p.basis.face_left[j];
    kp.phi[1][j] = p.basis.face_right[j];
    for (int d = 0; d < 3; ++d) kp.src_proj[d][j] = p.src_proj[d][j];
  }
  {
    double c = a.dt;  // the reference's sequence (stp_splitck.cpp:45,64)
    kp.cf[0] = c;
    for (int o = 1; o < N; ++o) {
      c *= a.dt / (o + 1);
      kp.cf[o] = c;
    }
  }
  source_amplitudes(p, a.t_start, N, kp.src_amp);
  kp.src_comp = p.src_comp;
  kp.m = p.m;
  kp.q_stride = p.q_stride;
  kp.out_stride = p.out_stride;
  kp.layout = p.layout;
  kp.check = p.check;
  kp.scale = p.gen.scale;
  kp.t_ptr = p.gen.t_ptr;
  kp.t_col = p.gen.t_col;
  kp.t_val = p.gen.t_val;
  kp.t_nnz = p.gen.t_nnz;
  kp.f_ptr = p.gen.f_ptr;
  kp.f_col = p.gen.f_col;
  kp.f_val = p.gen.f_val;
  kp.vol_mode = a.u_next != nullptr && a.vol_r != nullptr;
  if (a.n_elem == 0) return cudaSuccess;
  if (a.n_elem > 0x7fffffffLL) return cudaErrorInvalidValue;
  int dev = 0, max_smem = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err == cudaSuccess) err = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (err != cudaSuccess) return err;
  const bool scratch = general_smem<N>(p.m, false) > (size_t)max_smem;
  size_t smem = general_smem<N>(p.m, scratch);
  if (smem > (size_t)max_smem) return cudaErrorInvalidConfiguration;
  const size_t csr = sizeof(double) * p.gen.t_nnz + sizeof(int) * (p.gen.t_nnz + 3 * p.m + 1);
  // dense C (rows padded to whole target blocks) when the matrices are mostly nonzero
  kp.m_pad = (p.m + kSB - 1) / kSB * kSB;
  kp.t_dense = p.gen.t_dense;
  const size_t dense = sizeof(double) * (3 * p.m * kp.m_pad + 2);  // + alignment slack
  // (the blocks cut the task count by kSB: only where m N^2 keeps the CTA busy -- measured: m = 21
  // at nDof 8 +46 %, m = 21 at nDof 4 and m = 12 at nDof 6 -5 %)
  kp.dense = p.gen.t_dense != nullptr && 2 * p.gen.t_nnz >= 3 * p.m * p.m && p.m * N * N >= 1024 &&
             smem + dense <= (size_t)max_smem;
  kp.csr_smem = !kp.dense && smem + csr <= (size_t)max_smem;
  if (kp.dense) smem += dense;
  else if (kp.csr_smem) smem += csr;
  err = cudaFuncSetAttribute(scratch ? stp_general_kernel<N, true> : stp_general_kernel<N, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  if (!scratch) {
    kp.scratch = nullptr;
    stp_general_kernel<N, false><<<(unsigned)a.n_elem, gen_threads<N>(), smem, stream>>>(kp, a, p.d_status);
    return cudaGetLastError();
  }
  // iterate pair in global scratch from the plan's pool, in chunks of <= kGenScratchBytes
  if (!p.gen.pool) return cudaErrorInvalidValue;
  const long long per = 2ll * p.m * N * N * N;  // doubles per element
  long long chunk = kGenScratchBytes / (per * 8);
  if (chunk < 1) chunk = 1;
  if (chunk > a.n_elem) chunk = a.n_elem;
  double* buf = nullptr;
  err = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&buf), sizeof(double) * per * chunk, p.gen.pool, stream);
  if (err != cudaSuccess) return err;
  kp.scratch = buf;
  const long long qin = (long long)N * N * N * p.q_stride, qout = (long long)N * N * N * p.out_stride;
  const long long face = 6ll * N * N * p.m;
  for (long long e0 = 0; e0 < a.n_elem && err == cudaSuccess; e0 += chunk) {
    const long long c = a.n_elem - e0 < chunk ? a.n_elem - e0 : chunk;
    BatchArgs b = a;
    b.q = a.q + e0 * qin;
    b.qavg = a.qavg ? a.qavg + e0 * qout : nullptr;
    b.favg = a.favg ? a.favg + e0 * 3 * qout : nullptr;
    b.face_q = a.face_q ? a.face_q + e0 * face : nullptr;
    b.face_f = a.face_f ? a.face_f + e0 * face : nullptr;
    if (a.u_next) b.u_next = a.u_next + e0 * qin;
    if (a.vol_r) b.vol_r = a.vol_r + e0 * qout;
    b.n_elem = c;
    stp_general_kernel<N, true><<<(unsigned)c, gen_threads<N>(), smem, stream>>>(kp, b, p.d_status);
    err = cudaGetLastError();
  }
  cudaFreeAsync(buf, stream);
  return err;
}

}  // namespace

// S^(o)(t0) of the plan's Gaussian point source for o = 0..n-1, times the plan's source scale
// (ScaledPde, proj/src/solver.cpp:147-150): the Hermite recurrence of proj/src/pde.cpp:48-59
void source_amplitudes(const LaunchPlan& p, double t, int n, double* amp) {
  for (int o = 0; o < n; ++o) {
    double v = 0.0;
    if (p.src_comp >= 0) {
      const double u = (t - p.src_center) / p.src_width;
      double hm = 0.0, h = 1.0, scale = 1.0;
      for (int k = 0; k < o; ++k) {
        const double hn = u * h - k * hm;
        hm = h;
        h = hn;
      }
      for (int k = 0; k < o; ++k) scale *= -1.0 / p.src_width;
      v = p.src_amp * scale * h * std::exp(-0.5 * u * u) * p.src_scale;
    }
    amp[o] = v;
  }
}

bool general_selected(const LaunchPlan& p) { return p.kind != ADERSTP_PDE_ELASTIC && p.gen.t_ptr != nullptr; }

cudaError_t launch_general(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  if (gdense_applicable(p, a)) return launch_gdense(p, a, stream);
  switch (p.n) {
    case 2: return launch_general_n<2>(p, a, stream);
    case 3: return launch_general_n<3>(p, a, stream);
    case 4: return launch_general_n<4>(p, a, stream);
    case 5: return launch_general_n<5>(p, a, stream);
    case 6: return launch_general_n<6>(p, a, stream);
    case 7: return launch_general_n<7>(p, a, stream);
    case 8: return launch_general_n<8>(p, a, stream);
    case 9: return launch_general_n<9>(p, a, stream);
    case 10: return launch_general_n<10>(p, a, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace aderstp
