// sm_100a kernels of the linear ADER-DG Space-Time Predictor (Cauchy-Kowalewsky recursion).
//
// Algorithm = the reference's SplitCK (proj/src/stp_splitck.cpp:13-81) + extrapolate_faces
// (proj/src/predictor_common.cpp:311-341), re-organised for the GPU:
//   * one element's state p (m x n^3 fp64) is staged in shared memory, the time-integral
//     accumulator qavg lives next to it; nothing intermediate ever goes back to HBM;
//   * thread (s, k2, k1) owns the z-column of output quantity s at (k2, k1):
//       t_s = sum_d D_d * (sum_r c_{s,d,r} p_r)        (flux applied before the derivative,
//                                                        exactly the reference's D_d * F_d(p))
//     x/y contractions read rows of p from shared memory with the thread's row of D, the
//     z contraction loads the column once and uses compile-time D (constant-bank operands);
//   * qavg += c_o * t is fused into the write-back of t; favg = F_d(qavg) and the 12 face
//     arrays are produced in the epilogue from shared memory with flat, coalesced stores.
// DESIGN.md documents the data layout, the roofline and the measured profile.
#include <cmath>
#include <cstdint>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"

namespace aderstp {

namespace {

template <int N>
struct KParams {
  double d[N * N];          // d[k*N + l] = phi_l'(x_k)   (compile-time indexed: c[] operands)
  double phi[2][N];         // phi_k(0), phi_k(1)
  double src_proj[3][N];    // phi_dim(x_src)[k] / w[k]
  double src_amp[N];        // S^(o-1)(t0) for o = 1..N-1 (point source amplitude derivatives)
  int src_comp;
  int m, q_stride, out_stride, layout, par_kind, check, n_terms;
  signed char tr[kMaxM][3][kMaxTerms];
  signed char fr[kMaxM][3][kMaxTerms];
  double tc[kMaxM][3][kMaxTerms];
  double fc[kMaxM][3][kMaxTerms];
};

// Elastic flux table (proj/src/pde.cpp:180-218), state (sxx,syy,szz,sxy,sxz,syz,u,v,w):
// F_d(q)_s = coef(s,d) * q[in(s,d)], with coef in {lambda+2mu, lambda, mu, 1/rho, 0}.
__device__ __constant__ signed char kElasticIn[9][3] = {
    {6, 7, 8}, {6, 7, 8}, {6, 7, 8}, {7, 6, 0}, {8, 0, 6}, {0, 8, 7}, {0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
// 0: lambda+2mu, 1: lambda, 2: mu, 3: 1/rho, 4: zero
__device__ __constant__ signed char kElasticCoef[9][3] = {
    {0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {2, 2, 4}, {2, 4, 2}, {4, 2, 2}, {3, 3, 3}, {3, 3, 3}, {3, 3, 3}};

template <int N>
constexpr int row_stride() {
  return (N % 2 == 0) ? N + 1 : N;  // odd row stride: conflict-free broadcast rows
}

// Index of (s, k3, k2, k1) inside one element's shared-memory tensor.
template <int N>
__device__ __forceinline__ int sidx(int s, int k3, int k2, int k1) {
  constexpr int RS = row_stride<N>(), PL = N * RS, VS = N * PL;
  return s * VS + k3 * PL + k2 * RS + k1;
}

template <int N>
constexpr int elem_smem_doubles(int m) {
  return 2 * m * N * N * row_stride<N>();  // p and the qavg accumulator
}

// Element material -> (lambda+2mu, lambda, mu, 1/rho) with the reference's validity check
// (proj/src/pde.cpp:175-176).
__device__ __forceinline__ bool elastic_coefs(const double* par, int par_kind, double* c4) {
  const double a = par[0], b = par[1], c = par[2];
  double lam, mu, rho;
  if (par_kind == ADERSTP_PAR_RHO_CP_CS) {
    rho = a;
    mu = __dmul_rn(__dmul_rn(a, c), c);
    lam = __dsub_rn(__dmul_rn(__dmul_rn(a, b), b), __dmul_rn(2.0, mu));
  } else {
    lam = a;
    mu = b;
    rho = c;
  }
  c4[0] = lam + 2.0 * mu;
  c4[1] = lam;
  c4[2] = mu;
  c4[3] = 1.0 / rho;
  return (rho > 0.0) && (mu >= 0.0) && (lam + 2.0 * mu > 0.0);
}

// c4 = (lambda+2mu, lambda, mu, 1/rho); index 4 = zero.  Selects keep c4 in registers.
__device__ __forceinline__ double pick(const double* c4, int idx) {
  return idx == 0 ? c4[0] : idx == 1 ? c4[1] : idx == 2 ? c4[2] : idx == 3 ? c4[3] : 0.0;
}

// ------------------------------------------------------------------------------------------
// The STP kernel.  ELASTIC: per-element terms from the material (one term per (s,d));
// otherwise a plan-wide table of up to n_terms terms per (s,d) plus an optional point source.
// Threads per element TPE = m * N^2; EPB elements per block.
// Elements per block of the elastic kernel: ~300-900 threads per block.
template <int N>
constexpr int elastic_epb() {
  return N <= 2 ? 8 : N == 3 ? 4 : N <= 5 ? 2 : 1;
}
template <int N, bool ELASTIC>
constexpr int max_threads() {
  return ELASTIC ? elastic_epb<N>() * 9 * N * N : 1024;
}

// MT: the block-size bound the kernel is compiled for (registers per thread = 64 K / MT).  The
// table kernel exists twice per order: MT = 1024 (any m) and MT = 9 N^2 rounded up to a warp
// (m <= 9: one element of the elastic size per block, up to 112 registers, no spills).
template <int N>
constexpr int table_small_threads() { return ((9 * N * N + 31) / 32) * 32; }

template <int N, bool ELASTIC, int MT = max_threads<N, ELASTIC>()>
__global__ void __launch_bounds__(MT) stp_kernel(KParams<N> kp, BatchArgs a, int epb, unsigned int* status) {
  extern __shared__ double smem[];
  constexpr int RS = row_stride<N>();
  constexpr int DS = N + 1;  // padded row stride of D in shared memory
  const int m = ELASTIC ? 9 : kp.m;
  const int tpe = m * N * N;
  const int es = elem_smem_doubles<N>(m);

  double* Ds = smem;  // N x (N+1)
  const int tid = threadIdx.x;
  for (int i = tid; i < N * N; i += blockDim.x) Ds[(i / N) * DS + (i % N)] = kp.d[i];

  const int el = tid / tpe;
  const int r = tid - el * tpe;
  const int s = r / (N * N);
  const int col = r - s * (N * N);
  const int k2 = col / N, k1 = col - k2 * N;
  const long long e = (long long)blockIdx.x * epb + el;
  const bool live = (el < epb) && (e < a.n_elem);
  double* P = smem + N * DS + (N * DS) % 2 + el * es;  // keep 16-byte alignment
  double* QA = P + es / 2;
  unsigned int flags = 0;

  // ---- per-thread terms for output quantity s ----------------------------------------
  // Terms of output quantity s: elastic -- the one term per (s, d) in registers; table PDEs in
  // the small-block variant (MT < 900) read theirs from the parameter bank at the point of use
  // (s is warp-uniform for N >= 6), which keeps 36 registers free; otherwise in registers.
  constexpr int K = ELASTIC ? 1 : kMaxTerms;
  constexpr bool TP = !ELASTIC && MT < 900;
  constexpr int KR = TP ? 1 : K;
  int in[3][KR];
  double cf[3][KR];
  double dt = a.dt;
  if (live) {
    if (ELASTIC) {
      double c4[4];
      if (!elastic_coefs(a.par + 3 * e, kp.par_kind, c4)) flags |= 2u;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        in[d][0] = kElasticIn[s][d];
        cf[d][0] = pick(c4, kElasticCoef[s][d]);
      }
    } else if (!TP) {
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          in[d][k] = kp.tr[s][d][k];
          cf[d][k] = kp.tc[s][d][k];
        }
    }
  } else {
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        in[d][k] = 0;
        cf[d][k] = 0.0;
      }
  }
  auto term_in = [&](int d, int k) -> int { return TP ? kp.tr[s][d][k] : in[d][TP ? 0 : k]; };
  auto term_cf = [&](int d, int k) -> double { return TP ? kp.tc[s][d][k] : cf[d][TP ? 0 : k]; };

  // ---- stage q (coalesced flat loop over this element's input region) ----------------
  if (el < epb && e < a.n_elem) {
    const int qs = kp.q_stride;
    const int vol_in = N * N * N * qs;
    const double* qe = a.q + e * (long long)vol_in;
    for (int i = r; i < vol_in; i += tpe) {
      int k3, k2i, k1i, si;
      if (kp.layout == ADERSTP_LAYOUT_AOSOA) {  // [k3][k2][s][k1]
        k1i = i % N;
        int t = i / N;
        si = t % qs;
        t /= qs;
        k2i = t % N;
        k3 = t / N;
      } else {  // [k3][k2][k1][s]
        si = i % qs;
        int t = i / qs;
        k1i = t % N;
        t /= N;
        k2i = t % N;
        k3 = t / N;
      }
      if (si < m) {
        const double v = __ldcs(qe + i);
        if (kp.check && !isfinite(v)) flags |= 1u;
        const int j = sidx<N>(si, k3, k2i, k1i);
        P[j] = v;
        QA[j] = dt * v;
      }
    }
  }
  __syncthreads();

  // ---- Cauchy-Kowalewsky recursion (stp_splitck.cpp:46-70) ---------------------------
  double coeff = dt;
#pragma unroll 1
  for (int o = 1; o < N; ++o) {
    double t[N];
#pragma unroll
    for (int k3 = 0; k3 < N; ++k3) t[k3] = 0.0;
    if (live) {
      // x: t[k3] += sum_l D[k1][l] * f(k3, k2, l)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!ELASTIC && k >= kp.n_terms) break;
        const double* px = P + sidx<N>(term_in(0, k), 0, k2, 0);
        const double c = term_cf(0, k);
#pragma unroll
        for (int l = 0; l < N; ++l) {
          const double cd = c * Ds[k1 * DS + l];
#pragma unroll
          for (int k3 = 0; k3 < N; ++k3) t[k3] = fma(cd, px[k3 * N * RS + l], t[k3]);
        }
      }
      // y: t[k3] += sum_l D[k2][l] * f(k3, l, k1)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!ELASTIC && k >= kp.n_terms) break;
        const double* py = P + sidx<N>(term_in(1, k), 0, 0, k1);
        const double c = term_cf(1, k);
#pragma unroll
        for (int l = 0; l < N; ++l) {
          const double cd = c * Ds[k2 * DS + l];
#pragma unroll
          for (int k3 = 0; k3 < N; ++k3) t[k3] = fma(cd, py[k3 * N * RS + l * RS], t[k3]);
        }
      }
      // z: t[k3] += c * sum_l D[k3][l] * f(l, k2, k1)   (D from the constant bank)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (!ELASTIC && k >= kp.n_terms) break;
        const double* pz = P + sidx<N>(term_in(2, k), 0, k2, k1);
        double colv[N];
#pragma unroll
        for (int l = 0; l < N; ++l) colv[l] = pz[l * N * RS];
        const double c = term_cf(2, k);
#pragma unroll
        for (int k3 = 0; k3 < N; ++k3) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = fma(kp.d[k3 * N + l], colv[l], acc);
          t[k3] = fma(c, acc, t[k3]);
        }
      }
      // point source: t_s += P[k] * S^(o-1)(t0)   (predictor_common.cpp:271-283)
      if (s == kp.src_comp) {
        const double amp = kp.src_amp[o - 1];
        const double pyx = kp.src_proj[1][k2] * kp.src_proj[0][k1];
#pragma unroll
        for (int k3 = 0; k3 < N; ++k3) t[k3] = fma(kp.src_proj[2][k3] * pyx, amp, t[k3]);
      }
    }
    coeff *= dt / (o + 1);  // dt^(o+1)/(o+1)!
    __syncthreads();
    if (live) {
#pragma unroll
      for (int k3 = 0; k3 < N; ++k3) {
        const int j = sidx<N>(s, k3, k2, k1);
        P[j] = t[k3];
        QA[j] = fma(coeff, t[k3], QA[j]);
      }
    }
    __syncthreads();
  }

  // ---- epilogue: qavg, favg = F_d(qavg), faces (predictor_common.cpp:311-341) ---------
  if (el < epb && e < a.n_elem) {
    const int os = kp.out_stride;
    const int vol_out = N * N * N * os;
    if (a.qavg) {
      double* out = a.qavg + e * (long long)vol_out;
      for (int i = r; i < vol_out; i += tpe) {
        int k3, k2i, k1i, si;
        if (kp.layout == ADERSTP_LAYOUT_AOSOA) {
          k1i = i % N;
          int tq = i / N;
          si = tq % os;
          tq /= os;
          k2i = tq % N;
          k3 = tq / N;
        } else {
          si = i % os;
          int tq = i / os;
          k1i = tq % N;
          tq /= N;
          k2i = tq % N;
          k3 = tq / N;
        }
        __stcs(out + i, si < m ? QA[sidx<N>(si, k3, k2i, k1i)] : 0.0);
      }
    }
    // flux coefficients for favg / face_f (elastic: the same table as t; table PDEs: A_d)
    double c4[4] = {0.0, 0.0, 0.0, 0.0};
    if (ELASTIC) elastic_coefs(a.par + 3 * e, kp.par_kind, c4);
    if (a.favg) {
      double* out = a.favg + e * 3LL * vol_out;
      for (int i = r; i < 3 * vol_out; i += tpe) {
        const int d = i / vol_out;
        const int ii = i - d * vol_out;
        int k3, k2i, k1i, si;
        if (kp.layout == ADERSTP_LAYOUT_AOSOA) {
          k1i = ii % N;
          int tq = ii / N;
          si = tq % os;
          tq /= os;
          k2i = tq % N;
          k3 = tq / N;
        } else {
          si = ii % os;
          int tq = ii / os;
          k1i = tq % N;
          tq /= N;
          k2i = tq % N;
          k3 = tq / N;
        }
        double v = 0.0;
        if (si < m) {
          if (ELASTIC) {
            v = pick(c4, kElasticCoef[si][d]) * QA[sidx<N>(kElasticIn[si][d], k3, k2i, k1i)];
          } else {
            for (int k = 0; k < kp.n_terms; ++k)
              v += kp.fc[si][d][k] * QA[sidx<N>(kp.fr[si][d][k], k3, k2i, k1i)];
          }
        }
        __stcs(out + i, v);
      }
    }
    if (a.face_q || a.face_f) {
      const int fvol = N * N * m;
      double* oq = a.face_q ? a.face_q + e * 6LL * fvol : nullptr;
      double* of = a.face_f ? a.face_f + e * 6LL * fvol : nullptr;
      for (int i = r; i < 6 * fvol; i += tpe) {
        const int f = i / fvol;
        int rem = i - f * fvol;
        const int si = rem % m;
        rem /= m;
        const int bb = rem % N, aa = rem / N;
        const int d = f >> 1, side = f & 1;
        // line start and stride along the normal dim d
        int base, stride;
        if (d == 0) {
          base = sidx<N>(0, aa, bb, 0);
          stride = 1;
        } else if (d == 1) {
          base = sidx<N>(0, aa, 0, bb);
          stride = RS;
        } else {
          base = sidx<N>(0, 0, aa, bb);
          stride = N * RS;
        }
        constexpr int VS = N * N * RS;
        double vq = 0.0;
        const double* lq = QA + base + si * VS;
#pragma unroll
        for (int j = 0; j < N; ++j) vq = fma(kp.phi[side][j], lq[j * stride], vq);
        if (oq) __stcs(oq + i, vq);
        if (of) {
          double vf = 0.0;
          if (ELASTIC) {
            const double* lf = QA + base + kElasticIn[si][d] * VS;
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) acc = fma(kp.phi[side][j], lf[j * stride], acc);
            vf = pick(c4, kElasticCoef[si][d]) * acc;
          } else {
            for (int k = 0; k < kp.n_terms; ++k) {
              const double* lf = QA + base + kp.fr[si][d][k] * VS;
              double acc = 0.0;
#pragma unroll
              for (int j = 0; j < N; ++j) acc = fma(kp.phi[side][j], lf[j * stride], acc);
              vf = fma(kp.fc[si][d][k], acc, vf);
            }
          }
          __stcs(of + i, vf);
        }
      }
    }
  }
  if (kp.check && flags) atomicOr(status, flags);
}

template <int N>
void fill_params(const LaunchPlan& p, const BatchArgs& a, KParams<N>& kp) {
  for (int i = 0; i < N * N; ++i) kp.d[i] = p.basis.d[i];
  for (int j = 0; j < N; ++j) {
    kp.phi[0][j] = p.basis.face_left[j];
    kp.phi[1][j] = p.basis.face_right[j];
  }
  kp.src_comp = p.src_comp;
  for (int d = 0; d < 3; ++d)
    for (int j = 0; j < N; ++j) kp.src_proj[d][j] = p.src_proj[d][j];
  // S^(o-1)(t0) for o = 1..N-1: Gaussian derivatives via the Hermite recurrence
  // (proj/src/pde.cpp:48-59), evaluated at this launch's t_start, times the source scale
  source_amplitudes(p, a.t_start, N, kp.src_amp);
  kp.m = p.m;
  kp.q_stride = p.q_stride;
  kp.out_stride = p.out_stride;
  kp.layout = p.layout;
  kp.par_kind = p.par_kind;
  kp.check = p.check;
  kp.n_terms = p.n_terms;
  for (int s = 0; s < kMaxM; ++s)
    for (int d = 0; d < 3; ++d)
      for (int k = 0; k < kMaxTerms; ++k) {
        kp.tr[s][d][k] = p.tr[s][d][k];
        kp.tc[s][d][k] = p.tc[s][d][k];
        kp.fr[s][d][k] = p.fr[s][d][k];
        kp.fc[s][d][k] = p.fc[s][d][k];
      }
}

template <int N, bool ELASTIC>
cudaError_t launch_order(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  KParams<N> kp;
  fill_params<N>(p, a, kp);
  const int m = p.m;
  const int tpe = m * N * N;
  constexpr int SMALL = table_small_threads<N>();
  const bool small = !ELASTIC && tpe <= SMALL;
  int epb = ELASTIC ? elastic_epb<N>() : (small ? SMALL : 1024) / tpe;
  if (epb < 1) return cudaErrorInvalidConfiguration;
  if (epb > 8) epb = 8;
  const size_t smem =
      sizeof(double) * (N * (N + 1) + (N * (N + 1)) % 2 + (size_t)epb * elem_smem_doubles<N>(m));
  auto kern = small ? stp_kernel<N, ELASTIC, (ELASTIC ? max_threads<N, ELASTIC>() : SMALL)> : stp_kernel<N, ELASTIC>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const long long blocks = (a.n_elem + epb - 1) / epb;
  if (blocks == 0) return cudaSuccess;
  kern<<<(unsigned)blocks, epb * tpe, smem, stream>>>(kp, a, epb, p.d_status);
  return cudaGetLastError();
}

template <bool ELASTIC>
cudaError_t dispatch(const LaunchPlan& p, const BatchArgs& a, cudaStream_t st) {
  switch (p.n) {
    case 2: return launch_order<2, ELASTIC>(p, a, st);
    case 3: return launch_order<3, ELASTIC>(p, a, st);
    case 4: return launch_order<4, ELASTIC>(p, a, st);
    case 5: return launch_order<5, ELASTIC>(p, a, st);
    case 6: return launch_order<6, ELASTIC>(p, a, st);
    case 7: return launch_order<7, ELASTIC>(p, a, st);
    case 8: return launch_order<8, ELASTIC>(p, a, st);
    case 9: return launch_order<9, ELASTIC>(p, a, st);
    case 10: return launch_order<10, ELASTIC>(p, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool kernel_available(int n) { return n >= kMinOrder && n <= kMaxOrder; }

namespace {
bool use_dmma8(const LaunchPlan& p, const BatchArgs& a) {
  // the tensor-core kernel moves 16-byte vectors: every batch pointer must be 16-byte aligned
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  const bool aligned = al16(a.q) && al16(a.qavg) && al16(a.favg) && al16(a.face_q) && al16(a.face_f) &&
                       al16(a.u_next);
  return !p.force_generic && !p.no_dmma8 && aligned && dmma8_applicable(p);
}
}  // namespace

namespace {
bool use_dmmap(const LaunchPlan& p, const BatchArgs& a) {
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  const bool aligned = al16(a.q) && al16(a.qavg) && al16(a.favg) && al16(a.face_q) && al16(a.face_f) &&
                       al16(a.u_next);
  return !p.force_generic && !p.no_dmmap && aligned && dmmap_applicable(p);
}
bool use_bip(const LaunchPlan& p, const BatchArgs& a) {
  return !p.force_generic && pass_applicable(p) && bip_selected(p, a);
}
}  // namespace

bool fused_supported(const LaunchPlan& p, const BatchArgs& a) {
  return use_dmma8(p, a) || use_dmmap(p, a) || use_bip(p, a);
}

cudaError_t launch_stp(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  const bool aligned = al16(a.q) && al16(a.qavg) && al16(a.favg) && al16(a.face_q) && al16(a.face_f);
  if (general_selected(p)) return launch_general(p, a, stream);
  if (use_dmma8(p, a)) return launch_dmma8(p, a, stream);
  if (dmma8_table_applicable(p, a)) return launch_dmma8_table(p, a, stream);
  if (dmmat_applicable(p, a)) return launch_dmmat(p, a, stream);
  if (tlp_applicable(p, a)) return launch_tlp(p, a, stream);
  if (a.u_next && use_dmmap(p, a)) return launch_dmmap(p, a, stream);
  if (a.u_next && use_bip(p, a)) return launch_pass(p, a, stream);
  if (a.u_next) return cudaErrorInvalidValue;  // the fused mode exists only where fused_supported()
  if (wpe_applicable(p, a)) return launch_wpe(p, a, stream);
  if (!p.force_generic && !p.no_dmmap && aligned && dmmap_applicable(p)) return launch_dmmap(p, a, stream);
  if (!p.force_generic && pass_applicable(p)) return launch_pass(p, a, stream);
  if (p.kind == ADERSTP_PDE_ELASTIC) return dispatch<true>(p, a, stream);
  return dispatch<false>(p, a, stream);
}

// ------------------------------------------------------------------------------------------
// Layout conversion AoS <-> AoSoA (proj/src/layout.cpp:168-194), one thread per destination
// entry; destination padding slots are written as zero.
__global__ void convert_kernel(int n, int m, long long total, int src_layout, int src_stride,
                               const double* __restrict__ src, int dst_layout, int dst_stride,
                               double* __restrict__ dst) {
  const long long per = (long long)n * n * n * dst_stride;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = i / per;
    int rem = (int)(i - e * per);
    int k3, k2, k1, s;
    if (dst_layout == ADERSTP_LAYOUT_AOSOA) {
      k1 = rem % n;
      rem /= n;
      s = rem % dst_stride;
      rem /= dst_stride;
      k2 = rem % n;
      k3 = rem / n;
    } else {
      s = rem % dst_stride;
      rem /= dst_stride;
      k1 = rem % n;
      rem /= n;
      k2 = rem % n;
      k3 = rem / n;
    }
    double v = 0.0;
    if (s < m) {
      const long long sper = (long long)n * n * n * src_stride;
      const long long j = src_layout == ADERSTP_LAYOUT_AOSOA
                              ? (((long long)k3 * n + k2) * src_stride + s) * n + k1
                              : (((long long)k3 * n + k2) * n + k1) * src_stride + s;
      v = src[e * sper + j];
    }
    dst[i] = v;
  }
}

// The same conversion by (k3, k2) rows: a row is n x src_stride doubles in one layout and
// n x dst_stride in the other, both contiguous, so a block stages ROWS rows in shared memory with
// coalesced loads and writes them back transposed with coalesced stores.
constexpr int kConvRows = 16;
__global__ void __launch_bounds__(256) convert_rows_kernel(int n, int m, long long rows, int src_layout, int src_stride,
                                                          const double* __restrict__ src, int dst_layout,
                                                          int dst_stride, double* __restrict__ dst) {
  extern __shared__ double tile[];  // kConvRows x n x src_stride
  const int srow = n * src_stride, drow = n * dst_stride;
  for (long long r0 = (long long)blockIdx.x * kConvRows; r0 < rows; r0 += (long long)gridDim.x * kConvRows) {
    const int nr = (int)(rows - r0 < kConvRows ? rows - r0 : kConvRows);
    const double* s0 = src + r0 * srow;
    for (int i = threadIdx.x; i < nr * srow; i += blockDim.x) tile[i] = s0[i];
    __syncthreads();
    double* d0 = dst + r0 * drow;
    for (int i = threadIdx.x; i < nr * drow; i += blockDim.x) {
      const int r = i / drow, j = i - r * drow;
      int s, k1;
      if (dst_layout == ADERSTP_LAYOUT_AOSOA) {
        s = j / n;
        k1 = j - s * n;
      } else {
        k1 = j / dst_stride;
        s = j - k1 * dst_stride;
      }
      double v = 0.0;
      if (s < m) v = tile[r * srow + (src_layout == ADERSTP_LAYOUT_AOSOA ? s * n + k1 : k1 * src_stride + s)];
      d0[i] = v;
    }
    __syncthreads();
  }
}

// Fast path of the conversion for the drop-in pair: the reference's AoS rows [k1][s < 16] (m = 9,
// padding slots 9..15) <-> compact AoSoA rows [s < 9][k1], even n.  16-byte loads and stores,
// compile-time indexing, the AoS padding slots neither read (AoS -> AoSoA: 80 of the 128 bytes of
// a node) nor staged (AoSoA -> AoS: written as zeros); the tile rows are padded (stride n + 1 per
// quantity) so that both sides of the transpose are bank-conflict free.
template <int N, bool TO_AOSOA>
__global__ void __launch_bounds__(256) convert_rows16_kernel(long long rows, const double* __restrict__ src,
                                                             double* __restrict__ dst) {
  constexpr int R = kConvRows, M = 9, TS = N + 1, TROW = M * TS;  // tile: [r][s][k1 (+1 pad)]
  constexpr int AROW = N * 16, CROW = N * M;                        // AoS / AoSoA row lengths
  __shared__ double tile[R * TROW];
  for (long long r0 = (long long)blockIdx.x * R; r0 < rows; r0 += (long long)gridDim.x * R) {
    const int nr = (int)(rows - r0 < R ? rows - r0 : R);
    if (TO_AOSOA) {
      // AoS source: per node k1 the pairs (s, s + 1), s = 0, 2, 4, 6, 8 (slot 9 is padding)
      const double* s0 = src + r0 * AROW;
      for (int i = threadIdx.x; i < nr * N * 5; i += blockDim.x) {
        const int r = i / (N * 5), j = i - r * (N * 5), k1 = j / 5, sp = 2 * (j - k1 * 5);
        const double2 v = *reinterpret_cast<const double2*>(s0 + r * AROW + k1 * 16 + sp);
        tile[r * TROW + sp * TS + k1] = v.x;
        if (sp + 1 < M) tile[r * TROW + (sp + 1) * TS + k1] = v.y;
      }
      __syncthreads();
      double* d0 = dst + r0 * CROW;
      for (int i = threadIdx.x; i < nr * CROW / 2; i += blockDim.x) {
        const int r = i / (CROW / 2), j = 2 * (i - r * (CROW / 2)), sq = j / N, k1 = j - sq * N;
        const double* t = tile + r * TROW + sq * TS + k1;
        *reinterpret_cast<double2*>(d0 + r * CROW + j) = make_double2(t[0], t[1]);
      }
    } else {
      const double* s0 = src + r0 * CROW;
      for (int i = threadIdx.x; i < nr * CROW / 2; i += blockDim.x) {
        const int r = i / (CROW / 2), j = 2 * (i - r * (CROW / 2)), sq = j / N, k1 = j - sq * N;
        const double2 v = *reinterpret_cast<const double2*>(s0 + r * CROW + j);
        tile[r * TROW + sq * TS + k1] = v.x;
        tile[r * TROW + sq * TS + k1 + 1] = v.y;
      }
      __syncthreads();
      double* d0 = dst + r0 * AROW;
      for (int i = threadIdx.x; i < nr * AROW / 2; i += blockDim.x) {
        const int r = i / (AROW / 2), j = i - r * (AROW / 2), k1 = j >> 3, sp = 2 * (j & 7);
        const double* t = tile + r * TROW + k1;
        const double a = sp < M ? t[sp * TS] : 0.0, b = sp + 1 < M ? t[(sp + 1) * TS] : 0.0;
        *reinterpret_cast<double2*>(d0 + r * AROW + 16 * k1 + sp) = make_double2(a, b);
      }
    }
    __syncthreads();
  }
}

template <int N>
cudaError_t launch_convert16(bool to_aosoa, long long rows, const double* src, double* dst, cudaStream_t stream) {
  long long blocks = (rows + kConvRows - 1) / kConvRows;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  if (to_aosoa)
    convert_rows16_kernel<N, true><<<(unsigned)blocks, 256, 0, stream>>>(rows, src, dst);
  else
    convert_rows16_kernel<N, false><<<(unsigned)blocks, 256, 0, stream>>>(rows, src, dst);
  return cudaGetLastError();
}

cudaError_t launch_convert(int n, int m, long long n_elem, int src_layout, int src_stride,
                           const double* src, int dst_layout, int dst_stride, double* dst,
                           cudaStream_t stream) {
  const long long total = n_elem * n * n * n * (long long)dst_stride;
  if (total == 0) return cudaSuccess;
  if (src_layout != dst_layout) {  // AoS <-> AoSoA: row transposes through shared memory
    const long long rows = n_elem * n * n;
    const bool al16 = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    const bool pair16 = m == 9 && al16 && n % 2 == 0 &&
                        ((src_layout == ADERSTP_LAYOUT_AOS && src_stride == 16 && dst_stride == 9) ||
                         (dst_layout == ADERSTP_LAYOUT_AOS && dst_stride == 16 && src_stride == 9));
    if (pair16) {
      const bool to_aosoa = dst_layout == ADERSTP_LAYOUT_AOSOA;
      switch (n) {
        case 2: return launch_convert16<2>(to_aosoa, rows, src, dst, stream);
        case 4: return launch_convert16<4>(to_aosoa, rows, src, dst, stream);
        case 6: return launch_convert16<6>(to_aosoa, rows, src, dst, stream);
        case 8: return launch_convert16<8>(to_aosoa, rows, src, dst, stream);
        case 10: return launch_convert16<10>(to_aosoa, rows, src, dst, stream);
      }
    }
    long long blocks = (rows + kConvRows - 1) / kConvRows;
    if (blocks > 148LL * 32) blocks = 148LL * 32;
    const size_t smem = sizeof(double) * kConvRows * n * src_stride;
    cudaError_t err = cudaSuccess;
    if (smem > 48 * 1024)
      err = cudaFuncSetAttribute(convert_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    convert_rows_kernel<<<(unsigned)blocks, 256, smem, stream>>>(n, m, rows, src_layout, src_stride, src, dst_layout,
                                                                 dst_stride, dst);
    return cudaGetLastError();
  }
  const int threads = 256;
  long long blocks = (total + threads - 1) / threads;
  if (blocks > 148LL * 64) blocks = 148LL * 64;
  convert_kernel<<<(unsigned)blocks, threads, 0, stream>>>(n, m, total, src_layout, src_stride,
                                                           src, dst_layout, dst_stride, dst);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Seeded synthetic inputs: the whole batch is one SplitMix64(seed)
// stream (proj/include/ader/util.hpp:72-90) read by random access, output k being
// mix(seed + (k+1)*gamma).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t sm_at(uint64_t seed, uint64_t k) {
  return mix64(seed + (k + 1) * 0x9e3779b97f4a7c15ull);
}
__device__ __forceinline__ double u01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
__device__ __forceinline__ double uab(uint64_t x, double a, double b) {
  return __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), u01(x)));
}

struct GenParams {
  double nodes[kMaxOrder];
  double wa[9][3], wk[9][3][3], wp[9][3];
};

__global__ void generate_kernel(int dist, uint64_t seed, int n, long long e0, long long n_elem,
                                int grid, int layout, int q_stride, GenParams gp,
                                double* __restrict__ q, double* __restrict__ par) {
  const int vol = n * n * n * 9;
  const long long total = n_elem * (long long)vol;
  const double two_pi = 6.283185307179586476925286766559;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total + n_elem;
       i += (long long)gridDim.x * blockDim.x) {
    if (i >= total) {  // one thread per element: material (rho, cp, cs)
      const long long le = i - total;
      const long long e = e0 + le;
      uint64_t mb;
      if (dist == 0) mb = (uint64_t)e * (uint64_t)(vol + 3) + vol;
      else if (dist == 1) mb = (uint64_t)e * (uint64_t)(2 * vol + 3) + 2 * vol;
      else mb = 135 + 3 * (uint64_t)e;
      if (par) {
        par[3 * le + 0] = uab(sm_at(seed, mb + 0), 2.0, 3.0);
        par[3 * le + 1] = uab(sm_at(seed, mb + 1), 4.0, 6.0);
        par[3 * le + 2] = uab(sm_at(seed, mb + 2), 2.0, 3.5);
      }
      continue;
    }
    if (!q) continue;
    const long long le = i / vol;
    const int k = (int)(i - le * vol);  // canonical (k3,k2,k1,s)
    const long long e = e0 + le;
    const int s = k % 9, node = k / 9;
    const int k1 = node % n, k2 = (node / n) % n, k3 = node / (n * n);
    double v;
    if (dist == 0) {
      const uint64_t base = (uint64_t)e * (uint64_t)(vol + 3);
      v = 2.0 * u01(sm_at(seed, base + k)) - 1.0;
    } else if (dist == 1) {
      const uint64_t base = (uint64_t)e * (uint64_t)(2 * vol + 3);
      const double a1 = ((double)(sm_at(seed, base + 2 * k) >> 11) + 1.0) * 0x1.0p-53;
      const double a2 = u01(sm_at(seed, base + 2 * k + 1));
      v = sqrt(-2.0 * log(a1)) * cos(two_pi * a2);
    } else {
      const long long ex = e % grid, ey = (e / grid) % grid, ez = e / ((long long)grid * grid);
      const double x = ex + gp.nodes[k1], y = ey + gp.nodes[k2], z = ez + gp.nodes[k3];
      v = 0.0;
      for (int j = 0; j < 3; ++j)
        v += gp.wa[s][j] *
             sin(two_pi * (gp.wk[s][j][0] * x + gp.wk[s][j][1] * y + gp.wk[s][j][2] * z) / grid +
                 gp.wp[s][j]);
    }
    const long long dst = layout == ADERSTP_LAYOUT_AOSOA
                              ? ((((long long)k3 * n + k2) * q_stride + s) * n + k1)
                              : ((((long long)k3 * n + k2) * n + k1) * q_stride + s);
    q[le * (long long)(n * n * n * q_stride) + dst] = v;
  }
}

cudaError_t launch_generate(int dist, uint64_t seed, int n, long long e0, long long n_elem,
                            int grid, int layout, int q_stride, const HostBasis& basis,
                            double* q, double* par, cudaStream_t stream) {
  GenParams gp;
  for (int i = 0; i < n; ++i) gp.nodes[i] = basis.nodes[i];
  if (dist == 2) {
    auto hmix = [](uint64_t z) {
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      return z ^ (z >> 31);
    };
    auto at = [&](uint64_t k) { return hmix(seed + (k + 1) * 0x9e3779b97f4a7c15ull); };
    auto hu01 = [](uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; };
    uint64_t g = 0;
    for (int s = 0; s < 9; ++s)
      for (int j = 0; j < 3; ++j) {
        gp.wa[s][j] = 0.5 + (1.0 - 0.5) * hu01(at(g++));
        for (int c = 0; c < 3; ++c) gp.wk[s][j][c] = (double)((int)(at(g++) % 7) - 3);
        gp.wp[s][j] = 2.0 * 3.14159265358979323846 * hu01(at(g++));
      }
  }
  // q slots >= 9 (e.g. the nVar+nPar=12 AoSoA layout) are zero-filled by the caller
  const long long total = n_elem * (long long)n * n * n * 9 + n_elem;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  long long blocks = (total + threads - 1) / threads;
  if (blocks > 148LL * 128) blocks = 148LL * 128;
  generate_kernel<<<(unsigned)blocks, threads, 0, stream>>>(dist, seed, n, e0, n_elem, grid, layout,
                                                            q_stride, gp, q, par);
  return cudaGetLastError();
}

}  // namespace aderstp
