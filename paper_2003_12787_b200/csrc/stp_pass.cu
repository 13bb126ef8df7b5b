// Line-pass elastic STP kernel for every order 2..10 (the nDof = 8 headline order has its own
// tensor-core kernel, stp_dmma8.cu).
//
// One CK step t = sum_d D_d * F_d(p) (proj/src/stp_splitck.cpp:46-70) is split into three passes,
// one per direction d.  In pass d every thread owns whole lines along d, so the 1-D contraction
// reads each line once and uses D with compile-time indices (uniform constant-cache operands):
//   pass x: task (source field f, x-line (k3,k2)),  pass y: (f, y-line (k3,k1)),
//   pass z: (f, z-line (k2,k1)).
// For the elastic flux (proj/src/pde.cpp:180-218) each direction has exactly six source fields,
// and every output quantity receives at most one of them per direction, so a task computes
// D_d f once and writes (pass x) or accumulates (passes y, z) coef * D_d f into the line of each
// target quantity without races:
//   d = x: u -> sxx(L), syy(lam), szz(lam); v -> sxy(mu); w -> sxz(mu); sxx,sxy,sxz -> u,v,w (1/rho)
//   d = y: v -> sxx(lam), syy(L), szz(lam); u -> sxy(mu); w -> syz(mu); sxy,syy,syz -> u,v,w
//   d = z: w -> sxx(lam), syy(lam), szz(L); u -> sxz(mu); v -> syz(mu); sxz,syz,szz -> u,v,w
// The Gauss-Legendre derivative matrix is skew-centrosymmetric (D[n-1-k][n-1-l] = -D[k][l]), so
// each line contraction is done in even/odd form: e = p_l + p_{n-1-l}, o = p_l - p_{n-1-l},
// alpha = A e, beta = B o, out_k = alpha_k + beta_k, out_{n-1-k} = beta_k - alpha_k
// (A, B = half-sums / half-differences of D's columns): n^2/2 FMAs per line instead of n^2.
// The next iterate accumulates in a second shared buffer T (one barrier per pass), qavg lives
// in registers (flat ownership in output order, so its stores are coalesced), and the epilogue
// writes favg = F_d(qavg) and the 12 face arrays with flat coalesced stores.
#include <cstdint>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"
#include "tmem.cuh"

// Even/odd derivative operator per order (uploaded once per device at plan creation), rows
// padded to 6 doubles so they load as 16-byte pairs: [A: h x 6][B: h x 6][M: 6], h = n/2,
// stored at offset order*80.
extern "C" {
__constant__ __align__(16) double aderstp_kEO[11 * 80];
#ifdef ADERSTP_EXPT_TIMING
__device__ long long aderstp_dbg_clock[4096 * 8];
int aderstp_dbg_clock_copy(long long* host, int count) {
  return (int)cudaMemcpyFromSymbol(host, aderstp_dbg_clock, sizeof(long long) * count);
}
#define TMB(i) if (threadIdx.x == 0 && blockIdx.x < 4096) aderstp_dbg_clock[blockIdx.x * 8 + (i)] = clock64()
#else
#define TMB(i)
#endif
}

namespace aderstp {

namespace {

constexpr int NVE = 9;

// pass tables: for pass d, source slot k: field, number of targets, targets, coefficient index
// (0: lambda+2mu, 1: lambda, 2: mu, 3: 1/rho)
struct PassSlot {
  int8_t src, nt, tgt[3], coef[3];
};
__constant__ PassSlot kPass[3][6] = {
    {{6, 3, {0, 1, 2}, {0, 1, 1}}, {7, 1, {3}, {2}}, {8, 1, {4}, {2}}, {0, 1, {6}, {3}}, {3, 1, {7}, {3}}, {4, 1, {8}, {3}}},
    {{7, 3, {0, 1, 2}, {1, 0, 1}}, {6, 1, {3}, {2}}, {8, 1, {5}, {2}}, {3, 1, {6}, {3}}, {1, 1, {7}, {3}}, {5, 1, {8}, {3}}},
    {{8, 3, {0, 1, 2}, {1, 1, 0}}, {6, 1, {4}, {2}}, {7, 1, {5}, {2}}, {4, 1, {6}, {3}}, {5, 1, {7}, {3}}, {2, 1, {8}, {3}}}};

#ifndef PASS_GROUP_FACES
#define PASS_GROUP_FACES 1
#endif
// 9-lane group faces up to nDof 7 (measured: nDof 2 / 3 +63 / +23 % (the default path there), the
// fallback at nDof 4-7 +2..+13 %; nDof 8 -9 %)
#ifndef PASS_GROUP_FACES_MAXN
#define PASS_GROUP_FACES_MAXN 7
#endif
template <int N, int SL = 6>
struct Geo {
  static constexpr int RS = (N % 2 == 0) ? N + 1 : N;  // odd row stride: conflict-free lines
  static constexpr int PL = N * RS;                    // k3 plane
  static constexpr int VS = N * PL;                    // one quantity
  static constexpr int ES = NVE * VS;                  // one tensor
  static constexpr int LINES = N * N;
  static constexpr int TASKS = SL * LINES;             // per element per pass
  static constexpr int EPB = N <= 2 ? 16 : N == 3 ? 8 : N <= 4 ? 4 : N <= 6 ? 2 : 1;
  static constexpr int THREADS = ((TASKS * EPB + 31) / 32) * 32;
  static constexpr int QPT = (ES * EPB + THREADS - 1) / THREADS;  // qavg values per thread
  static constexpr int FQV = 6 * N * N * NVE;                        // face staging
  static constexpr int EB = ES + (ES > FQV ? ES : FQV);             // per-element doubles
  static constexpr int SMEM = EB * EPB * 8;
  static constexpr int MINB = N >= 10 ? 1 : 2;
};

__device__ __forceinline__ double2 ceo2(int i) {
#ifdef ADERSTP_EXPT_NO_CONST
  return make_double2(0.01 * (i & 7), 0.02);
#endif
  double2 v;
  asm volatile("{\n .reg .u64 ca;\n cvta.to.const.u64 ca, %2;\n ld.const.v2.f64 {%0, %1}, [ca];\n}\n"
               : "=d"(v.x), "=d"(v.y)
               : "l"(&aderstp_kEO[i]));
  return v;
}

// row r of length L (<= 6) at constant offset i, loaded as 16-byte pairs
template <int L>
__device__ __forceinline__ void ceo_row(int i, double (&r)[6]) {
#pragma unroll
  for (int l = 0; l < L; l += 2) {
    const double2 v = ceo2(i + l);
    r[l] = v.x;
    r[l + 1] = v.y;
  }
}

// e_in / e_coef of output quantity s (runtime index) in direction D, from 4-bit packed tables
template <int D>
__device__ __forceinline__ int e_in_rt(int s) {
  constexpr unsigned long long v = [] {
    unsigned long long r = 0;
    for (int q = 0; q < NVE; ++q) r |= (unsigned long long)e_in(q, D) << (4 * q);
    return r;
  }();
  return (int)((v >> (4 * s)) & 15);
}
template <int D>
__device__ __forceinline__ int e_coef_rt(int s) {
  constexpr unsigned long long v = [] {
    unsigned long long r = 0;
    for (int q = 0; q < NVE; ++q) r |= (unsigned long long)e_coef(q, D) << (4 * q);
    return r;
  }();
  return (int)((v >> (4 * s)) & 15);
}
__device__ __forceinline__ double pick4(const double c[4], int i) {
  return i == 0 ? c[0] : i == 1 ? c[1] : i == 2 ? c[2] : c[3];
}

// out[k] = sum_l D[k][l] p[l] via the even/odd split.
template <int N>
__device__ __forceinline__ void eo_apply(const double (&p)[N], double (&out)[N]) {
  constexpr int H = N / 2;
  constexpr int LA = H + (N % 2);  // A acts on e[0..H) and, for odd N, the middle node
  const int base = N * 80;
  double e[H + 1], o[H];
#pragma unroll
  for (int l = 0; l < H; ++l) {
    e[l] = p[l] + p[N - 1 - l];
    o[l] = p[l] - p[N - 1 - l];
  }
  if (N % 2) e[H] = p[H];
#pragma unroll
  for (int k = 0; k < H; ++k) {
    double ra[6], rb[6];
    ceo_row<LA>(base + k * 6, ra);
    ceo_row<H>(base + 30 + k * 6, rb);
    double al = 0.0, be = 0.0;
#pragma unroll
    for (int l = 0; l < LA; ++l) al = fma(ra[l], e[l], al);
#pragma unroll
    for (int l = 0; l < H; ++l) be = fma(rb[l], o[l], be);
    out[k] = al + be;
    out[N - 1 - k] = be - al;
  }
  if (N % 2) {
    double rm[6];
    ceo_row<H + 1>(base + 60, rm);
    double mid = 0.0;
#pragma unroll
    for (int l = 0; l < H; ++l) mid = fma(rm[l], o[l], mid);
    out[H] = fma(rm[H], e[H], mid);
  }
}

// One task of pass D: contract the line (la, lb) of the slot's source field along direction D
// and write (pass x; pass y's first touch of syz) or accumulate coef * D_D f into each target.
template <int N, int D, int SL>
__device__ __forceinline__ void line_pass(const double* P, double* T, int slot, int la, int lb,
                                          const double (&c4)[4]) {
  using G = Geo<N, SL>;
  constexpr int ST = D == 0 ? 1 : D == 1 ? G::RS : G::PL;
  const int start = D == 0 ? la * G::PL + lb * G::RS : D == 1 ? la * G::PL + lb : la * G::RS + lb;
  const PassSlot& ps = kPass[D][slot];
  double p[N], out[N];
  const double* src = P + ps.src * G::VS + start;
#pragma unroll
  for (int l = 0; l < N; ++l) p[l] = src[l * ST];
  eo_apply<N>(p, out);
  const bool write = D == 0 || (D == 1 && slot == 2);
  const int nt = slot == 0 ? 3 : 1;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k < nt) {
      const double c = pick4(c4, ps.coef[k]);
      double* dst = T + ps.tgt[k] * G::VS + start;
      if (write) {
#pragma unroll
        for (int l = 0; l < N; ++l) dst[l * ST] = c * out[l];
      } else {
#pragma unroll
        for (int l = 0; l < N; ++l) dst[l * ST] = fma(c, out[l], dst[l * ST]);
      }
    }
  }
}

template <int N>
struct PassParams {
  double phi[2][N];
  double cf[N];  // cf[o] = dt^(o+1)/(o+1)! (Horner coefficients, stp_splitck.cpp:45,64)
  int check, par_kind, q_stride;
  int prefetch;  // L2 prefetch distance in elements (0: off)
};

// L2 prefetch of [ptr, ptr + bytes) rounded out to 16-byte bounds (cp.async.bulk.prefetch.L2)
__device__ __forceinline__ void prefetch_l2(const void* ptr, unsigned long long bytes) {
  const unsigned long long a0 = reinterpret_cast<unsigned long long>(ptr) & ~15ull;
  const unsigned long long a1 = (reinterpret_cast<unsigned long long>(ptr) + bytes + 15ull) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
}


template <int N>
void fill_pass_params(const LaunchPlan& p, const BatchArgs& a, PassParams<N>& kp) {
  for (int j = 0; j < N; ++j) {
    kp.phi[0][j] = p.basis.face_left[j];
    kp.phi[1][j] = p.basis.face_right[j];
  }
  double c = a.dt;
  kp.cf[0] = c;
  for (int o = 1; o < N; ++o) {
    c *= a.dt / (o + 1);
    kp.cf[o] = c;
  }
  kp.check = p.check;
  kp.par_kind = p.par_kind;
  kp.q_stride = p.q_stride;
  kp.prefetch = p.dmma8_prefetch;
}


template <int N, int SL>
__global__ void __launch_bounds__(Geo<N, SL>::THREADS, Geo<N, SL>::MINB)
stp_pass_kernel(PassParams<N> kp, BatchArgs a, unsigned int* status) {
  using G = Geo<N, SL>;
  extern __shared__ __align__(16) double smp[];
  const int tid = threadIdx.x;
  unsigned int flags = 0;
  const double dt = a.dt;
  const long long e0 = (long long)blockIdx.x * G::EPB;
  auto buf = [&](int ee, int which) { return smp + ee * G::EB + which * G::ES; };
  constexpr int N3 = N * N * N;

  // line task of this thread in every pass: element el, source slot, line index
  const int el = tid / G::TASKS;
  const int slot = (tid - el * G::TASKS) / G::LINES;
  const int line = tid - el * G::TASKS - slot * G::LINES;
  const bool active = el < G::EPB && e0 + el < a.n_elem;
  const int la = line / N, lb = line - la * N;

  // material (proj/src/pde.cpp:171-178) of the task's element
  double c4[4] = {0.0, 0.0, 0.0, 0.0};
  if (active) {
    const double* pr = a.par + 3 * (e0 + el);
    double lam, mu, rho;
    if (kp.par_kind == ADERSTP_PAR_RHO_CP_CS) {
      rho = pr[0];
      mu = __dmul_rn(__dmul_rn(pr[0], pr[2]), pr[2]);
      lam = __dsub_rn(__dmul_rn(__dmul_rn(pr[0], pr[1]), pr[1]), __dmul_rn(2.0, mu));
    } else {
      lam = pr[0];
      mu = pr[1];
      rho = pr[2];
    }
    if (!((rho > 0.0) && (mu >= 0.0) && (lam + 2.0 * mu > 0.0))) flags |= 2u;
    c4[0] = lam + 2.0 * mu;
    c4[1] = lam;
    c4[2] = mu;
    c4[3] = 1.0 / rho;
  }

#ifdef ADERSTP_EXPT_TIMING
  long long tclk[16];
  int tn = 0;
  tclk[tn++] = clock64();
#define TMARK() tclk[tn++] = clock64()
#else
#define TMARK()
#endif
  // ---- stage q: one node (k3,k2,k1) per task, 9 coalesced loads (AoSoA [k3][k2][s][k1]) --
  {
    const int qs = kp.q_stride;
    for (int i = tid; i < G::EPB * N3; i += G::THREADS) {
      const int ee = i / N3, node = i - ee * N3;
      if (e0 + ee >= a.n_elem) continue;
      const int k1 = node % N, k32 = node / N;  // k32 = k3*N + k2
      const double* src = a.q + (e0 + ee) * (long long)(N3 * qs) + k32 * qs * N + k1;
      double* dst = buf(ee, 0) + (k32 / N) * G::PL + (k32 % N) * G::RS + k1;
      double v[NVE];
#pragma unroll
      for (int s = 0; s < NVE; ++s) v[s] = __ldcs(src + s * N);
#pragma unroll
      for (int s = 0; s < NVE; ++s) {
        if (kp.check && !isfinite(v[s])) flags |= 1u;
        dst[s * G::VS] = v[s];
      }
    }
  }
  __syncthreads();
  // qavg accumulator in registers, owned in the shared-memory linear order of the padded
  // tensor (entry j of this thread = offset tid + j*THREADS over all elements of the block)
  double qa[G::QPT];
#pragma unroll
  for (int j = 0; j < G::QPT; ++j) {
    const int i = tid + j * G::THREADS;
    const int ee = i / G::ES;
    qa[j] = (ee < G::EPB) ? dt * buf(ee, 0)[i - ee * G::ES] : 0.0;
  }

  TMARK();
  double coeff = dt;
  int cur = 0;  // buffer holding the current iterate p
#pragma unroll 1
  for (int o = 1; o < N; ++o) {
    const double* P = buf(el < G::EPB ? el : 0, cur);
    double* T = buf(el < G::EPB ? el : 0, cur ^ 1);
    if (active) line_pass<N, 0, SL>(P, T, slot, la, lb, c4);
    __syncthreads();
    if (active) line_pass<N, 1, SL>(P, T, slot, la, lb, c4);
    __syncthreads();
    if (active) line_pass<N, 2, SL>(P, T, slot, la, lb, c4);
    __syncthreads();
    // T = sum_d D_d F_d(p) is the next iterate: qavg += c_o T  (stp_splitck.cpp:64-69)
    coeff *= dt / (o + 1);
    cur ^= 1;
#pragma unroll
    for (int j = 0; j < G::QPT; ++j) {
      const int i = tid + j * G::THREADS;
      const int ee = i / G::ES;
      if (ee < G::EPB) qa[j] = fma(coeff, buf(ee, cur)[i - ee * G::ES], qa[j]);
    }
    // no barrier: the next pass x only reads buf(cur) and writes buf(cur ^ 1), whose readers
    // (this step's passes) are all behind the pass-z barrier
  }
  __syncthreads();  // the qavg reads of the last iterate are done
  TMARK();
#pragma unroll
  for (int j = 0; j < G::QPT; ++j) {
    const int i = tid + j * G::THREADS;
    const int ee = i / G::ES;
    if (ee < G::EPB) buf(ee, 0)[i - ee * G::ES] = qa[j];
  }
  __syncthreads();

  // ---- epilogue --------------------------------------------------------------------------
  // per node: qavg (9 values) and favg (27 values, F_d(qavg) with compile-time (s, d)) to
  // AoSoA [k3][k2][s][k1]; consecutive threads = consecutive k1, so every store is coalesced
  for (int i = tid; i < G::EPB * N3; i += G::THREADS) {
    const int ee = i / N3, node = i - ee * N3;
    if (e0 + ee >= a.n_elem) continue;
    const int k1 = node % N, k32 = node / N;
    const double* qs = buf(ee, 0) + (k32 / N) * G::PL + (k32 % N) * G::RS + k1;
    double v[NVE];
#pragma unroll
    for (int s = 0; s < NVE; ++s) v[s] = qs[s * G::VS];
    const long long ob = (e0 + ee) * (long long)(NVE * N3) + k32 * NVE * N + k1;
#pragma unroll
    for (int s = 0; s < NVE; ++s) __stcs(a.qavg + ob + s * N, v[s]);
    if (a.favg) {
      double cc[4];
      {
        const double* pr = a.par + 3 * (e0 + ee);
        if (kp.par_kind == ADERSTP_PAR_RHO_CP_CS) {
          const double mu = __dmul_rn(__dmul_rn(pr[0], pr[2]), pr[2]);
          const double lam = __dsub_rn(__dmul_rn(__dmul_rn(pr[0], pr[1]), pr[1]), __dmul_rn(2.0, mu));
          cc[0] = lam + 2.0 * mu;
          cc[1] = lam;
          cc[2] = mu;
          cc[3] = 1.0 / pr[0];
        } else {
          cc[0] = pr[0] + 2.0 * pr[1];
          cc[1] = pr[0];
          cc[2] = pr[1];
          cc[3] = 1.0 / pr[2];
        }
      }
      double* fo = a.favg + (e0 + ee) * (long long)(3 * NVE * N3) + k32 * NVE * N + k1;
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int s = 0; s < NVE; ++s)
          __stcs(fo + d * (NVE * N3) + s * N, e_coef(s, d) == 4 ? 0.0 : cc[e_coef(s, d)] * v[e_in(s, d)]);
    }
  }
#if PASS_GROUP_FACES
  if constexpr (N <= PASS_GROUP_FACES_MAXN) {
  if (a.face_q || a.face_f) {
    // nDof <= 7: faces by 9-lane groups as in stp_bip (a warp takes three face nodes, lane =
    // quantity; face_f = F_d(face_q) from the group's lanes by shuffles; 27 consecutive doubles
    // per warp store)
    constexpr int FV = N * N * NVE;
    constexpr int T = G::EPB * 3 * N * N;
    const int lane = tid & 31, grp = lane / NVE, s = lane - grp * NVE;
    const bool live = lane < 3 * NVE;
    for (int it = tid >> 5; 3 * it < T; it += G::THREADS / 32) {
      const int node = 3 * it + (live ? grp : 0);
      const int nd = node < T ? node : 0;
      const int ee = nd / (3 * N * N);
      const bool ok = live && node < T && e0 + ee < a.n_elem;
      const int r = nd - ee * 3 * N * N;
      const int d = r / (N * N), ab = r - d * N * N;
      const int aa = ab / N, bb = ab - aa * N;
      const int start = d == 0 ? aa * G::PL + bb * G::RS : d == 1 ? aa * G::PL + bb : aa * G::RS + bb;
      const int stride = d == 0 ? 1 : d == 1 ? G::RS : G::PL;
      const double* q0 = buf(ee, 0) + start + (live ? s : 0) * G::VS;
      double x0 = 0.0, x1 = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double x = q0[j * stride];
        x0 = fma(kp.phi[0][j], x, x0);
        x1 = fma(kp.phi[1][j], x, x1);
      }
      const long long fb = (e0 + ee) * 6LL * FV + (2 * d) * FV + ab * NVE + s;
      if (ok && a.face_q) {
        __stcs(a.face_q + fb, x0);
        __stcs(a.face_q + fb + FV, x1);
      }
      if (a.face_f) {
        const int so = live ? s : 0;
        const int ci = d == 0 ? e_coef_rt<0>(so) : d == 1 ? e_coef_rt<1>(so) : e_coef_rt<2>(so);
        const int src = d == 0 ? e_in_rt<0>(so) : d == 1 ? e_in_rt<1>(so) : e_in_rt<2>(so);
        const int sl2 = (live ? grp : 0) * NVE + src;
        const double y0 = __shfl_sync(0xffffffffu, x0, sl2), y1 = __shfl_sync(0xffffffffu, x1, sl2);
        if (ok) {
          double c = 0.0;
          if (ci != 4) {
            const double* pr = a.par + 3 * (e0 + ee);
            double cc[4];
            if (kp.par_kind == ADERSTP_PAR_RHO_CP_CS) {
              const double mu = __dmul_rn(__dmul_rn(pr[0], pr[2]), pr[2]);
              const double lam = __dsub_rn(__dmul_rn(__dmul_rn(pr[0], pr[1]), pr[1]), __dmul_rn(2.0, mu));
              cc[0] = lam + 2.0 * mu;
              cc[1] = lam;
              cc[2] = mu;
              cc[3] = 1.0 / pr[0];
            } else {
              cc[0] = pr[0] + 2.0 * pr[1];
              cc[1] = pr[0];
              cc[2] = pr[1];
              cc[3] = 1.0 / pr[2];
            }
            c = pick4(cc, ci);
          }
          __stcs(a.face_f + fb, c * y0);
          __stcs(a.face_f + fb + FV, c * y1);
        }
      }
    }
  }
  } else
#endif
  {
  if (a.face_q || a.face_f) {
    // one task per (normal d, in-face node a, b): all 9 quantities of the normal line, both
    // sides; face_f = F_d(face_q) on the spot.  Output [f][a][b][s]: 9 contiguous doubles per
    // (f, ab) and consecutive tasks = consecutive ab.
    constexpr int FV = N * N * NVE;
    for (int i = tid; i < G::EPB * 3 * N * N; i += G::THREADS) {
      const int ee = i / (3 * N * N);
      if (e0 + ee >= a.n_elem) continue;
      int r = i - ee * 3 * N * N;
      const int d = r / (N * N);
      const int ab = r - d * N * N;
      const int aa = ab / N, bb = ab - aa * N;
      const int start = d == 0 ? aa * G::PL + bb * G::RS : d == 1 ? aa * G::PL + bb : aa * G::RS + bb;
      const int stride = d == 0 ? 1 : d == 1 ? G::RS : G::PL;
      const double* q0 = buf(ee, 0) + start;
      double f0[NVE], f1[NVE];
#pragma unroll
      for (int s = 0; s < NVE; ++s) {
        double x0 = 0.0, x1 = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double x = q0[s * G::VS + j * stride];
          x0 = fma(kp.phi[0][j], x, x0);
          x1 = fma(kp.phi[1][j], x, x1);
        }
        f0[s] = x0;
        f1[s] = x1;
      }
      const long long fb = (e0 + ee) * 6LL * FV + (2 * d) * FV + ab * NVE;
      if (a.face_q) {
#pragma unroll
        for (int s = 0; s < NVE; ++s) {
          __stcs(a.face_q + fb + s, f0[s]);
          __stcs(a.face_q + fb + FV + s, f1[s]);
        }
      }
      if (a.face_f) {
        double cc[4];
        const double* pr = a.par + 3 * (e0 + ee);
        if (kp.par_kind == ADERSTP_PAR_RHO_CP_CS) {
          const double mu = __dmul_rn(__dmul_rn(pr[0], pr[2]), pr[2]);
          const double lam = __dsub_rn(__dmul_rn(__dmul_rn(pr[0], pr[1]), pr[1]), __dmul_rn(2.0, mu));
          cc[0] = lam + 2.0 * mu;
          cc[1] = lam;
          cc[2] = mu;
          cc[3] = 1.0 / pr[0];
        } else {
          cc[0] = pr[0] + 2.0 * pr[1];
          cc[1] = pr[0];
          cc[2] = pr[1];
          cc[3] = 1.0 / pr[2];
        }
        // d is a runtime value here: select the flux row per direction
#pragma unroll
        for (int s = 0; s < NVE; ++s) {
          double g0, g1;
          if (d == 0) {
            g0 = e_coef(s, 0) == 4 ? 0.0 : cc[e_coef(s, 0)] * f0[e_in(s, 0)];
            g1 = e_coef(s, 0) == 4 ? 0.0 : cc[e_coef(s, 0)] * f1[e_in(s, 0)];
          } else if (d == 1) {
            g0 = e_coef(s, 1) == 4 ? 0.0 : cc[e_coef(s, 1)] * f0[e_in(s, 1)];
            g1 = e_coef(s, 1) == 4 ? 0.0 : cc[e_coef(s, 1)] * f1[e_in(s, 1)];
          } else {
            g0 = e_coef(s, 2) == 4 ? 0.0 : cc[e_coef(s, 2)] * f0[e_in(s, 2)];
            g1 = e_coef(s, 2) == 4 ? 0.0 : cc[e_coef(s, 2)] * f1[e_in(s, 2)];
          }
          __stcs(a.face_f + fb + s, g0);
          __stcs(a.face_f + fb + FV + s, g1);
        }
      }
    }
  }
  }
  if (kp.check && flags) atomicOr(status, flags);
#ifdef ADERSTP_EXPT_TIMING
  __syncthreads();
  TMARK();
  if (threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned long long* dbg = reinterpret_cast<unsigned long long*>(a.face_f) + 0;  // scratch
    (void)dbg;
    for (int i = 0; i < tn; ++i) aderstp_dbg_clock[blockIdx.x * 8 + i] = tclk[i];
  }
#endif
}

template <int N, int SL>
cudaError_t launch_pass_n(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  using G = Geo<N, SL>;
  PassParams<N> kp;
  fill_pass_params(p, a, kp);
  auto kern = stp_pass_kernel<N, SL>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  const long long blocks = (a.n_elem + G::EPB - 1) / G::EPB;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)blocks, G::THREADS, G::SMEM, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}


// =============================================================================================
// Bipartite + tensor-memory variant (nDof 9, 10).
//
// The elastic operator couples stresses and velocities only (proj/src/pde.cpp:180-218): stress
// targets read velocity sources and vice versa.  A CK step therefore runs as
//   phase V: new (u, v, w) from the stress fields            -> TEMP (3 spare field slots)
//   phase S: new stresses from the OLD (u, v, w)             -> in place over the stresses
// (the stresses are dead once phase V is done) and the velocity slots swap with TEMP: twelve
// field slots per element instead of eighteen, so nDof 10 fits two CTAs per SM.
// The series is evaluated in Horner form, r <- c_o q + L r (as in stp_dmma8.cu), so there is no
// qavg accumulator at all -- the last iterate IS qavg.  The c_o q term is added by the thread
// that finishes a target line (its z pass); that thread keeps the q values of exactly those
// z-lines in tensor memory (thread-private TMEM columns, tcgen05.ld), off the shared-memory pipe
// and out of the register file.
template <int N>
struct GeoB {
  static_assert(N >= 9 && N <= 10, "TMEM column layout below assumes nDof 9 or 10");
  // Padding chosen by an exhaustive bank-conflict search over the six passes' access patterns
  // (half-warp / quarter-warp bank-pair model, tools/bank_model.py): rows unpadded, planes
  // padded so that y- and z-line starts of consecutive tasks fall on distinct banks; for even N
  // the x lines are read and written as 16-byte pairs.  nDof 10: 4490 vs 6610 wavefronts/step.
  static constexpr int RS = N;
  // (nDof 9 with three CTAs per SM -- 12 x 737 doubles -- measured 4 % slower: the kernel is
  // bound by the shared-memory pipe, not by latency)
  static constexpr int PL = N == 10 ? 106 : 89;
  // nDof 10: 1070 = 14 mod 16 (round 2; was 1060 = 4 mod 16) spreads the 9 quantities of a face node
  // over 8 bank groups in the face groups' line loads (the CK passes touch one slot per warp and are
  // unaffected): C4 +0.7 %
  static constexpr int VS = N == 10 ? 1070 : 801;
  static constexpr bool X128 = N % 2 == 0;
  static constexpr int EB = 12 * VS;  // field slots: 0-5 stresses, 6-8 / 9-11 velocities
  static constexpr int LINES = N * N;
  static constexpr int TASKS = 3 * LINES;
  static constexpr int THREADS = ((TASKS + 31) / 32) * 32;
  static constexpr int NW = THREADS / 32;
  static constexpr int SMEM = EB * 8;
  static constexpr int MINB = 2;  // CTAs per SM
  // TMEM: block k of a thread = the 2N columns [2N k, 2N k + 2N) of its warp's range; warp w
  // needs nb(w) blocks (1 + the phase-S targets of its first lane's slot: 3, 2, 1), and the warps
  // of one lane quarter (w % 4) take consecutive column ranges.
  static constexpr int QC = 2 * N;
  static constexpr int nb(int w) {
    return 32 * w >= TASKS ? 1 : 1 + (3 - (32 * w) / LINES);
  }
  static constexpr int base(int w) {
    int b = 0;
    for (int v = w % 4; v < w; v += 4) b += nb(v) * QC;
    return b;
  }
  static constexpr int tc() {
    int m = 0;
    for (int w = 0; w < NW; ++w) m = base(w) + nb(w) * QC > m ? base(w) + nb(w) * QC : m;
    return m;
  }
  static constexpr int TCOLS = tc() <= 32 ? 32 : tc() <= 64 ? 64 : tc() <= 128 ? 128 : tc() <= 256 ? 256 : 512;
  static_assert(MINB * TCOLS <= 512, "tensor memory of the resident CTAs");
};

// q z-line of TMEM target k (warp-collective: every lane of the warp executes it)
template <int N>
__device__ __forceinline__ void tm_load_q(uint32_t ta, int k, double (&q)[N]) {
  uint32_t r[2 * N];
  tm_ld16(ta + 2 * N * k, r);
  if constexpr (N == 10) tm_ld4(ta + 2 * N * k + 16, r + 16);
  if constexpr (N == 9) tm_ld2(ta + 2 * N * k + 16, r + 16);
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; ++i) q[i] = __hiloint2double(r[2 * i + 1], r[2 * i]);
}
template <int N>
__device__ __forceinline__ void tm_store_q(uint32_t ta, int k, const double (&q)[N]) {
  uint32_t r[2 * N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    r[2 * i] = __double2loint(q[i]);
    r[2 * i + 1] = __double2hiint(q[i]);
  }
  tm_st16(ta + 2 * N * k, r);
  if constexpr (N == 10) tm_st4(ta + 2 * N * k + 16, r + 16);
  if constexpr (N == 9) tm_st2(ta + 2 * N * k + 16, r + 16);
}

// nDof 9, passes x: task line -> x-line.  With the conflict-free y/z padding the x-line starts of
// consecutive lines collide (address = 9 (k3 + k2) mod 16 banks); this permutation, found by
// annealing the bank model (tools/bank_model.py), cuts the x-pass wavefronts by 11 %.
__constant__ uint8_t kXPerm9[81] = {12, 60, 27, 70, 79, 55, 73, 67, 34, 80, 8, 61, 54, 56, 78, 63, 71, 42, 0, 10, 19, 1, 28, 43, 72, 30, 5, 77, 68, 41, 62, 31, 3, 65, 37, 59, 22, 13, 11, 47, 64, 6, 25, 51, 74, 40, 4, 15, 76, 52, 46, 21, 48, 49, 18, 69, 17, 32, 39, 20, 50, 66, 75, 23, 45, 26, 58, 14, 38, 9, 57, 33, 24, 2, 36, 29, 53, 7, 35, 16, 44};

// nDof 10, passes x: the 16-byte x-line accesses of a quarter-warp hit bank group
// (la PL + lb RS) / 2 mod 8 = 5 (la + lb) mod 8; this permutation (annealed with the same bank model,
// started from a periodic residue sequence) spreads every quarter-warp over distinct groups:
// modelled x-pass wavefronts 1400 -> 980 per CK step (ideal 890).
__constant__ uint8_t kXPerm10[100] = {62, 9, 99, 61, 93, 18, 95, 3, 17, 76, 20, 87, 83, 22, 42, 90, 82, 67, 71, 16, 13, 89, 77, 92, 79, 5, 91, 70, 68, 98, 66, 12, 50, 64, 97, 7, 72, 57, 6, 56, 96, 94, 55, 88, 48, 45, 59, 47, 53, 49, 11, 52, 4, 65, 51, 10, 80, 32, 19, 43, 84, 36, 24, 21, 34, 41, 2, 35, 31, 27, 33, 74, 44, 14, 46, 25, 39, 29, 86, 1, 26, 23, 37, 78, 38, 54, 15, 75, 8, 73, 85, 69, 30, 63, 60, 40, 0, 28, 58, 81};

// phase-V pass D, slot j: stress source -> velocity target (coefficient 1/rho)
__constant__ int8_t kBipV[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
// phase-S pass D: slot 0 source (u, v, w)[D] -> sxx, syy, szz with (coef idx); slots 1, 2 shear
__constant__ int8_t kBipS0[3][3] = {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}};
__constant__ int8_t kBipS12[3][2][2] = {{{7, 3}, {8, 4}}, {{6, 3}, {8, 5}}, {{6, 4}, {7, 5}}};  // (src, tgt)

template <int N, int D>
__device__ __forceinline__ int bip_start(int la, int lb) {
  using G = GeoB<N>;
  return D == 0 ? la * G::PL + lb * G::RS : D == 1 ? la * G::PL + lb : la * G::RS + lb;
}

// Passes x and y: contract the source line and write (first touch) or accumulate into targets.
template <int N, int D>
__device__ __forceinline__ void bip_line(const double* src, double* const* dst, const double* cf, int nt,
                                         bool write) {
  using G = GeoB<N>;
  constexpr int ST = D == 0 ? 1 : D == 1 ? G::RS : G::PL;
  double p[N], out[N];
  if constexpr (D == 0 && G::X128) {  // x lines: contiguous, 16-byte aligned
#pragma unroll
    for (int l = 0; l < N; l += 2) {
      const double2 v = *reinterpret_cast<const double2*>(src + l);
      p[l] = v.x;
      p[l + 1] = v.y;
    }
    eo_apply<N>(p, out);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k < nt) {
        double2* d = reinterpret_cast<double2*>(dst[k]);
        const double c = cf[k];
#pragma unroll
        for (int l = 0; l < N; l += 2) {
          if (write) {
            d[l / 2] = make_double2(c * out[l], c * out[l + 1]);
          } else {
            const double2 v = d[l / 2];
            d[l / 2] = make_double2(fma(c, out[l], v.x), fma(c, out[l + 1], v.y));
          }
        }
      }
    }
  } else {
#pragma unroll
    for (int l = 0; l < N; ++l) p[l] = src[l * ST];
    eo_apply<N>(p, out);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k < nt) {
        double* d = dst[k];
        const double c = cf[k];
        if (write) {
#pragma unroll
          for (int l = 0; l < N; ++l) d[l * ST] = c * out[l];
        } else {
#pragma unroll
          for (int l = 0; l < N; ++l) d[l * ST] = fma(c, out[l], d[l * ST]);
        }
      }
    }
  }
}

// Pass z: the last contribution to each target line, plus the Horner term c_o q (TMEM target
// k0 + k).  Warp-collective (the TMEM loads): every thread of the CTA calls it; ntw is the
// warp-uniform maximum target count, nt this thread's (0 for idle threads).
template <int N>
__device__ __forceinline__ void bip_line_z(const double* src, double* const* dst, const double* cf, int nt,
                                           int ntw, uint32_t ta, int k0, double co) {
  using G = GeoB<N>;
  double out[N];
  if (nt > 0) {
    double p[N];
#pragma unroll
    for (int l = 0; l < N; ++l) p[l] = src[l * G::PL];
    eo_apply<N>(p, out);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k >= ntw) break;
    double q[N];
    tm_load_q<N>(ta, k0 + k, q);
    if (k < nt) {
      double* d = dst[k];
      const double c = cf[k];
#pragma unroll
      for (int l = 0; l < N; ++l) d[l * G::PL] = fma(co, q[l], fma(c, out[l], d[l * G::PL]));
    }
  }
}

// Pass z of phase S.  For the normal stresses (slot 0) the x and y passes left the raw derivatives
// a = Dx u in the sxx slot and b = Dy v in the syy slot; with c = Dz w of this z-line
//   sxx = (lambda+2mu) a + lambda (b + c),  syy = (lambda+2mu) b + lambda (a + c),
//   szz = (lambda+2mu) c + lambda (a + b),  plus the Horner term c_o q (TMEM targets k0..k0+2):
// one write per target instead of three read-modify-writes (the sxx/syy/szz passes of the
// per-direction scheme), and the x / y passes of slot 0 store one line instead of three.
// Slots 1, 2 (shear) as bip_line_z.  Warp-collective TMEM loads (ntw = the warp's maximum).
template <int N>
__device__ __forceinline__ void bip_line_z_s(const double* src, double* const* dst, const double* cf, int nt, int ntw,
                                             bool normal, double* sxx, double L, double lam, uint32_t ta, int k0,
                                             double co) {
  using G = GeoB<N>;
  double out[N], a[N], b[N];
  if (nt > 0) {
    double p[N];
#pragma unroll
    for (int l = 0; l < N; ++l) p[l] = src[l * G::PL];
    eo_apply<N>(p, out);  // slot 0: c = Dz w
  }
  if (normal) {
#pragma unroll
    for (int l = 0; l < N; ++l) {
      a[l] = sxx[l * G::PL];
      b[l] = sxx[G::VS + l * G::PL];
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k >= ntw) break;
    double q[N];
    tm_load_q<N>(ta, k0 + k, q);
    if (normal) {
      double* d = sxx + k * G::VS;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const double own = k == 0 ? a[l] : k == 1 ? b[l] : out[l];
        const double rest = k == 0 ? b[l] + out[l] : k == 1 ? a[l] + out[l] : a[l] + b[l];
        d[l * G::PL] = fma(co, q[l], fma(L, own, lam * rest));
      }
    } else if (k < nt) {
      double* d = dst[k];
      const double c = cf[k];
#pragma unroll
      for (int l = 0; l < N; ++l) d[l * G::PL] = fma(co, q[l], fma(c, out[l], d[l * G::PL]));
    }
  }
}

// AOS: the reference's ElementTensor / PredictorOutput node rows [k3][k2][k1][s < 16] in and out
// (proj/src/layout.cpp:9-21): q is staged node-wise from the rows, qavg / favg leave as whole
// 128-byte node rows (4 nodes per warp instruction, padding slots as zeros).
template <int N, bool FUSED = false, bool AOS = false>
__global__ void __launch_bounds__(GeoB<N>::THREADS, GeoB<N>::MINB)
stp_bip_kernel(PassParams<N> kp, BatchArgs a, unsigned int* status) {
  static_assert(!(FUSED && AOS), "the time loop runs on AoSoA");
  using G = GeoB<N>;
  // phase S with raw a = Dx u, b = Dy v combined in the z pass (bip_line_z_s): measured +3.5 % at
  // nDof 9 (5.33 -> 5.52 M elem/s); at nDof 10 the combining pass spills at the 96-register
  // bound of two 320-thread CTAs per SM (-14 %; -8 % with the pass split into half lines), so
  // nDof 10 keeps the per-direction scheme
#ifdef BIP_NO_RAWAB
  constexpr bool kRawAB = false;
#else
  constexpr bool kRawAB = N == 9;
#endif
  extern __shared__ __align__(16) double smb[];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  unsigned int flags = 0;
  const long long e = blockIdx.x;
  constexpr int N3 = N * N * N;
  constexpr int OUTV = NVE * N3;
  double* E = smb;

  TMB(0);
  const int slot = tid / G::LINES;  // 0..2; 3 = padding thread
  const int line = tid - slot * G::LINES;
  const bool active = slot < 3;
  const int sl = active ? slot : 0;
  const int la = line / N, lb = line - la * N;
  const int xline = N == 9 ? kXPerm9[line < 81 ? line : 0] : N == 10 ? kXPerm10[line < 100 ? line : 0] : line;  // x passes
  const int lax = xline / N, lbx = xline - lax * N;

  if (kp.prefetch && tid == 0 && e + kp.prefetch < a.n_elem)
    prefetch_l2(a.q + (e + kp.prefetch) * (long long)(N3 * kp.q_stride), 8ull * N3 * kp.q_stride);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base_s)),
                 "n"(G::TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }

  double c4[4];
  {
    const double* pr = a.par + 3 * e;
    double lam, mu, rho;
    if (kp.par_kind == ADERSTP_PAR_RHO_CP_CS) {
      rho = pr[0];
      mu = __dmul_rn(__dmul_rn(pr[0], pr[2]), pr[2]);
      lam = __dsub_rn(__dmul_rn(__dmul_rn(pr[0], pr[1]), pr[1]), __dmul_rn(2.0, mu));
    } else {
      lam = pr[0];
      mu = pr[1];
      rho = pr[2];
    }
    if (!((rho > 0.0) && (mu >= 0.0) && (lam + 2.0 * mu > 0.0))) flags |= 2u;
    c4[0] = lam + 2.0 * mu;
    c4[1] = lam;
    c4[2] = mu;
    c4[3] = 1.0 / rho;
  }

  // ---- stage q -> field slots 0..8 (node-wise, coalesced AoSoA loads; k1 pairs for even N) --
  if constexpr (AOS) {  // node rows: slots 0..8 as four 16-byte pairs and one scalar
    for (int i = tid; i < N3; i += G::THREADS) {
      const double* src = a.q + e * (long long)(N3 * 16) + i * 16;
      double* dst = E + (i / (N * N)) * G::PL + ((i / N) % N) * G::RS + i % N;
      double2 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = __ldcs(reinterpret_cast<const double2*>(src + 2 * j));
      const double v8 = __ldcs(src + 8);
      if (kp.check && !isfinite(v8)) flags |= 1u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (kp.check && !(isfinite(v[j].x) && isfinite(v[j].y))) flags |= 1u;
        dst[(2 * j) * G::VS] = v[j].x;
        dst[(2 * j + 1) * G::VS] = v[j].y;
      }
      dst[8 * G::VS] = v8;
    }
  } else {
    const int qs = kp.q_stride;
    constexpr int V = N % 2 == 0 ? 2 : 1;  // nodes per task
    for (int i = tid; i < N3 / V; i += G::THREADS) {
      const int k1 = V * (i % (N / V)), k32 = i / (N / V);
      const double* src = a.q + e * (long long)(N3 * qs) + k32 * qs * N + k1;
      double* dst = E + (k32 / N) * G::PL + (k32 % N) * G::RS + k1;
      if constexpr (V == 2) {
        double2 v[NVE];
#pragma unroll
        for (int s = 0; s < NVE; ++s) v[s] = __ldcs(reinterpret_cast<const double2*>(src + s * N));
#pragma unroll
        for (int s = 0; s < NVE; ++s) {
          if (kp.check && !(isfinite(v[s].x) && isfinite(v[s].y))) flags |= 1u;
          *reinterpret_cast<double2*>(dst + s * G::VS) = v[s];
        }
      } else {
        double v[NVE];
#pragma unroll
        for (int s = 0; s < NVE; ++s) v[s] = __ldcs(src + s * N);
#pragma unroll
        for (int s = 0; s < NVE; ++s) {
          if (kp.check && !isfinite(v[s])) flags |= 1u;
          dst[s * G::VS] = v[s];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  int wbase = 0;  // G::base(warp), evaluated at run time
  for (int v = warp & 3; v < warp; v += 4) wbase += G::nb(v) * G::QC;
  const uint32_t ta = tmem_base_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)wbase;

  // ---- q of the target lines this thread finishes (its z pass) -> TMEM:
  //   block 0: the phase-V velocity 6 + slot
  //   blocks 1..: phase-S stresses -- slot 0: sxx, syy, szz; slot 1: sxz and sxy (sxy has no
  //   z term: the slot-1 z pass adds only its Horner term); slot 2: syz
  const int ntS = active ? (slot == 0 ? 3 : slot == 1 ? 2 : 1) : 0;
  const int ntS_w = __reduce_max_sync(0xffffffffu, (unsigned)ntS);
  const int zst = la * G::RS + lb;  // z-line (k2, k1) = (la, lb)
  // These z-lines cover every node of the nine fields exactly once, so the same loop also
  // writes the Horner start r = c_(n-1) q back in place.
  {
    const double c = kp.cf[N - 1];
    double v[N];
    double* z0 = E + (6 + sl) * G::VS + zst;
#pragma unroll
    for (int l = 0; l < N; ++l) v[l] = active ? z0[l * G::PL] : 0.0;
    tm_store_q<N>(ta, 0, v);
    if (active) {
#pragma unroll
      for (int l = 0; l < N; ++l) z0[l * G::PL] = c * v[l];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k >= ntS_w) break;
      const int f = slot == 0 ? k : slot == 1 ? (k == 0 ? 4 : 3) : 5;
      double* zk = E + f * G::VS + zst;
#pragma unroll
      for (int l = 0; l < N; ++l) v[l] = (k < ntS) ? zk[l * G::PL] : 0.0;
      tm_store_q<N>(ta, 1 + k, v);
      if (k < ntS) {
#pragma unroll
        for (int l = 0; l < N; ++l) zk[l * G::PL] = c * v[l];
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  __syncthreads();

  TMB(1);
  int vb = 6;  // slot of u (velocities occupy vb .. vb+2; the other three slots are TEMP)
  // ---- epilogue pieces (called after the recursion; in the fused time-step mode the faces are
  // taken from qavg before one more Horner step with coefficient 1 gives u + L(qavg)) ---------
  auto fld = [&](int s) { return s < 6 ? s : vb + (s - 6); };
  auto emit_qavg = [&]() {
  if constexpr (AOS) {
    // lane = (node ns of 4, slot pair c2): 4 x 128 contiguous bytes per warp instruction; the
    // flux table entries of the lane's two slots are fixed per lane
    const int lane = tid & 31, ns = lane >> 3, c2 = 2 * (lane & 7);
    int srcf[3][2], fl[2];
    double cfo[3][2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int so = c2 + j;
      fl[j] = so < NVE ? fld(so) : -1;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int ci = so < NVE ? e_coef(so, d) : 4;
        srcf[d][j] = so < NVE ? fld(e_in(so, d)) : 0;
        cfo[d][j] = ci == 4 ? 0.0 : pick4(c4, ci);
      }
    }
    double* qo = a.qavg + e * (long long)(N3 * 16);
    double* fo = a.favg ? a.favg + e * (long long)(3 * N3 * 16) : nullptr;
    for (int nb = 4 * warp + ns; nb < N3; nb += 4 * G::NW) {
      const int pos = (nb / (N * N)) * G::PL + ((nb / N) % N) * G::RS + nb % N;
      __stcs(reinterpret_cast<double2*>(qo + nb * 16 + c2),
             make_double2(fl[0] >= 0 ? E[fl[0] * G::VS + pos] : 0.0, fl[1] >= 0 ? E[fl[1] * G::VS + pos] : 0.0));
      if (fo) {
#pragma unroll
        for (int d = 0; d < 3; ++d)
          __stcs(reinterpret_cast<double2*>(fo + d * (N3 * 16) + nb * 16 + c2),
                 make_double2(cfo[d][0] != 0.0 ? cfo[d][0] * E[srcf[d][0] * G::VS + pos] : 0.0,
                              cfo[d][1] != 0.0 ? cfo[d][1] * E[srcf[d][1] * G::VS + pos] : 0.0));
      }
    }
  } else if constexpr (N % 2 == 0) {  // k1 pairs: 16-byte shared loads and global stores
    for (int i = tid; i < N3 / 2; i += G::THREADS) {
      const int k1 = 2 * (i % (N / 2)), k32 = i / (N / 2);
      const double* qs = E + (k32 / N) * G::PL + (k32 % N) * G::RS + k1;
      double2 v[NVE];
#pragma unroll
      for (int s = 0; s < NVE; ++s) v[s] = *reinterpret_cast<const double2*>(qs + fld(s) * G::VS);
      const long long ob = e * (long long)OUTV + k32 * NVE * N + k1;
#pragma unroll
      for (int s = 0; s < NVE; ++s) __stcs(reinterpret_cast<double2*>(a.qavg + ob + s * N), v[s]);
      if (a.favg) {
        double* fo = a.favg + e * (long long)(3 * OUTV) + k32 * NVE * N + k1;
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int s = 0; s < NVE; ++s) {
            const double c = c4[e_coef(s, d) == 4 ? 0 : e_coef(s, d)];
            const double2 x = v[e_in(s, d)];
            __stcs(reinterpret_cast<double2*>(fo + d * OUTV + s * N),
                   e_coef(s, d) == 4 ? make_double2(0.0, 0.0) : make_double2(c * x.x, c * x.y));
          }
      }
    }
  } else {
    for (int i = tid; i < N3; i += G::THREADS) {
      const int k1 = i % N, k32 = i / N;
      const double* qs = E + (k32 / N) * G::PL + (k32 % N) * G::RS + k1;
      double v[NVE];
#pragma unroll
      for (int s = 0; s < NVE; ++s) v[s] = qs[fld(s) * G::VS];
      const long long ob = e * (long long)OUTV + k32 * NVE * N + k1;
#pragma unroll
      for (int s = 0; s < NVE; ++s) __stcs(a.qavg + ob + s * N, v[s]);
      if (a.favg) {
        double* fo = a.favg + e * (long long)(3 * OUTV) + k32 * NVE * N + k1;
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int s = 0; s < NVE; ++s)
            __stcs(fo + d * OUTV + s * N, e_coef(s, d) == 4 ? 0.0 : c4[e_coef(s, d)] * v[e_in(s, d)]);
      }
    }
  }
  };
  // Faces: a warp takes three face nodes (d, a, b) at a time, one 9-lane group per node and one
  // lane per quantity s (lanes 27..31 idle): lane (node, s) contracts the normal line of quantity
  // s (both sides) and face_f[s] = F_d(face_q)_s = coef(s, d) face_q[in(s, d)] comes from lane
  // in(s, d) of its group by shuffles, so every face entry is computed once and a warp stores 27
  // consecutive doubles per array (coalesced, [f][a][b][s]).
  auto emit_faces = [&]() {
  if (a.face_q || a.face_f) {
    constexpr int FV = N * N * NVE;
    constexpr int T = 3 * N * N;  // face nodes (d, a, b)
    const int lane = tid & 31, grp = lane / NVE, s = lane - grp * NVE;
    const bool live = lane < 3 * NVE;
    for (int it = warp; 3 * it < T; it += G::NW) {
      const int node = 3 * it + (live ? grp : 0);
      const bool ok = live && node < T;
      const int nd = ok ? node : 0;
      const int d = nd / (N * N), ab = nd - d * N * N;
      const int aa = ab / N, bb = ab - aa * N;
      const int start = d == 0 ? aa * G::PL + bb * G::RS : d == 1 ? aa * G::PL + bb : aa * G::RS + bb;
      const int stride = d == 0 ? 1 : d == 1 ? G::RS : G::PL;
      const double* q0 = E + fld(live ? s : 0) * G::VS + start;
      double x0 = 0.0, x1 = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double x = q0[j * stride];
        x0 = fma(kp.phi[0][j], x, x0);
        x1 = fma(kp.phi[1][j], x, x1);
      }
      const long long fb = e * 6LL * FV + (2 * d) * FV + ab * NVE + s;
      if (ok && a.face_q) {
        __stcs(a.face_q + fb, x0);
        __stcs(a.face_q + fb + FV, x1);
      }
      if (a.face_f) {
        const int so = live ? s : 0;
        const int ci = d == 0 ? e_coef_rt<0>(so) : d == 1 ? e_coef_rt<1>(so) : e_coef_rt<2>(so);
        const int src = d == 0 ? e_in_rt<0>(so) : d == 1 ? e_in_rt<1>(so) : e_in_rt<2>(so);
        const int sl2 = (live ? grp : 0) * NVE + src;
        const double y0 = __shfl_sync(0xffffffffu, x0, sl2), y1 = __shfl_sync(0xffffffffu, x1, sl2);
        if (ok) {
          const double c = ci == 4 ? 0.0 : pick4(c4, ci);
          __stcs(a.face_f + fb, c * y0);
          __stcs(a.face_f + fb + FV, c * y1);
        }
      }
    }
  }
  };
  auto emit_state = [&]() {  // fused: u_next in q's layout from the nine fields
    const int qs = kp.q_stride;
    for (int i = tid; i < N3; i += G::THREADS) {
      const int k1 = i % N, k32 = i / N;
      const double* src = E + (k32 / N) * G::PL + (k32 % N) * G::RS + k1;
      double* dst = a.u_next + e * (long long)(N3 * qs) + k32 * qs * N + k1;
#pragma unroll
      for (int s = 0; s < NVE; ++s) __stcs(dst + s * N, src[fld(s) * G::VS]);
    }
  };
#pragma unroll 1
  for (int o = N - 2; o >= (FUSED ? -1 : 0); --o) {
    if (FUSED && o < 0) {  // faces of qavg, then the extra step overwrites the fields
      emit_faces();
      __syncthreads();
    }
    const double co = (!FUSED || o >= 0) ? kp.cf[o] : 1.0;
    const int tb = 15 - vb;  // TEMP base: 9 when vb = 6, 6 when vb = 9
    const double crho[3] = {c4[3], 0.0, 0.0};
    // phase V: velocity targets from stress sources, into TEMP
    if (active) {
      double* dst[3] = {E + (tb + sl) * G::VS + bip_start<N, 0>(lax, lbx), nullptr, nullptr};
      bip_line<N, 0>(E + kBipV[0][sl] * G::VS + bip_start<N, 0>(lax, lbx), dst, crho, 1, true);
    }
    __syncthreads();
    if (active) {
      double* dst[3] = {E + (tb + sl) * G::VS + bip_start<N, 1>(la, lb), nullptr, nullptr};
      bip_line<N, 1>(E + kBipV[1][sl] * G::VS + bip_start<N, 1>(la, lb), dst, crho, 1, false);
    }
    __syncthreads();
    {
      double* dst[3] = {E + (tb + sl) * G::VS + zst, nullptr, nullptr};
      bip_line_z<N>(E + kBipV[2][sl] * G::VS + zst, dst, crho, active ? 1 : 0, 1, ta, 0, co);
    }
    __syncthreads();
    // phase S: stress targets from the old velocities, in place over the (dead) stresses
    {
      double cf[3];
      double* dst[3];
      int srcf, nt;
      if (slot == 0) {
        srcf = vb;
        if constexpr (!kRawAB) {
          nt = 3;
#pragma unroll
          for (int k = 0; k < 3; ++k) cf[k] = pick4(c4, kBipS0[0][k]);
        } else {
          nt = 1;  // raw a = Dx u into the sxx slot (bip_line_z_s combines)
          cf[0] = 1.0;
          cf[1] = cf[2] = 0.0;
        }
      } else {
        srcf = vb + (kBipS12[0][sl > 0 ? sl - 1 : 0][0] - 6);
        nt = 1;
        cf[0] = c4[2];
        cf[1] = cf[2] = 0.0;
      }
      const int st = bip_start<N, 0>(lax, lbx);
      if (slot == 0) {
        dst[0] = E + st;
        dst[1] = E + G::VS + st;
        dst[2] = E + 2 * G::VS + st;
      } else {
        dst[0] = E + kBipS12[0][sl > 0 ? sl - 1 : 0][1] * G::VS + st;
        dst[1] = dst[2] = nullptr;
      }
      if (active) bip_line<N, 0>(E + srcf * G::VS + st, dst, cf, nt, true);
    }
    __syncthreads();
    {
      double cf[3];
      double* dst[3];
      int srcf, nt;
      if (slot == 0) {
        srcf = vb + 1;
        if constexpr (!kRawAB) {
          nt = 3;
#pragma unroll
          for (int k = 0; k < 3; ++k) cf[k] = pick4(c4, kBipS0[1][k]);
        } else {
          nt = 1;  // raw b = Dy v into the syy slot
          cf[0] = 1.0;
          cf[1] = cf[2] = 0.0;
        }
      } else {
        srcf = vb + (kBipS12[1][sl > 0 ? sl - 1 : 0][0] - 6);
        nt = 1;
        cf[0] = c4[2];
        cf[1] = cf[2] = 0.0;
      }
      const int st = bip_start<N, 1>(la, lb);
      if (slot == 0) {
        if constexpr (!kRawAB) {
          dst[0] = E + st;
          dst[1] = E + G::VS + st;
          dst[2] = E + 2 * G::VS + st;
        } else {
          dst[0] = E + G::VS + st;
          dst[1] = dst[2] = nullptr;
        }
      } else {
        dst[0] = E + kBipS12[1][sl > 0 ? sl - 1 : 0][1] * G::VS + st;
        dst[1] = dst[2] = nullptr;
      }
      // syz (slot 2) gets its first contribution here (and raw b in slot 0)
      if (active) bip_line<N, 1>(E + srcf * G::VS + st, dst, cf, nt, kRawAB ? slot != 1 : slot == 2);
    }
    __syncthreads();
    {
      double cf[3];
      double* dst[3];
      int srcf;
      if (slot == 0) {
        srcf = vb + 2;
#pragma unroll
        for (int k = 0; k < 3; ++k) cf[k] = pick4(c4, kBipS0[2][k]);
        dst[0] = E + zst;
        dst[1] = E + G::VS + zst;
        dst[2] = E + 2 * G::VS + zst;
      } else {
        srcf = vb + (kBipS12[2][sl > 0 ? sl - 1 : 0][0] - 6);
        cf[0] = c4[2];
        cf[1] = cf[2] = 0.0;  // slot 1, target 1 = sxy: coefficient 0, Horner term only
        dst[0] = E + kBipS12[2][sl > 0 ? sl - 1 : 0][1] * G::VS + zst;
        dst[1] = E + 3 * G::VS + zst;
        dst[2] = nullptr;
      }
      if constexpr (!kRawAB) {
        bip_line_z<N>(E + srcf * G::VS + zst, dst, cf, ntS, ntS_w, ta, 1, co);
      } else {
        // slot 0 (normal stresses) combines the raw a, b with c = Dz w; slots 1, 2 as before --
        // each warp runs the TMEM loads of the larger of its slots' target counts
        bip_line_z_s<N>(E + srcf * G::VS + zst, dst, cf, ntS, ntS_w, slot == 0, E + zst, c4[0], c4[1], ta, 1, co);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    vb = tb;  // the new velocities live in TEMP
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base_s), "n"(G::TCOLS)
                 : "memory");

  TMB(2);
  if (FUSED) {
    emit_state();
  } else {
    emit_qavg();
    TMB(3);
    emit_faces();
  }
#ifdef ADERSTP_EXPT_TIMING
  __syncthreads();
#endif
  TMB(4);
  if (kp.check && flags) atomicOr(status, flags);
}

template <int N>
cudaError_t launch_bip_n(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  using G = GeoB<N>;
  PassParams<N> kp;
  fill_pass_params(p, a, kp);
  auto kern = a.u_next ? stp_bip_kernel<N, true> : p.layout == ADERSTP_LAYOUT_AOS ? stp_bip_kernel<N, false, true>
                                                                                  : stp_bip_kernel<N, false>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  if (a.n_elem == 0) return cudaSuccess;
  if (a.n_elem > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)a.n_elem, G::THREADS, G::SMEM, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}


// =============================================================================================
// Table PDEs at nDof 9, 10 (the user-LinearPde path; stp_tlp): any constant-coefficient system
// with m <= 9 quantities given as term tables (build_terms: C_d = A_d + B_d, at most 4 nonzeros
// per row), as line passes on the bipartite kernel's machinery (even/odd D from the constant
// bank, the GeoB padding).  A CK step in Horner form, r <- c_o q + sum_d sum_k tc[s][d][k] D_d
// r_(tr[s][d][k]) (proj/src/stp_splitck.cpp:46-70 with D_d F_d(p) + B_d D_d p = C_d D_d p for
// constant coefficients), runs as three passes x, y, z over the lines of every target quantity:
// thread (s, line) owns one line of target s, contracts the lines of its sources and writes
// (pass x) or accumulates (y, z) the next iterate T; pass z adds c_o q from tensor memory
// (thread-private columns: the thread keeps exactly its z-line of q).  The iterate pair (P, T)
// is 2 m field slots of shared memory.  Outputs as in proj/src/predictor_common.cpp:311-341.
template <int N>
struct TlpParams {
  double phi[2][N];
  double cf[N];  // cf[o] = dt^(o+1)/(o+1)! (stp_splitck.cpp:45,64)
  int m, q_stride, out_stride, check, n_terms;
  signed char tr[kMaxM][3][kMaxTerms];
  signed char fr[kMaxM][3][kMaxTerms];
  double tc[kMaxM][3][kMaxTerms];
  double fc[kMaxM][3][kMaxTerms];
};
constexpr int kTlpM = 9;  // quantities per element of this kernel

template <int N, int MQ = kTlpM>  // MQ: quantities the instance is sized for (threads = MQ N^2)
struct GeoT {
  using B = GeoB<N>;
  static constexpr int LINES = N * N;
  static constexpr int THREADS = ((MQ * LINES + 31) / 32) * 32;
  static constexpr int NW = THREADS / 32;
  static constexpr int QC = 2 * N;  // TMEM columns per thread (its q z-line)
  static constexpr int TCOLS = ((NW + 3) / 4) * QC <= 128 ? 128 : 256;
};

// acc += c D line, for one line (start, stride) of a field slot: eo_apply with the update folded in
// (out[] never materialised: 2N registers fewer, the same operations and rounding as
// acc = fma(c, out, acc) after eo_apply)
template <int N>
__device__ __forceinline__ void tlp_contract_acc(const double* src, int stride, double c, double (&acc)[N]) {
  constexpr int H = N / 2;
  constexpr int LA = H + (N % 2);
  const int base = N * 80;
  double e[H + 1], o[H];
#pragma unroll
  for (int l = 0; l < H; ++l) {
    const double a0 = src[l * stride], a1 = src[(N - 1 - l) * stride];
    e[l] = a0 + a1;
    o[l] = a0 - a1;
  }
  if (N % 2) e[H] = src[H * stride];
#pragma unroll
  for (int k = 0; k < H; ++k) {
    double ra[6], rb[6];
    ceo_row<LA>(base + k * 6, ra);
    ceo_row<H>(base + 30 + k * 6, rb);
    double al = 0.0, be = 0.0;
#pragma unroll
    for (int l = 0; l < LA; ++l) al = fma(ra[l], e[l], al);
#pragma unroll
    for (int l = 0; l < H; ++l) be = fma(rb[l], o[l], be);
    acc[k] = fma(c, al + be, acc[k]);
    acc[N - 1 - k] = fma(c, be - al, acc[N - 1 - k]);
  }
  if (N % 2) {
    double rm[6];
    ceo_row<H + 1>(base + 60, rm);
    double mid = 0.0;
#pragma unroll
    for (int l = 0; l < H; ++l) mid = fma(rm[l], o[l], mid);
    acc[H] = fma(c, fma(rm[H], e[H], mid), acc[H]);
  }
}

template <int N, int MQ>
__global__ void __launch_bounds__(GeoT<N, MQ>::THREADS, 1)
stp_tlp_kernel(TlpParams<N> kp, BatchArgs a, unsigned int* status) {
  using B = GeoB<N>;
  using G = GeoT<N, MQ>;
  extern __shared__ __align__(16) double smt[];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int m = kp.m;
  const long long e = blockIdx.x;
  constexpr int N3 = N * N * N;
  const int s = tid / G::LINES, line = tid - s * G::LINES;
  const bool active = s < m;
  const int sa = active ? s : 0;
  const int la = line / N, lb = line - la * N;
  // the iterate pair: step i reads smt + (i & 1) * mvs and writes the other half (computed, not
  // indexed: a runtime-indexed pointer array turns every access into a generic load)
  const int mvs = m * B::VS;
  unsigned int flags = 0;

  if (warp == 0) tm_alloc<G::TCOLS>(&tmem_base_s);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t ta = tmem_base_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * G::QC);

  // ---- stage: thread (s, k2 = la, k1 = lb) loads the z-line of q_s: c_(N-1) q -> P, q -> TMEM
  {
    double qz[N];
    const int qs = kp.q_stride;
    const double* src = a.q + e * (long long)(N3 * qs) + (la * qs + sa) * N + lb;
#pragma unroll
    for (int l = 0; l < N; ++l) qz[l] = active ? __ldcs(src + (long long)l * N * qs * N) : 0.0;
    if (kp.check && active) {
#pragma unroll
      for (int l = 0; l < N; ++l)
        if (!isfinite(qz[l])) flags |= 1u;
    }
    double* pz = smt + sa * B::VS + la * B::RS + lb;
    const double c0 = kp.cf[N - 1];
    if (active) {
#pragma unroll
      for (int l = 0; l < N; ++l) pz[l * B::PL] = c0 * qz[l];
    }
    tm_store_q<N>(ta, 0, qz);
    tm_wait_st();
  }
  __syncthreads();

  // ---- CK recursion, Horner form: step i reads half i & 1 of the pair, writes the other -------
  const int nterm = kp.n_terms;
  int i = 0;
#pragma unroll 1
  for (int o = N - 2; o >= 0; --o, ++i) {
    const double* P = smt + (i & 1) * mvs;
    double* T = smt + ((i + 1) & 1) * mvs;
    // pass x: line (k3 = la, k2 = lb) of target s, written
    if (active) {
      double acc[N];
#pragma unroll
      for (int l = 0; l < N; ++l) acc[l] = 0.0;
      const int st = la * B::PL + lb * B::RS;
#pragma unroll 1
      for (int k = 0; k < nterm; ++k) {
        const double c = kp.tc[s][0][k];
        if (c == 0.0) continue;
        tlp_contract_acc<N>(P + kp.tr[s][0][k] * B::VS + st, 1, c, acc);
      }
#pragma unroll
      for (int l = 0; l < N; ++l) T[s * B::VS + st + l] = acc[l];
    }
    __syncthreads();
    // pass y: line (k3 = la, k1 = lb), accumulated
    if (active) {
      const int st = la * B::PL + lb;
      double acc[N];
      double* tl = T + s * B::VS + st;
#pragma unroll
      for (int l = 0; l < N; ++l) acc[l] = tl[l * B::RS];
#pragma unroll 1
      for (int k = 0; k < nterm; ++k) {
        const double c = kp.tc[s][1][k];
        if (c == 0.0) continue;
        tlp_contract_acc<N>(P + kp.tr[s][1][k] * B::VS + st, B::RS, c, acc);
      }
#pragma unroll
      for (int l = 0; l < N; ++l) tl[l * B::RS] = acc[l];
    }
    __syncthreads();
    // pass z: line (k2 = la, k1 = lb), accumulated, plus the Horner term c_o q (TMEM, all lanes)
    {
      const int st = la * B::RS + lb;
      double acc[N];
      double* tl = T + sa * B::VS + st;
      if (active) {
#pragma unroll
        for (int l = 0; l < N; ++l) acc[l] = tl[l * B::PL];
#pragma unroll 1
        for (int k = 0; k < nterm; ++k) {
          const double c = kp.tc[s][2][k];
          if (c == 0.0) continue;
          tlp_contract_acc<N>(P + kp.tr[s][2][k] * B::VS + st, B::PL, c, acc);
        }
      }
      double q[N];
      tm_load_q<N>(ta, 0, q);
      const double co = kp.cf[o];
      if (active) {
#pragma unroll
        for (int l = 0; l < N; ++l) tl[l * B::PL] = fma(co, q[l], acc[l]);
      }
    }
    __syncthreads();
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 0) {
    tm_fence_after();
    tm_dealloc<G::TCOLS>(tmem_base_s);
  }

  // ---- epilogue: qavg = the last iterate; favg_d = A_d qavg; faces (predictor_common.cpp:311-341)
  const double* Q = smt + (i & 1) * mvs;
  const int os = kp.out_stride;
  // x / os and x / m by a float reciprocal: (x + 0.5) / d is at least 0.5 / d <= 1/128 away from
  // an integer, x < 2^15 and the float product is within 2^-23 relative: it truncates to the
  // exact quotient
  const float inv_os = 1.0f / (float)os, inv_m = 1.0f / (float)m;
  auto qdiv = [](int x, float inv) { return (int)(((float)x + 0.5f) * inv); };
  auto qv = [&](int q, int k3, int k2, int k1) { return Q[q * B::VS + k3 * B::PL + k2 * B::RS + k1]; };
  if (a.qavg) {
    double* out = a.qavg + e * (long long)(N3 * os);
    for (int j = tid; j < N3 * os; j += G::THREADS) {
      const int r = j / N, k1 = j - r * N, k32 = qdiv(r, inv_os), so = r - k32 * os;
      __stcs(out + j, so < m ? qv(so, k32 / N, k32 % N, k1) : 0.0);
    }
  }
  if (a.favg) {
    double* out = a.favg + e * (long long)(3 * N3 * os);
    for (int j = tid; j < 3 * N3 * os; j += G::THREADS) {
      const int r0 = j / N, k1 = j - r0 * N, dk = qdiv(r0, inv_os), so = r0 - dk * os;
      const int d = dk / (N * N), k32 = dk - d * N * N;
      double v = 0.0;
      if (so < m)
        for (int k = 0; k < nterm; ++k) {
          const double c = kp.fc[so][d][k];
          if (c != 0.0) v = fma(c, qv(kp.fr[so][d][k], k32 / N, k32 % N, k1), v);
        }
      __stcs(out + j, v);
    }
  }
  if (a.face_q || a.face_f) {
    // faces by m-lane groups (32 / m face nodes per warp, one lane per quantity): lane (node, s)
    // contracts the normal line of quantity s for both sides; face_f[s] = sum_k fc[s][d][k]
    // face_q[fr[s][d][k]] comes from the group's lanes by shuffles; a warp stores consecutive
    // entries of [f][a][b][s]
    const int FV = N * N * m;
    const int gpw = 32 / m;  // groups per warp
    const int lane = tid & 31, grp = lane / m, sq = lane - grp * m;
    const bool live = grp < gpw;
    for (int it = warp; it * gpw < 3 * N * N; it += G::NW) {
      const int node = it * gpw + (live ? grp : 0);
      const bool ok = live && node < 3 * N * N;
      const int nd = ok ? node : 0, d = nd / (N * N), ab = nd - d * N * N;
      const int aa = ab / N, bb = ab - aa * N;
      const int st = d == 0 ? aa * B::PL + bb * B::RS : d == 1 ? aa * B::PL + bb : aa * B::RS + bb;
      const int stride = d == 0 ? 1 : d == 1 ? B::RS : B::PL;
      const double* l0 = Q + (live ? sq : 0) * B::VS + st;
      double x0 = 0.0, x1 = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const double v = l0[l * stride];
        x0 = fma(kp.phi[0][l], v, x0);
        x1 = fma(kp.phi[1][l], v, x1);
      }
      const long long fb = e * 6ll * FV + (2 * d) * FV + ab * m + sq;
      if (ok && a.face_q) {
        __stcs(a.face_q + fb, x0);
        __stcs(a.face_q + fb + FV, x1);
      }
      if (a.face_f) {
        double g0 = 0.0, g1 = 0.0;
        for (int k = 0; k < nterm; ++k) {  // warp-uniform trip count: every lane shuffles
          const double c = ok ? kp.fc[sq][d][k] : 0.0;
          const int src = (live ? grp : 0) * m + (ok ? kp.fr[sq][d][k] : 0);
          const double y0 = __shfl_sync(0xffffffffu, x0, src), y1 = __shfl_sync(0xffffffffu, x1, src);
          g0 = fma(c, y0, g0);
          g1 = fma(c, y1, g1);
        }
        if (ok) {
          __stcs(a.face_f + fb, g0);
          __stcs(a.face_f + fb + FV, g1);
        }
      }
    }
  }
  if (kp.check && flags) atomicOr(status, flags);
}

template <int N, int MQ>
cudaError_t launch_tlp_n(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  using B = GeoB<N>;
  using G = GeoT<N, MQ>;
  TlpParams<N> kp;
  for (int j = 0; j < N; ++j) {
    kp.phi[0][j] = p.basis.face_left[j];
    kp.phi[1][j] = p.basis.face_right[j];
  }
  double c = a.dt;  // the reference's operation sequence (stp_splitck.cpp:45,64)
  kp.cf[0] = c;
  for (int o = 1; o < N; ++o) {
    c *= a.dt / (o + 1);
    kp.cf[o] = c;
  }
  kp.m = p.m;
  kp.q_stride = p.q_stride;
  kp.out_stride = p.out_stride;
  kp.check = p.check;
  kp.n_terms = p.n_terms;
  for (int q = 0; q < kMaxM; ++q)
    for (int d = 0; d < 3; ++d)
      for (int k = 0; k < kMaxTerms; ++k) {
        kp.tr[q][d][k] = p.tr[q][d][k];
        kp.fr[q][d][k] = p.fr[q][d][k];
        kp.tc[q][d][k] = p.tc[q][d][k];
        kp.fc[q][d][k] = p.fc[q][d][k];
      }
  const int smem = 2 * p.m * B::VS * 8;
  auto kern = stp_tlp_kernel<N, MQ>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * MQ * B::VS * 8);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  if (a.n_elem == 0) return cudaSuccess;
  if (a.n_elem > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)a.n_elem, G::THREADS, smem, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}
}  // namespace

// table PDEs at nDof 9, 10 (stp_tlp): term tables, no point source, compact or padded AoSoA
bool tlp_applicable(const LaunchPlan& p, const BatchArgs& a) {
  return (p.n == 9 || p.n == 10) && p.kind != ADERSTP_PDE_ELASTIC && p.kind != ADERSTP_PDE_ELASTIC_SOURCE &&
         p.src_comp < 0 && p.gen.t_ptr == nullptr && p.m >= 1 && p.m <= kTlpM &&
         p.layout == ADERSTP_LAYOUT_AOSOA && p.out_stride >= p.m && p.q_stride >= p.m && p.q_stride <= 64 &&
         p.n_terms <= kMaxTerms && !p.force_generic && !a.u_next;
}

// m <= 6 / m <= 8 / m = 9 instances: fewer threads leave more registers per thread (nDof 10:
// 608 / 800 / 928 threads)
cudaError_t launch_tlp(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  const int mq = p.m <= 6 ? 6 : p.m <= 8 ? 8 : 9;
  switch (p.n * 16 + mq) {
    case 9 * 16 + 6: return launch_tlp_n<9, 6>(p, a, stream);
    case 9 * 16 + 8: return launch_tlp_n<9, 8>(p, a, stream);
    case 9 * 16 + 9: return launch_tlp_n<9, 9>(p, a, stream);
    case 10 * 16 + 6: return launch_tlp_n<10, 6>(p, a, stream);
    case 10 * 16 + 8: return launch_tlp_n<10, 8>(p, a, stream);
    case 10 * 16 + 9: return launch_tlp_n<10, 9>(p, a, stream);
  }
  return cudaErrorInvalidValue;
}

bool pass_applicable(const LaunchPlan& p) {
  return p.n >= 2 && p.n <= 10 && p.kind == ADERSTP_PDE_ELASTIC && p.src_comp < 0 &&
         p.layout == ADERSTP_LAYOUT_AOSOA && p.out_stride == 9 && p.q_stride >= 9 && p.q_stride <= 64;
}

// Even/odd split of D (see the file comment), per order, into aderstp_kEO[n*64 ...].
cudaError_t init_pass(const LaunchPlan& p) {
  const int n = p.n, h = n / 2;
  double buf[80] = {0};
  const double* D = p.basis.d;
  for (int k = 0; k < h; ++k) {
    for (int l = 0; l < h; ++l) {
      buf[k * 6 + l] = 0.5 * (D[k * n + l] + D[k * n + (n - 1 - l)]);       // A
      buf[30 + k * 6 + l] = 0.5 * (D[k * n + l] - D[k * n + (n - 1 - l)]);  // B
    }
    if (n % 2) buf[k * 6 + h] = D[k * n + h];  // middle column acts on e[h] = p[h]
  }
  if (n % 2) {
    for (int l = 0; l < h; ++l) buf[60 + l] = 0.5 * (D[h * n + l] - D[h * n + (n - 1 - l)]);
    buf[60 + h] = D[h * n + h];
  }
  return cudaMemcpyToSymbol(aderstp_kEO, buf, sizeof(buf), sizeof(double) * 80 * n);
}

// the reference's own layout straight into the bipartite kernel (nDof 9, 10)
bool bip_aos_applicable(const LaunchPlan& p, const BatchArgs& a) {
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  return (p.n == 9 || p.n == 10) && p.kind == ADERSTP_PDE_ELASTIC && p.src_comp < 0 &&
         p.layout == ADERSTP_LAYOUT_AOS && p.q_stride == 16 && p.out_stride == 16 && !p.force_generic &&
         !p.aos_staged && p.pass_slots == 0 && !a.u_next && al16(a.q) && al16(a.qavg) && al16(a.favg);
}

bool bip_selected(const LaunchPlan& p, const BatchArgs& a) {
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  const bool vec_ok = (p.n % 2) || (al16(a.q) && al16(a.qavg) && al16(a.favg));
  return vec_ok && (p.n == 9 || p.n == 10) && (p.pass_slots == 12 || (p.pass_slots == 0 && p.n >= 9));
}

cudaError_t launch_bip(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  switch (p.n) {
    case 9: return launch_bip_n<9>(p, a, stream);
    case 10: return launch_bip_n<10>(p, a, stream);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_pass(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  // bipartite + TMEM kernel: the default for nDof 9 and 10 (ADERSTP_PASS_SLOTS=6 selects the
  // older line-pass kernel)
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  const bool vec_ok = (p.n % 2) || (al16(a.q) && al16(a.qavg) && al16(a.favg));  // 16-byte accesses
  if (vec_ok && (p.pass_slots == 12 || (p.pass_slots == 0 && p.n >= 9))) {
    switch (p.n) {
      case 9: return launch_bip_n<9>(p, a, stream);
      case 10: return launch_bip_n<10>(p, a, stream);
    }
  }
#define ADERSTP_PASS_CASE(NN) \
  case NN: return launch_pass_n<NN, 6>(p, a, stream);
  switch (p.n) {
    ADERSTP_PASS_CASE(2)
    ADERSTP_PASS_CASE(3)
    ADERSTP_PASS_CASE(4)
    ADERSTP_PASS_CASE(5)
    ADERSTP_PASS_CASE(6)
    ADERSTP_PASS_CASE(7)
    ADERSTP_PASS_CASE(8)
    ADERSTP_PASS_CASE(9)
    ADERSTP_PASS_CASE(10)
  }
#undef ADERSTP_PASS_CASE
  return cudaErrorInvalidValue;
}

}  // namespace aderstp
