// Elastic STP on the fp64 tensor cores for nDof 4..7: the stp_dmma8.cu scheme on zero-padded
// 8 x 8 (k2, k1) planes.  (The nDof 8 kernel is the unpadded special case; see that file for the
// full description.)
//
// One CTA = one element, 8 warps; lane (g, t) owns nodes (k2 = g, k1 = 2t, 2t+1) of every k3
// plane (k3 < N).  Rows and columns k2, k1 >= N and the rows/columns of D beyond N are exact
// zeros, so every 8x8x4 DMMA (x: A = p slice, B = c D^T; y: A = c D, B = p slice) produces exact
// zeros on the padding and the real nodes see exactly the N-term sums; N <= 4 needs a single
// k-step.  z contractions: register DFMA over the N planes with D from the constant cache.
// Roles (no redundant derivative fields): velocities (warps 0-2), shear (3, 6, 7), normal
// stresses on two k3 halves sharing Dx u, Dy v, Dz w (4, 5).  The CK series in Horner form (see
// stp_dmma8.cu).  Shared memory: r and q, 2 x 9 x N x 64 doubles, XOR-swizzled rows
// (bank-conflict free fragment loads).
#include <cstdint>
#include <type_traits>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"
#include "tmem.cuh"

// zero-padded 8 x 8 D per order (row k = node, col l), uploaded at plan creation
extern "C" {
__constant__ __align__(16) double aderstp_kDP[9 * 64];
#ifdef ADERSTP_EXPT_TIMING
__device__ long long aderstp_dbg_clock2[4096 * 8];
int aderstp_dbg_clock2_copy(long long* host, int count) {
  return (int)cudaMemcpyFromSymbol(host, aderstp_dbg_clock2, sizeof(long long) * count);
}
#define TM2(i) if (threadIdx.x == 0 && blockIdx.x < 4096) aderstp_dbg_clock2[blockIdx.x * 8 + (i)] = clock64()
#else
#define TM2(i)
#endif
}

#ifndef DMMAP_ODD_OUT
#define DMMAP_ODD_OUT 1
#endif
#ifndef DMMAP_MAXN
#define DMMAP_MAXN 7
#endif

namespace aderstp {

namespace {

constexpr int NVP = 9;
constexpr int NWP = 8;
constexpr int THREADSP = NWP * 32;

template <int N>
struct GeoP {
  // one quantity: N planes of 8 x 8, plus 6 doubles so that PV / 2 = 3 mod 8: the epilogue's
  // output-ordered 16-byte reads (k1 pair fastest, then the quantity) hit 8 distinct bank groups
  static constexpr int PV = N * 64 + 6;
  static constexpr int FACE = N * N * NVP;           // one face array
  static constexpr int SMEM = 2 * NVP * PV * 8;      // p + qavg accumulator
  static constexpr int KS = N > 4 ? 2 : 1;           // k-steps of 4
  static constexpr int H0 = (N + 1) / 2, H1 = N / 2; // normal-stress k3 halves
  // TMEM columns for q: 4N (lower warps) + max(12 H0, 4N) (upper warps), power of two >= 32
  static constexpr int TC = 4 * N + (12 * H0 > 4 * N ? 12 * H0 : 4 * N);
  static constexpr int TCOLS = TC <= 32 ? 32 : TC <= 64 ? 64 : 128;
};

struct ParamsP {
  double d[64];      // zero-padded D
  double phi[2][8];  // zero-padded phi(0), phi(1)
  double cf[8];      // cf[o] = dt^(o+1)/(o+1)! (Horner coefficients, stp_splitck.cpp:45,64)
  int check, par_kind, q_stride;
  int prefetch;      // L2 prefetch distance in elements (0: off)
};

// L2 prefetch of [ptr, ptr + bytes) rounded out to 16-byte bounds (cp.async.bulk.prefetch.L2)
__device__ __forceinline__ void prefetch_l2(const void* ptr, unsigned long long bytes) {
  const unsigned long long a0 = reinterpret_cast<unsigned long long>(ptr) & ~15ull;
  const unsigned long long a1 = (reinterpret_cast<unsigned long long>(ptr) + bytes + 15ull) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0), "r"((unsigned)(a1 - a0)) : "memory");
}


#ifdef DMMAP_ROLES_OLD
__constant__ int kRoleP[NWP] = {6, 7, 8, 4, -1, -2, 3, 5};
#else
// warps w and w + 4 share an SM sub-partition (and its fp64 / tensor pipe): per CK step at N = 6
// (16 cycles per DMMA, 2 per warp DFMA on a sub-partition) u, v, w cost 528, sxy 384, sxz and
// syz 336, the normal-stress halves 264 each; pairing (u, n0) (v, n1) (w, sxz) (sxy, syz) puts
// at most 864 on one sub-partition (the alternative pairing with sxy beside w: 912)
__constant__ int kRoleP[NWP] = {6, 7, 8, 3, -1, -2, 4, 5};
#endif
__constant__ int kInP[NVP][3] = {{6, 7, 8}, {6, 7, 8}, {6, 7, 8}, {7, 6, 0}, {8, 0, 6},
                                 {0, 8, 7}, {0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
__constant__ int kCoefP[NVP][3] = {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {2, 2, 4}, {2, 4, 2},
                                   {4, 2, 2}, {3, 3, 3}, {3, 3, 3}, {3, 3, 3}};

// e_in(s, d) (coef: e_coef) of the 9 output quantities packed 4 bits each, quantity s at bit 4 s
constexpr unsigned long long pack_flux(int d, bool coef) {
  unsigned long long v = 0;
  for (int s = 0; s < NVP; ++s) v |= (unsigned long long)(coef ? e_coef(s, d) : e_in(s, d)) << (4 * s);
  return v;
}

__device__ __forceinline__ double ldcp(const double* p) {
  double v;
  asm volatile("{\n .reg .u64 ca;\n cvta.to.const.u64 ca, %1;\n ld.const.f64 %0, [ca];\n}\n" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int physp(int k2, int k1) { return k2 * 8 + (k1 ^ ((k2 & 2) << 1)); }
__device__ __forceinline__ void dmmap(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double selp(const double c[4], int i) {
  return i == 0 ? c[0] : i == 1 ? c[1] : i == 2 ? c[2] : i == 3 ? c[3] : 0.0;
}
__device__ __forceinline__ double2 lds2p(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2p(double* p, double a, double b) {
  __builtin_assume(__isShared(p));
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// node pair (k1 = 2t, 2t+1) of an output row; one 16-byte streaming store when N is even (the
// pair is then 16-byte aligned), scalar stores otherwise
template <int N>
__device__ __forceinline__ void st_pair(double* p, double x, double y, bool ok0, bool ok1) {
  if (N % 2 == 0) {
    if (ok0) asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(x), "d"(y) : "memory");
  } else {
    if (ok0) __stcs(p, x);
    if (ok1) __stcs(p + 1, y);
  }
}

template <int N, int NT>
__device__ __forceinline__ void mma_xp(double (&acc)[NT][2], const double* f, int K0, int g, int t, double b0,
                                       double b1) {
  const double* p0 = f + K0 * 64 + physp(g, t);
  const double* p1 = f + K0 * 64 + physp(g, 4 + t);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    dmmap(acc[k][0], acc[k][1], p0[k * 64], b0);
    if (GeoP<N>::KS > 1) dmmap(acc[k][0], acc[k][1], p1[k * 64], b1);
  }
}

template <int N, int NT>
__device__ __forceinline__ void mma_yp(double (&acc)[NT][2], const double* f, int K0, int g, int t, double a0,
                                       double a1) {
  const double* p0 = f + K0 * 64 + physp(t, g);
  const double* p1 = f + K0 * 64 + physp(4 + t, g);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    dmmap(acc[k][0], acc[k][1], a0, p0[k * 64]);
    if (GeoP<N>::KS > 1) dmmap(acc[k][0], acc[k][1], a1, p1[k * 64]);
  }
}

// acc[k][j] += sum_{l<N} D[K0+k][l] (c f[l]) on the lane's two columns
template <int N, int NT>
__device__ __forceinline__ void dfma_zp(double (&acc)[NT][2], const double* f, int K0, int col, double c) {
  const double* dz = &aderstp_kDP[N * 64];
#pragma unroll
  for (int l = 0; l < N; ++l) {
    const double2 v = lds2p(f + l * 64 + col);
    const double c0 = c * v.x, c1 = c * v.y;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double dk = ldcp(dz + (K0 + k) * 8 + l);
      acc[k][0] = fma(dk, c0, acc[k][0]);
      acc[k][1] = fma(dk, c1, acc[k][1]);
    }
  }
}

// normal stresses on planes K0 .. K0+NT-1 from the iterate R: a = Dx u, b = Dy v, c = Dz w, then
// t_ii = lambda (a+b+c) + 2 mu {a,b,c}_i + co q_ii (Horner, see stp_dmma8.cu; q_ii from TMEM,
// 12 columns per plane at tq) -> W, the other buffer of the ping-pong pair.
// un (fused time-step mode): the step with co = 1 writes u_next = q + L(qavg) to HBM instead
template <int N, int NT>
__device__ __forceinline__ void normal_step(const double* R, double* W, uint32_t tq, int K0, int g, int t, int col,
                                            double d0, double d1, double lam, double two_mu, double co,
                                            double* un = nullptr, int uplane = 0) {
  constexpr int PV = GeoP<N>::PV;
  double ta[NT][2], tb[NT][2], tc[NT][2];
#pragma unroll
  for (int k = 0; k < NT; ++k) ta[k][0] = ta[k][1] = tb[k][0] = tb[k][1] = tc[k][0] = tc[k][1] = 0.0;
  mma_xp<N, NT>(ta, R + 6 * PV, K0, g, t, d0, d1);
  mma_yp<N, NT>(tb, R + 7 * PV, K0, g, t, d0, d1);
  dfma_zp<N, NT>(tc, R + 8 * PV, K0, col, 1.0);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    uint32_t r[12];
    tm_ld8(tq + 12 * k, r);
    tm_ld4(tq + 12 * k + 8, r + 8);
    tm_wait_ld();
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double sum = lam * (ta[k][j] + tb[k][j] + tc[k][j]);
      ta[k][j] = fma(co, tm_double(r, j), fma(two_mu, ta[k][j], sum));
      tb[k][j] = fma(co, tm_double(r, 2 + j), fma(two_mu, tb[k][j], sum));
      tc[k][j] = fma(co, tm_double(r, 4 + j), fma(two_mu, tc[k][j], sum));
    }
  }
  if (un) {  // fused: lane base un, uplane doubles per k3 plane of u_next
    if (g < N) {
      const bool ok0 = 2 * t < N, ok1 = 2 * t + 1 < N;
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        double* r = un + (K0 + k) * uplane;
        st_pair<N>(r, ta[k][0], ta[k][1], ok0, ok1);
        st_pair<N>(r + N, tb[k][0], tb[k][1], ok0, ok1);
        st_pair<N>(r + 2 * N, tc[k][0], tc[k][1], ok0, ok1);
      }
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const int off = (K0 + k) * 64 + col;
    sts2p(W + off, ta[k][0], ta[k][1]);
    sts2p(W + PV + off, tb[k][0], tb[k][1]);
    sts2p(W + 2 * PV + off, tc[k][0], tc[k][1]);
  }
}

// FUSED: the time-loop mode (BatchArgs::u_next), see stp_dmma8.cu.
// AOS: the reference's ElementTensor / PredictorOutput node rows [k3][k2][k1][s < 16] in and out
// (proj/src/layout.cpp:9-21): the node rows are first staged into the Q planes (real nodes only;
// the padding of Q is never read), qavg / favg leave as whole 128-byte node rows.
template <int N, bool FUSED = false, bool AOS = false>
__global__ void __maxnreg__(N <= 6 ? 64 : 80) stp_dmmap_kernel(ParamsP kp, BatchArgs a, unsigned int* status) {
  static_assert(!(FUSED && AOS), "the time loop runs on AoSoA");
  using G = GeoP<N>;
  constexpr int PV = G::PV, FACE = G::FACE;
  extern __shared__ __align__(16) double smq[];
  __shared__ uint32_t tmem_base_s;
  double* P = smq;              // c_(N-1) q (staging), then the Horner ping-pong pair (P, Q)
  double* Q = smq + NVP * PV;   // the other buffer of the Horner ping-pong pair
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int col = physp(g, 2 * t);
  unsigned int flags = 0;
  {
  const long long e = blockIdx.x;
  TM2(0);
  if (kp.prefetch && tid == 0 && e + kp.prefetch < a.n_elem)
    prefetch_l2(a.q + (e + kp.prefetch) * (long long)(N * N * N * kp.q_stride), 8ull * N * N * N * kp.q_stride);
  if (warp == 0) tm_alloc<G::TCOLS>(&tmem_base_s);
  double c4[4];
  {
    const double p0 = a.par[3 * e], p1 = a.par[3 * e + 1], p2 = a.par[3 * e + 2];
    double lam, mu, rho;
    if (kp.par_kind == ADERSTP_PAR_RHO_CP_CS) {
      rho = p0;
      mu = __dmul_rn(__dmul_rn(p0, p2), p2);
      lam = __dsub_rn(__dmul_rn(__dmul_rn(p0, p1), p1), __dmul_rn(2.0, mu));
    } else {
      lam = p0;
      mu = p1;
      rho = p2;
    }
    if (!((rho > 0.0) && (mu >= 0.0) && (lam + 2.0 * mu > 0.0))) flags |= 2u;
    c4[0] = lam + 2.0 * mu;
    c4[1] = lam;
    c4[2] = mu;
    c4[3] = 1.0 / rho;
  }

  const int role = kRoleP[warp];
  const double d0 = kp.d[g * 8 + t], d1 = kp.d[g * 8 + 4 + t];

  // ---- stage q straight into tensor memory and the first Horner iterate ---------------------
  // Every warp loads exactly the (quantity, k3) planes it keeps in TMEM -- role warps their
  // quantity on all N planes, the normal-stress warps sxx, syy, szz on their k3 half -- as the
  // node pair (k2 = g, k1 = 2t, 2t+1) of lane (g, t), i.e. in the C-fragment layout of the CK
  // step.  q goes register -> TMEM (thread-private columns: warps w and w + 4 share a lane
  // quarter, the upper four start at column 4N) and c_(N-1) q -> P, padding lanes writing the
  // zero padding; q never passes through shared memory.
  const bool ok0 = g < N && 2 * t < N, ok1 = g < N && 2 * t + 1 < N;
  const double* qe = a.q + e * (long long)(N * N * N * kp.q_stride);
  if constexpr (AOS) {  // node rows -> Q planes (5 slot pairs per node; slot 9 is padding)
    const double* qn = a.q + e * (long long)(N * N * N * 16);
    for (int i = tid; i < N * N * N * 5; i += THREADSP) {
      const int node = i / 5, sp = 2 * (i - node * 5), k1 = node % N, k32 = node / N;
      const double2 v = __ldcs(reinterpret_cast<const double2*>(qn + node * 16 + sp));
      const int j = sp * PV + (k32 / N) * 64 + physp(k32 % N, k1);
      Q[j] = v.x;
      if (sp < 8) Q[j + PV] = v.y;
    }
    __syncthreads();
  }
  // nDof 7, AoSoA: rows of N doubles are not 16-byte pairs, and lane-wise 8-byte loads of the
  // C-fragment positions scatter; the element's q is staged into the Q planes with coalesced
  // loads (consecutive threads = consecutive doubles of [k3][k2][s][k1], slots s >= 9 skipped)
  constexpr bool STAGEQ = AOS || N == 7;  // measured: nDof 7 +2.9 %, nDof 5 -1.2 %
  if constexpr (!AOS && N == 7) {
    const int qs = kp.q_stride;
    const int rowl = qs * N;  // one (k3, k2) row group: qs quantities x N nodes
    for (int i = tid; i < N * N * rowl; i += THREADSP) {
      const int k32 = i / rowl, rem = i - k32 * rowl, sq = rem / N, k1 = rem - sq * N;
      if (sq < NVP) Q[sq * PV + (k32 / N) * 64 + physp(k32 % N, k1)] = __ldcs(qe + i);
    }
    __syncthreads();
  }
  auto ldq = [&](int sq, int k3, double& v0, double& v1) {
    if constexpr (STAGEQ) {  // from the staged planes (C-fragment positions, padding lanes: 0)
      const double* src = Q + sq * PV + k3 * 64 + col;
      v0 = ok0 ? src[0] : 0.0;
      v1 = ok1 ? src[1] : 0.0;
      return;
    }
    const double* src = qe + ((k3 * N + g) * kp.q_stride + sq) * N + 2 * t;
    if (N % 2 == 0) {  // 16-byte aligned pair (q_stride * N even)
      double2 v = ok0 ? __ldcs(reinterpret_cast<const double2*>(src)) : make_double2(0.0, 0.0);
      v0 = v.x;
      v1 = v.y;
    } else {
      v0 = ok0 ? __ldcs(src) : 0.0;
      v1 = ok1 ? __ldcs(src + 1) : 0.0;
    }
  };
  tm_fence_before();
  __syncthreads();  // the TMEM base address (warp 0's tcgen05.alloc) is visible
  tm_fence_after();
  const uint32_t tq = tmem_base_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp < 4 ? 0 : 4 * N);
  {  // each plane: load, check, c_(n-1) q -> P, q -> TMEM (the compiler batches the loads ahead)
    const double c0 = kp.cf[N - 1];
    if (role >= 0) {
#pragma unroll
      for (int k3 = 0; k3 < N; ++k3) {
        double v0, v1;
        ldq(role, k3, v0, v1);
        if (kp.check && !(isfinite(v0) && isfinite(v1))) flags |= 1u;
        sts2p(P + role * PV + k3 * 64 + col, c0 * v0, c0 * v1);
        uint32_t r[4];
        tm_split(v0, r, 0);
        tm_split(v1, r, 1);
        tm_st4(tq + 4 * k3, r);
      }
    } else {
      const int h = -role - 1, K0 = h ? G::H0 : 0, NT = h ? G::H1 : G::H0;
#pragma unroll
      for (int k = 0; k < G::H0; ++k) {
        if (k >= NT) break;
        uint32_t r[12];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          double v0, v1;
          ldq(j, K0 + k, v0, v1);
          if (kp.check && !(isfinite(v0) && isfinite(v1))) flags |= 1u;
          sts2p(P + j * PV + (K0 + k) * 64 + col, c0 * v0, c0 * v1);
          tm_split(v0, r, 2 * j);
          tm_split(v1, r, 2 * j + 1);
        }
        tm_st8(tq + 12 * k, r);
        tm_st4(tq + 12 * k + 8, r + 8);
      }
    }
    tm_wait_st();
    __syncthreads();  // P = c_(N-1) q complete; Q takes the first Horner iterate
  }
  TM2(1);

  // ---- CK series in Horner form (stp_dmma8.cu): r <- c_o q + L r, o = N-2 .. 0 ----------
  // step i reads buffer i % 2 and writes (i + 1) % 2: 0 = P (c_(N-1) q), 1 = Q; one barrier
  // per step.  The Horner term c_o q (TMEM) initialises the accumulators.
  if (role >= 0) {
    const int s = role;
    const int in_x = kInP[s][0], in_y = kInP[s][1], in_z = kInP[s][2];
    const double cx = selp(c4, kCoefP[s][0]), cy = selp(c4, kCoefP[s][1]), cz = selp(c4, kCoefP[s][2]);
    const bool has_x = kCoefP[s][0] != 4, has_y = kCoefP[s][1] != 4, has_z = kCoefP[s][2] != 4;
    const double bx0 = cx * d0, bx1 = cx * d1, ay0 = cy * d0, ay1 = cy * d1;
    const int own = s * PV + col;
    constexpr int o_end = FUSED ? -1 : 0;
#pragma unroll 1
    for (int o = N - 2, i = 0; o >= o_end; --o, ++i) {
      const double co = (!FUSED || o >= 0) ? kp.cf[o] : 1.0;
      const double* R = smq + (i & 1) * (NVP * PV);
      double tt[N][2];
      {  // two halves of the planes per TMEM round trip
        constexpr int HA = (N + 1) / 2;
        uint32_t r[4 * HA];
#pragma unroll
        for (int k3 = 0; k3 < HA; ++k3) tm_ld4(tq + 4 * k3, r + 4 * k3);
        tm_wait_ld();
#pragma unroll
        for (int k3 = 0; k3 < HA; ++k3) {
          tt[k3][0] = co * tm_double(r + 4 * k3, 0);
          tt[k3][1] = co * tm_double(r + 4 * k3, 1);
        }
#pragma unroll
        for (int k3 = HA; k3 < N; ++k3) tm_ld4(tq + 4 * k3, r + 4 * (k3 - HA));
        tm_wait_ld();
#pragma unroll
        for (int k3 = HA; k3 < N; ++k3) {
          tt[k3][0] = co * tm_double(r + 4 * (k3 - HA), 0);
          tt[k3][1] = co * tm_double(r + 4 * (k3 - HA), 1);
        }
      }
      if (has_x) mma_xp<N, N>(tt, R + in_x * PV, 0, g, t, bx0, bx1);
      if (has_y) mma_yp<N, N>(tt, R + in_y * PV, 0, g, t, ay0, ay1);
      if (has_z) dfma_zp<N, N>(tt, R + in_z * PV, 0, col, cz);
      if (FUSED && o < 0) {  // u_next = q + L(qavg): the corrector's volume term, straight to HBM
        if (g < N) {
          const int qs = kp.q_stride;
          double* un = a.u_next + e * (long long)(N * N * N * qs) + (g * qs + s) * N + 2 * t;
#pragma unroll
          for (int k3 = 0; k3 < N; ++k3)
            st_pair<N>(un + k3 * N * qs * N, tt[k3][0], tt[k3][1], 2 * t < N, 2 * t + 1 < N);
        }
        break;
      }
      double* W = smq + ((i + 1) & 1) * (NVP * PV);
#pragma unroll
      for (int k3 = 0; k3 < N; ++k3) sts2p(W + own + k3 * 64, tt[k3][0], tt[k3][1]);
      __syncthreads();
    }
  } else {
    const int h = -role - 1;
    const double lam = c4[1], two_mu = 2.0 * c4[2];
#pragma unroll 1
    for (int o = N - 2, i = 0; o >= 0; --o, ++i) {
      const double co = kp.cf[o];
      if (h == 0) normal_step<N, G::H0>(smq + (i & 1) * (NVP * PV), smq + ((i + 1) & 1) * (NVP * PV), tq, 0, g, t, col, d0, d1, lam, two_mu, co);
      else normal_step<N, G::H1>(smq + (i & 1) * (NVP * PV), smq + ((i + 1) & 1) * (NVP * PV), tq, G::H0, g, t, col, d0, d1, lam, two_mu, co);
      __syncthreads();
    }
    if (FUSED) {
      const int qs = kp.q_stride;
      double* un = a.u_next + e * (long long)(N * N * N * qs) + g * qs * N + 2 * t;
      const double* R = smq + ((N - 1) & 1) * (NVP * PV);
      if (h == 0) normal_step<N, G::H0>(R, nullptr, tq, 0, g, t, col, d0, d1, lam, two_mu, 1.0, un, N * qs * N);
      else normal_step<N, G::H1>(R, nullptr, tq, G::H0, g, t, col, d0, d1, lam, two_mu, 1.0, un, N * qs * N);
    }
  }
  // every TMEM read has completed (tcgen05.wait::ld); the allocating warp frees the columns
  tm_fence_before();
  __syncthreads();
  if (warp == 0) {
    tm_fence_after();
    tm_dealloc<G::TCOLS>(tmem_base_s);
  }
  P = smq + ((N - 1) & 1) * (NVP * PV);  // qavg: the last Horner iterate
  Q = smq + (N & 1) * (NVP * PV);        // free: the face staging buffer

  TM2(2);
  // ---- epilogue: 9 quantities x k3 planes over the 8 warps ------------------------------
  double* FQ = Q;  // face staging [6][N][N][9] over the dead q buffer
  const bool faces = a.face_q || a.face_f;
  const double bphi0 = (g < 2) ? kp.phi[g][t] : 0.0;
  const double bphi1 = (g < 2) ? kp.phi[g][4 + t] : 0.0;
  const bool rowok = g < N;
  const bool k1a = 2 * t < N, k1b = 2 * t + 1 < N;
  // qavg / favg: warp w emits the k3 planes w, w + 8, ...; the plane's 9 quantities are read
  // once and every output row (9 qavg, 27 favg = F_d(qavg)) is stored with compile-time indices
  if constexpr (AOS) {
    // node rows: lane = (node ns of 4, slot pair c2), 4 x 128 contiguous bytes per instruction
    const int ns = lane >> 3, c2 = 2 * (lane & 7);
    int srcq[3][2];
    double cfo[3][2];
    bool val[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int so = c2 + j;
      val[j] = so < NVP;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int ci = val[j] ? e_coef(so, d) : 4;
        srcq[d][j] = val[j] ? e_in(so, d) : 0;
        cfo[d][j] = ci == 4 ? 0.0 : selp(c4, ci);
      }
    }
    constexpr int N3 = N * N * N;
    double* qo = a.qavg + e * (long long)(N3 * 16);
    double* fo = a.favg ? a.favg + e * (long long)(3 * N3 * 16) : nullptr;
#pragma unroll 1
    for (int nb = 4 * warp + ns; nb < N3; nb += 4 * NWP) {
      const int k32 = nb / N, pos = (k32 / N) * 64 + physp(k32 % N, nb % N);
      __stcs(reinterpret_cast<double2*>(qo + nb * 16 + c2),
             make_double2(val[0] ? P[c2 * PV + pos] : 0.0, val[1] ? P[(c2 + 1) * PV + pos] : 0.0));
      if (fo) {
#pragma unroll
        for (int d = 0; d < 3; ++d)
          __stcs(reinterpret_cast<double2*>(fo + d * (N3 * 16) + nb * 16 + c2),
                 make_double2(cfo[d][0] != 0.0 ? cfo[d][0] * P[srcq[d][0] * PV + pos] : 0.0,
                              cfo[d][1] != 0.0 ? cfo[d][1] * P[srcq[d][1] * PV + pos] : 0.0));
      }
    }
  } else {
    double* qout = FUSED ? nullptr : a.qavg + e * (long long)(N * N * N * NVP);
    double* fout = a.favg ? a.favg + e * (long long)(3 * N * N * N * NVP) : nullptr;
#if DMMAP_ODD_OUT
    if constexpr (N == 7) {
      // nDof 7: rows of 7 doubles give only scattered 8-byte stores in the plane-per-warp scheme;
      // every output array is written in its own order by all warps instead (consecutive lanes
      // store consecutive doubles), each value read from the planes (favg: flux source x coef).
      // Measured: nDof 7 +8.7 %, nDof 5 -10 % (kept plane-per-warp)
      constexpr int N3 = N * N * N, UNITS = NVP * N3;
      constexpr unsigned long long IN[3] = {pack_flux(0, false), pack_flux(1, false), pack_flux(2, false)};
      constexpr unsigned long long CO[3] = {pack_flux(0, true), pack_flux(1, true), pack_flux(2, true)};
#pragma unroll 1
      for (int u = tid; u < UNITS; u += THREADSP) {
        const int k1 = u % N, r1 = u / N, so = r1 % NVP, r2 = r1 / NVP, k2 = r2 % N, k3 = r2 / N;
        const double* pl = P + k3 * 64 + physp(k2, k1);
        if (qout) __stcs(qout + u, pl[so * PV]);
        if (fout) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const int src = (int)((IN[d] >> (4 * so)) & 15), ci = (int)((CO[d] >> (4 * so)) & 15);
            const double c = ci == 0 ? c4[0] : ci == 1 ? c4[1] : ci == 2 ? c4[2] : ci == 3 ? c4[3] : 0.0;
            __stcs(fout + d * UNITS + u, c * pl[src * PV]);
          }
        }
      }
    } else
#endif
#pragma unroll 1
    for (int k3 = warp; k3 < N; k3 += NWP) {
      double2 v[NVP];
#pragma unroll
      for (int s = 0; s < NVP; ++s) v[s] = lds2p(P + s * PV + k3 * 64 + col);
      if (rowok) {
        const int base = (k3 * N + g) * NVP * N + 2 * t;
        if (!FUSED) {
#pragma unroll
          for (int s = 0; s < NVP; ++s) st_pair<N>(qout + base + s * N, v[s].x, v[s].y, k1a, k1b);
        }
        if (fout) {
#pragma unroll
          for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int so = 0; so < NVP; ++so) {
              const int ci = e_coef(so, d), si = e_in(so, d);
              const double c = ci == 4 ? 0.0 : c4[ci & 3];
              st_pair<N>(fout + d * (N * N * N * NVP) + base + so * N, ci == 4 ? 0.0 : c * v[si].x,
                         ci == 4 ? 0.0 : c * v[si].y, k1a, k1b);
            }
        }
      }
    }
  }
  TM2(3);
  if (faces) {
    // Face extrapolations as line tasks over all 8 warps (FMAs; a DMMA against phi would use 2
    // of its 8 output columns): task (direction, line, quantity) reads its line of the padded
    // qavg planes (16-byte pairs where the line runs along k1) and writes both sides; the
    // quantity is the fastest task index, so 8 consecutive lanes read 8 distinct bank groups
    // (PV / 2 = 3 mod 8) and store consecutive face entries.
    {
      constexpr int KP = (N + 1) / 2;            // k1 pairs (the last one half padding for odd N)
      constexpr int TX = N * N * NVP, TY = N * KP * NVP;
      for (int i = tid; i < TX + 2 * TY; i += THREADSP) {
        if (i < TX) {  // x: row (k3, k2) of quantity s
          const int s = i % NVP, r = i / NVP, k2 = r % N, k3 = r / N;
          const double* row = P + s * PV + k3 * 64 + k2 * 8;
          double f0 = 0.0, f1 = 0.0;
#pragma unroll
          for (int k = 0; k < KP; ++k) {
            const double2 v = lds2p(row + ((2 * k) ^ ((k2 & 2) << 1)));
            f0 = fma(kp.phi[0][2 * k], v.x, f0);
            f1 = fma(kp.phi[1][2 * k], v.x, f1);
            if (2 * k + 1 < N) {
              f0 = fma(kp.phi[0][2 * k + 1], v.y, f0);
              f1 = fma(kp.phi[1][2 * k + 1], v.y, f1);
            }
          }
          FQ[0 * FACE + (k3 * N + k2) * NVP + s] = f0;
          FQ[1 * FACE + (k3 * N + k2) * NVP + s] = f1;
        } else {  // y: column pair (k3, k1 = 2 kp, 2 kp + 1) over k2; z: (k2, k1 pair) over k3
          const bool ydir = i < TX + TY;
          const int j = i - (ydir ? TX : TX + TY);
          const int s = j % NVP, r = j / NVP, kq = r % KP, a0 = r / KP;
          double f0[2] = {0.0, 0.0}, f1[2] = {0.0, 0.0};
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const double2 v = ydir ? lds2p(P + s * PV + a0 * 64 + physp(k, 2 * kq)) : lds2p(P + s * PV + k * 64 + physp(a0, 2 * kq));
            f0[0] = fma(kp.phi[0][k], v.x, f0[0]);
            f0[1] = fma(kp.phi[0][k], v.y, f0[1]);
            f1[0] = fma(kp.phi[1][k], v.x, f1[0]);
            f1[1] = fma(kp.phi[1][k], v.y, f1[1]);
          }
          const int fb = ydir ? 2 : 4;
          const int o = (a0 * N + 2 * kq) * NVP + s;
          FQ[fb * FACE + o] = f0[0];
          FQ[(fb + 1) * FACE + o] = f1[0];
          if (2 * kq + 1 < N) {
            FQ[fb * FACE + o + NVP] = f0[1];
            FQ[(fb + 1) * FACE + o + NVP] = f1[1];
          }
        }
      }
    }
    // face_q is complete and leaves at once (TMA bulk store, UBLKCP), overlapping the face_f pass
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0 && a.face_q) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                       a.face_q + e * (long long)(6 * FACE)),
                   "r"((unsigned)__cvta_generic_to_shared(FQ)), "r"((unsigned)(6 * FACE * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    TM2(4);
    // face_f = F_d(face_q) staged over qavg; it leaves as a second bulk store.
    // Thread = (face f, in-face node ab): 9 loads, 9 stores, compile-time flux per direction.
    double* FF = P;  // qavg (P) is no longer read
    if (a.face_f) {
#pragma unroll 1
      for (int i = tid; i < 6 * N * N; i += THREADSP) {
        const int f = i / (N * N), d = f >> 1;
        const double* src = FQ + f * FACE + (i - f * N * N) * NVP;
        double* dst = FF + f * FACE + (i - f * N * N) * NVP;
        double v[NVP];
#pragma unroll
        for (int s = 0; s < NVP; ++s) v[s] = src[s];
        auto emit = [&](auto dd) {
          constexpr int D = decltype(dd)::value;
#pragma unroll
          for (int so = 0; so < NVP; ++so) {
            const int ci = e_coef(so, D);
            dst[so] = ci == 4 ? 0.0 : c4[ci & 3] * v[e_in(so, D)];
          }
        };
        if (d == 0) emit(std::integral_constant<int, 0>{});
        else if (d == 1) emit(std::integral_constant<int, 1>{});
        else emit(std::integral_constant<int, 2>{});
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      const unsigned bytes = 6 * FACE * 8;
      if (a.face_f)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                         a.face_f + e * (long long)(6 * FACE)),
                     "r"((unsigned)__cvta_generic_to_shared(FF)), "r"(bytes)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
  }
  }
  if (kp.check && flags) atomicOr(status, flags);
  TM2(5);
}

template <int N>
cudaError_t launch_dmmap_n(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  using G = GeoP<N>;
  ParamsP kp;
  for (int i = 0; i < 64; ++i) kp.d[i] = 0.0;
  for (int k = 0; k < N; ++k)
    for (int l = 0; l < N; ++l) kp.d[k * 8 + l] = p.basis.d[k * N + l];
  for (int j = 0; j < 8; ++j) {
    kp.phi[0][j] = j < N ? p.basis.face_left[j] : 0.0;
    kp.phi[1][j] = j < N ? p.basis.face_right[j] : 0.0;
  }
  kp.check = p.check;
  kp.par_kind = p.par_kind;
  kp.q_stride = p.q_stride;
  kp.prefetch = p.dmma8_prefetch;
  {
    double c = a.dt;  // same operation sequence as proj/src/stp_splitck.cpp:45,64
    kp.cf[0] = c;
    for (int o = 1; o < 8; ++o) {
      c *= a.dt / (o + 1);
      kp.cf[o] = c;
    }
  }
  auto kern = a.u_next ? stp_dmmap_kernel<N, true> : p.layout == ADERSTP_LAYOUT_AOS ? stp_dmmap_kernel<N, false, true>
                                                                                    : stp_dmmap_kernel<N, false>;
  const int smem = G::SMEM;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  if (a.n_elem == 0) return cudaSuccess;
  if (a.n_elem > 0x7fffffffLL) return cudaErrorInvalidValue;
  const long long grid = a.n_elem;
  kern<<<(unsigned)grid, THREADSP, smem, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}

}  // namespace

bool dmmap_applicable(const LaunchPlan& p) {
  return p.n >= 4 && p.n <= DMMAP_MAXN && p.kind == ADERSTP_PDE_ELASTIC && p.src_comp < 0 &&
         p.layout == ADERSTP_LAYOUT_AOSOA && p.out_stride == 9 && p.q_stride >= 9 && p.q_stride <= 64;
}

// the reference's own layout straight into the padded-DMMA kernel (nDof 4..7)
bool dmmap_aos_applicable(const LaunchPlan& p, const BatchArgs& a) {
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  return p.n >= 4 && p.n <= DMMAP_MAXN && p.kind == ADERSTP_PDE_ELASTIC && p.src_comp < 0 &&
         p.layout == ADERSTP_LAYOUT_AOS && p.q_stride == 16 && p.out_stride == 16 && !p.force_generic &&
         !p.no_dmmap && !p.aos_staged && !a.u_next && al16(a.q) && al16(a.qavg) && al16(a.favg) &&
         al16(a.face_q) && al16(a.face_f);
}

cudaError_t init_dmmap(const LaunchPlan& p) {
  double buf[64] = {0};
  for (int k = 0; k < p.n; ++k)
    for (int l = 0; l < p.n; ++l) buf[k * 8 + l] = p.basis.d[k * p.n + l];
  return cudaMemcpyToSymbol(aderstp_kDP, buf, sizeof(buf), sizeof(double) * 64 * p.n);
}

cudaError_t launch_dmmap(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  switch (p.n) {
    case 4: return launch_dmmap_n<4>(p, a, stream);
    case 5: return launch_dmmap_n<5>(p, a, stream);
    case 6: return launch_dmmap_n<6>(p, a, stream);
    case 7: return launch_dmmap_n<7>(p, a, stream);
#if DMMAP_MAXN >= 8
    case 8: return launch_dmmap_n<8>(p, a, stream);
#endif
  }
  return cudaErrorInvalidValue;
}

}  // namespace aderstp
