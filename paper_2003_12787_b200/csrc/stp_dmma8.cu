// nDof = 8 elastic STP kernel on the fp64 tensor cores (sm_100a DMMA, mma.sync m8n8k4 f64).
//
// One CTA = one element, 8 warps.  Lane (g = lane/4, t = lane%4) of a warp owns node pairs
// (k2 = g, k1 = 2t, 2t+1) -- exactly the C-fragment of an 8x8 MMA tile C[k2][k1] at fixed k3 --
// so the three 1-D contractions of a CK step are
//   x:  C[k2][k1] += sum_l P[k3][k2][l] (cD)[k1][l]    DMMA, A = p slice (smem), B = c D^T
//   y:  C[k2][k1] += sum_l (cD)[k2][l] P[k3][l][k1]    DMMA, A = c D,            B = p slice
//   z:  C[k3]     += sum_l D[k3][l] (c p)[l]            DFMA on the lane's own columns, D from
//                                                        the constant cache
// all accumulating into the same registers.  The elastic system (proj/src/pde.cpp:180-218)
// needs 18 derivative fields per step; the warps split them with no redundancy:
//   warps 4, 5  normal stresses (sxx, syy, szz) on k3 half h: a = Dx u, b = Dy v, c = Dz w,
//               t_ii = lambda (a + b + c) + 2 mu {a, b, c}_i
//   warps 3,6,7 shear sxz, sxy, syz:  mu (Dx w + Dz u), mu (Dx v + Dy u), mu (Dy w + Dz v)
//   warps 0-2   velocities u, v, w:   (1/rho) (Dx s_x. + Dy s_y. + Dz s_z.)
// paired on the SM sub-partitions (warp % 4) so that every SMSP carries about the same fp64 work.
// Flux-first exactly like the reference's D_d * F_d(p) (proj/src/stp_splitck.cpp:53-55).
//
// The series is evaluated in Horner form (see ck_quantity below).
//
// Shared memory (73,728 B, 3 CTAs per SM): the Horner iterate r and q, each 9 x 8 x 8 x 8 fp64
// with an XOR swizzle on k1 (bit 2 flipped on rows with k2 & 2) that makes every fragment load,
// column load and store bank-conflict free.  Epilogue: qavg and favg go out from registers
// (st.global.cs, 64-byte segments); the 12 face arrays are contracted by DMMA (x, y normals) and
// DFMA (z normal) from qavg, staged in the reference's [f][a][b][s] order and leave as TMA bulk
// stores, face_f = F_d(face_q).
#include <cstdint>
#include <type_traits>
#include <cstdlib>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"

// D of the nDof = 8 Gauss-Legendre basis (the same for every plan), uploaded once per device.
// The z-contraction reads it at the point of use through volatile ld.const (constant cache,
// broadcast), so ptxas cannot hoist 64 doubles of D into registers and spill.
extern "C" {
__constant__ __align__(16) double aderstp_kD8[64];
#ifdef ADERSTP_EXPT_TIMING
__device__ long long aderstp_dbg_clock3[4096 * 8];
int aderstp_dbg_clock3_copy(long long* host, int count) {
  return (int)cudaMemcpyFromSymbol(host, aderstp_dbg_clock3, sizeof(long long) * count);
}
#define TM3(i) if (threadIdx.x == 0 && blockIdx.x < 4096) aderstp_dbg_clock3[blockIdx.x * 8 + (i)] = clock64()
#else
#define TM3(i)
#endif
}

namespace aderstp {

namespace {

constexpr int N8 = 8;
constexpr int NV = 9;
constexpr int NWARP = 8;  // default CTA: 8 warps, 3 CTAs/SM
constexpr int PV = N8 * N8 * N8;    // doubles per quantity plane
constexpr int FACE = N8 * N8 * NV;  // doubles per face array (576)
// r and q, 73,728 B: 3 CTAs/SM, two barriers per CK step.
#ifndef D8_FPAD
#define D8_FPAD 8
#endif
constexpr int kSmem8 = 2 * NV * (PV + 8) * 8;
// staged face arrays [6][64][9], FACES doubles apart (FACE + 8: the y-face stores of lanes g = 0, 1
// fall on different banks); they leave as one bulk copy per face
constexpr int FACES = FACE + D8_FPAD;

struct Params8 {
  double d[64];      // d[k*8+l] = phi_l'(x_k)
  double phi[2][8];  // phi(0), phi(1)
  double cf[8];      // cf[o] = dt^(o+1)/(o+1)!, the reference's running coefficient
  int check;
  int par_kind;
  int q_stride;
  int prefetch;  // element distance of the L2 prefetch (0: off)
  // volume mode (the corrector's volume term, solver.cpp:199-207): the iterate starts from r_src
  // (qavg, compact AoSoA) instead of c_(n-1) q and only the coefficient-1 step runs (o_start = -1)
  const double* r_src;
  int o_start;
};

// role of each warp: a single output quantity (0..8), or -1 / -2 for the normal-stress warps on
// k3 half 0 / 1.  SMSP pairs (w, w+4): {u, N0}, {v, N1}, {w, sxy}, {sxz, syz}.
__constant__ int kRole[NWARP] = {6, 7, 8, 4, -1, -2, 3, 5};
// epilogue units (quantity s, k3 half h) -> unit id 2s + h, per warp, balanced by cost (favg
// stores 1/3/5 planes per unit, z faces on h = 0): the natural round-robin put three z-face
// units on warp 0 (cost model 318 vs 204 for this table, ideal 189)
__constant__ int kUnits[NWARP][3] = {{5, 11, 1}, {16, 13, -1}, {12, 15, -1}, {2, 8, -1},
                                     {10, 0, -1}, {4, 6, -1}, {7, 17, 3}, {14, 9, -1}};
// elastic flux table F_d(q)_s = coef(s,d) q[in(s,d)]; coef 0: lambda+2mu, 1: lambda, 2: mu,
// 3: 1/rho, 4: 0
__constant__ int kIn[NV][3] = {{6, 7, 8}, {6, 7, 8}, {6, 7, 8}, {7, 6, 0}, {8, 0, 6},
                               {0, 8, 7}, {0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
__constant__ int kCoef[NV][3] = {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {2, 2, 4}, {2, 4, 2},
                                 {4, 2, 2}, {3, 3, 3}, {3, 3, 3}, {3, 3, 3}};
// outgoing flux entries of each source quantity r: (s, d, coef) with in(s,d) = r, plus the three
// identically-zero entries (coef 4) assigned to the shear quantities.  Used for favg.
__constant__ int kOutN[NV] = {1, 1, 1, 3, 3, 3, 5, 5, 5};
__constant__ int kOut[NV][5][3] = {
    {{6, 0, 3}}, {{7, 1, 3}}, {{8, 2, 3}},
    {{6, 1, 3}, {7, 0, 3}, {3, 2, 4}},
    {{6, 2, 3}, {8, 0, 3}, {4, 1, 4}},
    {{7, 2, 3}, {8, 1, 3}, {5, 0, 4}},
    {{0, 0, 0}, {1, 0, 1}, {2, 0, 1}, {3, 1, 2}, {4, 2, 2}},
    {{0, 1, 1}, {1, 1, 0}, {2, 1, 1}, {3, 0, 2}, {5, 2, 2}},
    {{0, 2, 1}, {1, 2, 1}, {2, 2, 0}, {4, 0, 2}, {5, 1, 2}}};

__device__ __forceinline__ double2 ldc2(const double* p) {
  double2 v;
  asm volatile("{\n .reg .u64 ca;\n cvta.to.const.u64 ca, %2;\n ld.const.v2.f64 {%0, %1}, [ca];\n}\n"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ int phys(int k2, int k1) { return k2 * 8 + (k1 ^ ((k2 & 2) << 1)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double sel4(const double c[4], int i) {
  return i == 0 ? c[0] : i == 1 ? c[1] : i == 2 ? c[2] : i == 3 ? c[3] : 0.0;
}

__device__ __forceinline__ void st_cs2(double* p, double a, double b) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(a), "d"(b) : "memory");
}

__device__ __forceinline__ double2 ld_nc2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// acc[K][j] += x-contraction of field f over tiles k3 = K0 .. K0+NT-1 (B = scaled D^T frags)
template <int NT>
__device__ __forceinline__ void mma_x(double (&acc)[NT][2], const double* f, int K0, int g, int t,
                                      double b0, double b1) {
  const double* p0 = f + K0 * 64 + phys(g, t);
  const double* p1 = f + K0 * 64 + phys(g, 4 + t);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    dmma(acc[k][0], acc[k][1], p0[k * 64], b0);
    dmma(acc[k][0], acc[k][1], p1[k * 64], b1);
  }
}

// acc[K][j] += y-contraction (A = scaled D frags)
template <int NT>
__device__ __forceinline__ void mma_y(double (&acc)[NT][2], const double* f, int K0, int g, int t,
                                      double a0, double a1) {
  const double* p0 = f + K0 * 64 + phys(t, g);
  const double* p1 = f + K0 * 64 + phys(4 + t, g);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    dmma(acc[k][0], acc[k][1], a0, p0[k * 64]);
    dmma(acc[k][0], acc[k][1], a1, p1[k * 64]);
  }
}

// acc[K][j] += sum_l D[K0+K][l] * (c f[l]) on this lane's two columns (full column l = 0..7)
template <int NT>
__device__ __forceinline__ void dfma_z(double (&acc)[NT][2], const double* f, int K0, int col, double c) {
  const double* pz = f + col;
#pragma unroll
  for (int lq = 0; lq < 4; ++lq) {
    const double2 v0 = lds2(pz + (2 * lq) * 64);
    const double2 v1 = lds2(pz + (2 * lq + 1) * 64);
    const double c00 = c * v0.x, c01 = c * v1.x, c10 = c * v0.y, c11 = c * v1.y;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double2 dk = ldc2(&aderstp_kD8[(K0 + k) * 8 + 2 * lq]);
      acc[k][0] = fma(dk.x, c00, acc[k][0]);
      acc[k][1] = fma(dk.x, c10, acc[k][1]);
      acc[k][0] = fma(dk.y, c01, acc[k][0]);
      acc[k][1] = fma(dk.y, c11, acc[k][1]);
    }
  }
}


// The CK series qavg = sum_o c_o L^o q (c_o = dt^(o+1)/(o+1)!, L q = sum_d D_d F_d(q)) evaluated
// in Horner form, r <- c_o q + L r for o = n-2 .. 0 from r = c_(n-1) q: the same n-1 applications
// of L as the reference's forward recursion (proj/src/stp_splitck.cpp:46-70), but each step reads
// the constant q instead of read-modify-writing a qavg accumulator -- 20% less shared-memory
// traffic, which is what bounds this kernel.  P holds r (updated in place between two barriers),
// Q holds q.

// One Horner step loop for output quantity s on k3 tiles K0 .. K0+NT-1.
// un (fused time-step mode, else null): this lane's base in the next state u_next; one more step
// with coefficient 1 then gives u_next = q + L(qavg) (the corrector's volume term) in registers
// and goes straight to HBM.  urow = doubles per (k3, k2) row of u_next.
template <int NT, bool FUSED, int PS>
__device__ __forceinline__ void ck_quantity(double* P, const double* Q, const double* cf, int s, int K0, int g,
                                            int t, int col, double d0, double d1, const double (&c4)[4],
                                            double* un, int urow, int o_start) {
  const int in_x = kIn[s][0], in_y = kIn[s][1], in_z = kIn[s][2];
  const double cx = sel4(c4, kCoef[s][0]), cy = sel4(c4, kCoef[s][1]), cz = sel4(c4, kCoef[s][2]);
  const bool has_x = kCoef[s][0] != 4, has_y = kCoef[s][1] != 4, has_z = kCoef[s][2] != 4;
  const double bx0 = cx * d0, bx1 = cx * d1;  // B-fragments of c_x D^T
  const double ay0 = cy * d0, ay1 = cy * d1;  // A-fragments of c_y D
  const int own = s * PS + K0 * 64 + col;
  constexpr int o_end = FUSED ? -1 : 0;
#pragma unroll 1
  for (int o = o_start; o >= o_end; --o) {
    const double co = (!FUSED || o >= 0) ? cf[o] : 1.0;
    double tt[NT][2];
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double2 v = lds2(Q + own + k * 64);
      tt[k][0] = co * v.x;
      tt[k][1] = co * v.y;
    }
    if (has_x) mma_x<NT>(tt, P + in_x * PS, K0, g, t, bx0, bx1);
    if (has_y) mma_y<NT>(tt, P + in_y * PS, K0, g, t, ay0, ay1);
    if (has_z) dfma_z<NT>(tt, P + in_z * PS, K0, col, cz);
    if (FUSED && o < 0) {  // fused: u_next = q + L(qavg)
#pragma unroll
      for (int k = 0; k < NT; ++k) st_cs2(un + ((K0 + k) * 8) * urow + s * 8, tt[k][0], tt[k][1]);
      break;
    }
    __syncthreads();  // every warp has finished reading r
#pragma unroll
    for (int k = 0; k < NT; ++k) sts2(P + own + k * 64, tt[k][0], tt[k][1]);
    __syncthreads();  // new r complete
  }
}

// Normal stresses on k3 tiles K0 .. K0+NT-1: a = Dx u, b = Dy v, c = Dz w (unscaled), then
// t_sxx = lambda (a+b+c) + 2 mu a, etc. (proj/src/pde.cpp:180-190)
template <int NT, bool FUSED, int PS>
__device__ __forceinline__ void ck_normal(double* P, const double* Q, const double* cf, int K0, int g, int t,
                                          int col, double d0, double d1, const double (&c4)[4], double* un,
                                          int urow, int o_start) {
  const double lam = c4[1], two_mu = 2.0 * c4[2];
  constexpr int o_end = FUSED ? -1 : 0;
#pragma unroll 1
  for (int o = o_start; o >= o_end; --o) {
    const double co = (!FUSED || o >= 0) ? cf[o] : 1.0;
    double ta[NT][2], tb[NT][2], tc[NT][2];
#pragma unroll
    for (int k = 0; k < NT; ++k) ta[k][0] = ta[k][1] = tb[k][0] = tb[k][1] = tc[k][0] = tc[k][1] = 0.0;
    mma_x<NT>(ta, P + 6 * PS, K0, g, t, d0, d1);
    mma_y<NT>(tb, P + 7 * PS, K0, g, t, d0, d1);
    dfma_z<NT>(tc, P + 8 * PS, K0, col, 1.0);
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const int off = (K0 + k) * 64 + col;
      const double2 qa = lds2(Q + off), qb = lds2(Q + PS + off), qc = lds2(Q + 2 * PS + off);
      const double qv[3][2] = {{qa.x, qa.y}, {qb.x, qb.y}, {qc.x, qc.y}};
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const double sum = lam * (ta[k][j] + tb[k][j] + tc[k][j]);
        ta[k][j] = fma(co, qv[0][j], fma(two_mu, ta[k][j], sum));
        tb[k][j] = fma(co, qv[1][j], fma(two_mu, tb[k][j], sum));
        tc[k][j] = fma(co, qv[2][j], fma(two_mu, tc[k][j], sum));
      }
    }
    if (FUSED && o < 0) {  // fused: u_next = q + L(qavg)
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        double* r = un + ((K0 + k) * 8) * urow;
        st_cs2(r, ta[k][0], ta[k][1]);
        st_cs2(r + 8, tb[k][0], tb[k][1]);
        st_cs2(r + 16, tc[k][0], tc[k][1]);
      }
      break;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const int off = (K0 + k) * 64 + col;
      sts2(P + off, ta[k][0], ta[k][1]);
      sts2(P + PS + off, tb[k][0], tb[k][1]);
      sts2(P + 2 * PS + off, tc[k][0], tc[k][1]);
    }
    __syncthreads();
  }
}

// AOS: the reference's own layout, ElementTensor rows [k3][k2][k1][s < 16] in and PredictorOutput
// rows out (proj/src/layout.cpp:9-21, padding slots 9..15 written as zeros), no transposes: the
// quantity planes are staged from the node rows, and qavg / favg leave as whole 128-byte node rows
// (4 nodes per warp instruction) from the planes after the recursion.  Shared-memory planes are
// then 514 doubles apart, so that the 5 slot pairs of a node stored by neighbouring lanes fall on
// different banks (a uniform shift per plane: the fragment and column accesses stay conflict free).
template <bool AOS>
constexpr int plane_stride() { return AOS ? PV + 2 : PV + 8; }

template <bool FUSED, bool AOS = false, bool VOLM = false>
__global__ void __maxnreg__(80)
stp_dmma8_kernel(Params8 kp, BatchArgs a, unsigned int* status) {
  static_assert(!(FUSED && AOS), "the time loop runs on AoSoA");
  static_assert(!VOLM || FUSED, "the volume mode writes u_next");
  constexpr int THREADS8 = NWARP * 32;
  constexpr int PS = plane_stride<AOS>();
  extern __shared__ __align__(16) double sm8[];
  double* P = sm8;            // Horner iterate r   [9][8][8][8] swizzled; qavg at the end
  double* Q = sm8 + NV * PS;  // q (constant during the recursion)
  const long long e = blockIdx.x;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int col = phys(g, 2 * t);  // + k3*64: this lane's node pair within a quantity plane
  unsigned int flags = 0;
  TM3(0);
  // L2 prefetch of the q of element e + prefetch (one wave of SMs ahead: CTAs start in order),
  // issued first thing, so that CTA stages from L2 instead of HBM (cp.async.bulk.prefetch.L2)
  // Only the 9 used quantity slots of each (k3, k2) row are fetched when q_stride > 9 (C3: 12),
  // one 576-byte row per thread of the first two warps.
  if (kp.prefetch && tid < 64) {
    const long long nx = e + kp.prefetch;
    if (nx < a.n_elem) {
      const double* row = a.q + nx * (long long)(PV * kp.q_stride) + tid * kp.q_stride * 8;
      // AOS: the (k3, k2) row is 8 whole node rows (the used slots are not contiguous)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(row), "r"(AOS ? 8 * 16 * 8 : NV * 8 * 8)
                   : "memory");
    }
  }

  // ---- material (proj/src/pde.cpp:171-178) -------------------------------------------
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

  // ---- stage q: AoSoA [k3][k2][s < QS][k1] -> Q = q and P = c_(n-1) q ------------------
  // 64 rows (k3,k2) x 9 quantities x 4 k1-pairs = 2304 pairs = 9 per thread; every load is
  // issued before the first shared store so their latencies overlap.
  if constexpr (AOS) {  // node rows [k3][k2][k1][s < 16]: 512 nodes x 5 slot pairs (slot 9 unused)
    const double* qe = a.q + e * (long long)(PV * 16);
    constexpr int IT = 512 * 5 / THREADS8;
    double2 v[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int i = tid + it * THREADS8, node = i / 5, sp = 2 * (i - node * 5);
      v[it] = ld_nc2(qe + node * 16 + sp);
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int i = tid + it * THREADS8, node = i / 5, sp = 2 * (i - node * 5);
      if (kp.check && !(isfinite(v[it].x) && (sp == 8 || isfinite(v[it].y)))) flags |= 1u;
      const int j = sp * PS + (node >> 6) * 64 + phys((node >> 3) & 7, node & 7);
      Q[j] = v[it].x;
      P[j] = kp.cf[N8 - 1] * v[it].x;
      if (sp < 8) {
        Q[j + PS] = v[it].y;
        P[j + PS] = kp.cf[N8 - 1] * v[it].y;
      }
    }
  } else {
    const double* qe = a.q + e * (long long)(PV * kp.q_stride);
    constexpr int IT = (2304 + THREADS8 - 1) / THREADS8;
    double2 v[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int i = tid + it * THREADS8;
      const int r9 = i >> 2, k32 = r9 / NV, si = r9 - k32 * NV;
      if (2304 % THREADS8 == 0 || i < 2304) v[it] = ld_nc2(qe + (k32 * kp.q_stride + si) * 8 + 2 * (i & 3));
    }
    double2 w[VOLM ? IT : 1];  // volume mode: the iterate qavg, compact AoSoA (stride 9)
    if (VOLM) {
      const double* re = kp.r_src + e * (long long)(PV * NV);
#pragma unroll
      for (int it = 0; it < (VOLM ? IT : 1); ++it) {
        const int i = tid + it * THREADS8;
        const int r9 = i >> 2, k32 = r9 / NV, si = r9 - k32 * NV;
        if (2304 % THREADS8 == 0 || i < 2304) w[it] = ld_nc2(re + (k32 * NV + si) * 8 + 2 * (i & 3));
      }
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int i = tid + it * THREADS8;
      if (2304 % THREADS8 != 0 && i >= 2304) break;
      const int r9 = i >> 2, k32 = r9 / NV, si = r9 - k32 * NV;
      if (kp.check && !(isfinite(v[it].x) && isfinite(v[it].y))) flags |= 1u;
      const int j = si * PS + (k32 >> 3) * 64 + phys(k32 & 7, 2 * (i & 3));
      sts2(Q + j, v[it].x, v[it].y);
      if (VOLM)
        sts2(P + j, w[VOLM ? it : 0].x, w[VOLM ? it : 0].y);
      else
        sts2(P + j, kp.cf[N8 - 1] * v[it].x, kp.cf[N8 - 1] * v[it].y);
    }
  }
  __syncthreads();

  TM3(1);
  // ---- per-warp constants ---------------------------------------------------------------
  const double d0 = kp.d[g * 8 + t], d1 = kp.d[g * 8 + 4 + t];  // D[g][kh*4 + t]

  // ---- Cauchy-Kowalewsky recursion, Horner form ------------------------------------------
  {
    const int role = kRole[warp];
    const int urow = kp.q_stride * 8;
    double* un = FUSED ? a.u_next + e * (long long)(PV * kp.q_stride) + g * urow + 2 * t : nullptr;
    if (role >= 0)
      ck_quantity<8, FUSED, PS>(P, Q, kp.cf, role, 0, g, t, col, d0, d1, c4, un, urow, VOLM ? -1 : N8 - 2);
    else
      ck_normal<4, FUSED, PS>(P, Q, kp.cf, 4 * (-role - 1), g, t, col, d0, d1, c4, un, urow, VOLM ? -1 : N8 - 2);
    if (FUSED) __syncthreads();  // q (the Q region) is read until here; faces stage over it
  }

  TM3(2);
  // ---- epilogue ------------------------------------------------------------------------
  // 18 units (quantity s, k3 half h) over the 8 warps (kUnits): qavg and favg from registers, x/y faces
  // by DMMA from the accumulator (staged into the dead p buffers); the unit with h = 0 also does
  // the z faces, which need the whole column.
  double* FQ = Q;  // face_q staging [6][8][8][9] (q is dead after the last barrier)
  const bool faces = a.face_q || a.face_f;
  const double bphi0 = (g < 2) ? kp.phi[g][t] : 0.0;  // padded phi (rows / cols = side)
  const double bphi1 = (g < 2) ? kp.phi[g][4 + t] : 0.0;
#pragma unroll 1
  for (int ku = 0; ku < 3; ++ku) {
    const int unit = kUnits[warp][ku];
    if (unit < 0) break;
    const int s = unit >> 1, h = unit & 1, K0 = 4 * h;
    const double* qs = P + s * PS;
    double qa[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 v = lds2(qs + (K0 + k) * 64 + col);
      qa[k][0] = v.x;
      qa[k][1] = v.y;
    }
    if (!AOS && (!FUSED || a.qavg)) {
      double* qout = a.qavg + e * (long long)(PV * NV) + s * 8 + 2 * t;
#pragma unroll
      for (int k = 0; k < 4; ++k) st_cs2(qout + ((K0 + k) * 8 + g) * NV * 8, qa[k][0], qa[k][1]);
    }
    if (!AOS && a.favg) {
      double* fout = a.favg + e * (long long)(3 * PV * NV) + 2 * t;
      const int nout = kOutN[s];
#pragma unroll 1
      for (int k = 0; k < nout; ++k) {
        const int so = kOut[s][k][0], d = kOut[s][k][1];
        const double c = sel4(c4, kOut[s][k][2]);
        double* base = fout + d * (PV * NV) + so * 8;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          st_cs2(base + ((K0 + kk) * 8 + g) * NV * 8, c * qa[kk][0], c * qa[kk][1]);
      }
    }
    if (faces) {
      // x normal (faces 0, 1): C[k2][side] = sum_l Q[k3][k2][l] phi[side][l]   (B = phi^T)
      // y normal (faces 2, 3): C[side][k1] = sum_l phi[side][l] Q[k3][l][k1]   (A = phi)
      double xf[4][2], yf[4][2];
#pragma unroll
      for (int k = 0; k < 4; ++k) xf[k][0] = xf[k][1] = yf[k][0] = yf[k][1] = 0.0;
      mma_x<4>(xf, qs, K0, g, t, bphi0, bphi1);
      mma_y<4>(yf, qs, K0, g, t, bphi0, bphi1);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int k3 = K0 + k;
        if (t == 0) {  // lane (g, 0) holds C[k2 = g][side 0, 1]
          FQ[0 * FACES + (k3 * 8 + g) * NV + s] = xf[k][0];
          FQ[1 * FACES + (k3 * 8 + g) * NV + s] = xf[k][1];
        }
        if (g < 2) {  // lane (side = g, t) holds C[side][k1 = 2t, 2t+1]
          FQ[(2 + g) * FACES + (k3 * 8 + 2 * t) * NV + s] = yf[k][0];
          FQ[(2 + g) * FACES + (k3 * 8 + 2 * t + 1) * NV + s] = yf[k][1];
        }
      }
      if (h == 0) {  // z normal (faces 4, 5): (a, b) = (k2, k1), full column
        double z0[2] = {0.0, 0.0}, z1[2] = {0.0, 0.0};
#pragma unroll
        for (int k3 = 0; k3 < 8; ++k3) {
          const double2 v = lds2(qs + k3 * 64 + col);
          z0[0] = fma(kp.phi[0][k3], v.x, z0[0]);
          z0[1] = fma(kp.phi[0][k3], v.y, z0[1]);
          z1[0] = fma(kp.phi[1][k3], v.x, z1[0]);
          z1[1] = fma(kp.phi[1][k3], v.y, z1[1]);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          FQ[4 * FACES + (g * 8 + 2 * t + j) * NV + s] = z0[j];
          FQ[5 * FACES + (g * 8 + 2 * t + j) * NV + s] = z1[j];
        }
      }
    }
  }
  if constexpr (AOS) {
    // qavg and favg as whole node rows [node][s < 16]: lane = (node ns of 4, slot pair c), so a
    // warp instruction writes 4 x 128 contiguous bytes; the flux table entries of the lane's two
    // slots are fixed per lane (F_d(q)_so = coef(so, d) q[in(so, d)], proj/src/pde.cpp:180-218)
    const int ns = lane >> 3, c2 = 2 * (lane & 7);
    int src[3][2];
    double cfo[3][2];
    bool val[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int so = c2 + j;
      val[j] = so < NV;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int ci = val[j] ? kCoef[so][d] : 4;
        src[d][j] = val[j] ? kIn[so][d] : 0;
        cfo[d][j] = ci == 4 ? 0.0 : sel4(c4, ci);
      }
    }
    double* qo = a.qavg + e * (long long)(PV * 16);
    double* fo = a.favg ? a.favg + e * (long long)(3 * PV * 16) : nullptr;
#pragma unroll 1
    for (int nb = 4 * warp + ns; nb < PV; nb += 4 * NWARP) {
      const int pos = (nb >> 6) * 64 + phys((nb >> 3) & 7, nb & 7);
      st_cs2(qo + nb * 16 + c2, val[0] ? P[c2 * PS + pos] : 0.0, val[1] ? P[(c2 + 1) * PS + pos] : 0.0);
      if (fo) {
#pragma unroll
        for (int d = 0; d < 3; ++d)
          st_cs2(fo + d * (PV * 16) + nb * 16 + c2, cfo[d][0] != 0.0 ? cfo[d][0] * P[src[d][0] * PS + pos] : 0.0,
                 cfo[d][1] != 0.0 ? cfo[d][1] * P[src[d][1] * PS + pos] : 0.0);
      }
    }
  }
  if (faces) {
    // FQ complete; qavg (P) is no longer read, so face_f is staged over it.  face_q leaves at once
    // (TMA bulk store, SASS UBLKCP) and its copy overlaps the face_f pass below.
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid < 6 && a.face_q) {  // one bulk copy per face (the staged faces are FACES apart)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                       a.face_q + e * (long long)(6 * FACE) + tid * FACE),
                   "r"((unsigned)__cvta_generic_to_shared(FQ + tid * FACES)), "r"((unsigned)(FACE * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    TM3(3);
    double* FF = P;
    // face_f[f][ab][so] = coef(so, d) face_q[f][ab][in(so, d)]: thread = (face f, node ab), 9 loads
    // and 9 stores with the compile-time flux of direction d = f / 2
    if (a.face_f) {
#pragma unroll 1
      for (int i = tid; i < 6 * 64; i += THREADS8) {
        const int f = i >> 6, d = f >> 1;
        const double* src = FQ + f * FACES + (i & 63) * NV;
        double* dst = FF + f * FACES + (i & 63) * NV;
        double w[NV];
#pragma unroll
        for (int s = 0; s < NV; ++s) w[s] = src[s];
        auto emit = [&](auto dd) {
          constexpr int D = decltype(dd)::value;
#pragma unroll
          for (int so = 0; so < NV; ++so) {
            const int ci = e_coef(so, D);
            dst[so] = ci == 4 ? 0.0 : c4[ci & 3] * w[e_in(so, D)];
          }
        };
        if (d == 0) emit(std::integral_constant<int, 0>{});
        else if (d == 1) emit(std::integral_constant<int, 1>{});
        else emit(std::integral_constant<int, 2>{});
      }
    }
    TM3(4);
    // face_f leaves as a second TMA bulk store; thread 0 then waits until both copies have read
    // the shared memory (the CTA's shared memory must outlive them)
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    TM3(5);
    if (tid < 6) {
      if (a.face_f)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                         a.face_f + e * (long long)(6 * FACE) + tid * FACE),
                     "r"((unsigned)__cvta_generic_to_shared(FF + tid * FACES)), "r"((unsigned)(FACE * 8))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
  }
  if (kp.check && flags) atomicOr(status, flags);
  TM3(6);
}

// ---- table PDEs (any constant-coefficient LinearPde given as term tables, m <= 9) -----------
// The user-PDE path on the tensor cores: warp s owns output quantity s (s < 8; a ninth quantity is
// split over the warps by k3 plane, compiled only into the HAS9 instance), and a CK step
// is  t_s = c_o q_s + sum_d sum_k tc[s][d][k] D_d r_{tr[s][d][k]}  (build_terms folds the ncp
// matrices in: D_d (A_d + B_d) p, proj/src/stp_splitck.cpp:53-61 for constant coefficients) --
// every term one more pair of DMMAs (x, y) or register DFMAs (z) into the same accumulators, the
// coefficient folded into the D fragments.  favg_d = A_d qavg and face_f = A_d face_q from the
// favg tables (fr, fc); faces and bulk stores as in the elastic kernel.
constexpr int GM = 9;  // quantities of the table kernel (the 9th is split over the warps by plane)
struct ParamsG {
  double d[64];
  double phi[2][8];
  double cf[8];
  double tc[GM][3][kMaxTerms];
  double fc[GM][3][kMaxTerms];
  signed char tr[GM][3][kMaxTerms];
  signed char fr[GM][3][kMaxTerms];
  int m, n_terms, q_stride, check;
};

// HAS9: m == 9 (the ninth quantity's accumulators and branches); m <= 8 compiles without them and
// keeps its registers (80, no ninth-quantity spill traffic)
template <bool HAS9>
__global__ void __maxnreg__(80) stp_dmma8_table_kernel(ParamsG kp, BatchArgs a, unsigned int* status) {
  constexpr int THREADS8 = NWARP * 32;
  extern __shared__ __align__(16) double smg[];
  const int m = kp.m, nt = kp.n_terms;
  double* P = smg;           // iterate r [m][8][8][8] swizzled; qavg at the end
  double* Q = smg + m * PV;  // q
  const long long e = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int col = phys(g, 2 * t);
  unsigned int flags = 0;
  // ---- stage q: AoSoA [k3][k2][s < q_stride][k1] -> Q = q, P = c_(n-1) q -------------------
  {
    const double* qe = a.q + e * (long long)(PV * kp.q_stride);
    const int pairs = 64 * m * 4;
    for (int i = tid; i < pairs; i += THREADS8) {
      const int r = i >> 2, k32 = r / m, si = r - k32 * m;
      const double2 v = ld_nc2(qe + (k32 * kp.q_stride + si) * 8 + 2 * (i & 3));
      if (kp.check && !(isfinite(v.x) && isfinite(v.y))) flags |= 1u;
      const int j = si * PV + (k32 >> 3) * 64 + phys(k32 & 7, 2 * (i & 3));
      sts2(Q + j, v.x, v.y);
      sts2(P + j, kp.cf[N8 - 1] * v.x, kp.cf[N8 - 1] * v.y);
    }
  }
  __syncthreads();
  const double d0 = kp.d[g * 8 + t], d1 = kp.d[g * 8 + 4 + t];
  const int s = warp;
  const bool own = s < m && s < 8;
  double tt[8][2];
  double t8[1][2];  // m = 9: plane k3 = warp of quantity 8
  // ---- Horner form of the CK series (see ck_quantity) ----------------------------------------
#pragma unroll 1
  for (int o = N8 - 2; o >= 0; --o) {
    if (own) {
      const double co = kp.cf[o];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double2 v = lds2(Q + s * PV + k * 64 + col);
        tt[k][0] = co * v.x;
        tt[k][1] = co * v.y;
      }
#pragma unroll 1
      for (int k = 0; k < nt; ++k) {
        const double cx = kp.tc[s][0][k], cy = kp.tc[s][1][k], cz = kp.tc[s][2][k];
        if (cx != 0.0) mma_x<8>(tt, P + kp.tr[s][0][k] * PV, 0, g, t, cx * d0, cx * d1);
        if (cy != 0.0) mma_y<8>(tt, P + kp.tr[s][1][k] * PV, 0, g, t, cy * d0, cy * d1);
        if (cz != 0.0) dfma_z<8>(tt, P + kp.tr[s][2][k] * PV, 0, col, cz);
      }
    }
    if (HAS9) {  // quantity 8: warp w takes plane k3 = w
      const double co = kp.cf[o];
      const double2 v = lds2(Q + 8 * PV + warp * 64 + col);
      t8[0][0] = co * v.x;
      t8[0][1] = co * v.y;
#pragma unroll 1
      for (int k = 0; k < nt; ++k) {
        const double cx = kp.tc[8][0][k], cy = kp.tc[8][1][k], cz = kp.tc[8][2][k];
        if (cx != 0.0) mma_x<1>(t8, P + kp.tr[8][0][k] * PV, warp, g, t, cx * d0, cx * d1);
        if (cy != 0.0) mma_y<1>(t8, P + kp.tr[8][1][k] * PV, warp, g, t, cy * d0, cy * d1);
        if (cz != 0.0) dfma_z<1>(t8, P + kp.tr[8][2][k] * PV, warp, col, cz);
      }
    }
    __syncthreads();  // every warp has finished reading r
    if (own) {
#pragma unroll
      for (int k = 0; k < 8; ++k) sts2(P + s * PV + k * 64 + col, tt[k][0], tt[k][1]);
    }
    if (HAS9) sts2(P + 8 * PV + warp * 64 + col, t8[0][0], t8[0][1]);
    __syncthreads();  // new r (qavg after the last step) complete
  }
  // ---- epilogue: qavg and favg of quantity s, x/y/z faces --------------------------------------
  double* FQ = Q;  // face_q staging [6][8][8][m] (q is dead)
  constexpr int FA = 64;  // in-face nodes
  const int FACE = FA * m;
  const bool faces = a.face_q || a.face_f;
  if (own) {
    double* qout = a.qavg + e * (long long)(PV * m) + s * 8 + 2 * t;
#pragma unroll
    for (int k = 0; k < 8; ++k) st_cs2(qout + (k * 8 + g) * m * 8, tt[k][0], tt[k][1]);
    if (a.favg) {
      double* fout = a.favg + e * (long long)(3 * PV * m) + s * 8 + 2 * t;
#pragma unroll 1
      for (int d = 0; d < 3; ++d) {
        double f[8][2];
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k][0] = f[k][1] = 0.0;
#pragma unroll 1
        for (int kt = 0; kt < nt; ++kt) {
          const double c = kp.fc[s][d][kt];
          if (c == 0.0) continue;
          const double* src = P + kp.fr[s][d][kt] * PV + col;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const double2 v = lds2(src + k * 64);
            f[k][0] = fma(c, v.x, f[k][0]);
            f[k][1] = fma(c, v.y, f[k][1]);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) st_cs2(fout + d * (PV * m) + (k * 8 + g) * m * 8, f[k][0], f[k][1]);
      }
    }
    if (faces) {
      const double bphi0 = (g < 2) ? kp.phi[g][t] : 0.0, bphi1 = (g < 2) ? kp.phi[g][4 + t] : 0.0;
      const double* qs = P + s * PV;
      double xf[8][2], yf[8][2];
#pragma unroll
      for (int k = 0; k < 8; ++k) xf[k][0] = xf[k][1] = yf[k][0] = yf[k][1] = 0.0;
      mma_x<8>(xf, qs, 0, g, t, bphi0, bphi1);
      mma_y<8>(yf, qs, 0, g, t, bphi0, bphi1);
#pragma unroll
      for (int k3 = 0; k3 < 8; ++k3) {
        if (t == 0) {
          FQ[0 * FACE + (k3 * 8 + g) * m + s] = xf[k3][0];
          FQ[1 * FACE + (k3 * 8 + g) * m + s] = xf[k3][1];
        }
        if (g < 2) {
          FQ[(2 + g) * FACE + (k3 * 8 + 2 * t) * m + s] = yf[k3][0];
          FQ[(2 + g) * FACE + (k3 * 8 + 2 * t + 1) * m + s] = yf[k3][1];
        }
      }
      double z0[2] = {0.0, 0.0}, z1[2] = {0.0, 0.0};
#pragma unroll
      for (int k3 = 0; k3 < 8; ++k3)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          z0[j] = fma(kp.phi[0][k3], tt[k3][j], z0[j]);
          z1[j] = fma(kp.phi[1][k3], tt[k3][j], z1[j]);
        }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        FQ[4 * FACE + (g * 8 + 2 * t + j) * m + s] = z0[j];
        FQ[5 * FACE + (g * 8 + 2 * t + j) * m + s] = z1[j];
      }
    }
  }
  if (HAS9) {  // quantity 8, plane k3 = warp: qavg, favg, x / y faces; warp 0 also the z faces
    const int k3 = warp;
    double* qout = a.qavg + e * (long long)(PV * m) + 8 * 8 + 2 * t;
    st_cs2(qout + (k3 * 8 + g) * m * 8, t8[0][0], t8[0][1]);
    if (a.favg) {
      double* fout = a.favg + e * (long long)(3 * PV * m) + 8 * 8 + 2 * t;
#pragma unroll 1
      for (int d = 0; d < 3; ++d) {
        double f0 = 0.0, f1 = 0.0;
#pragma unroll 1
        for (int kt = 0; kt < nt; ++kt) {
          const double c = kp.fc[8][d][kt];
          if (c == 0.0) continue;
          const double2 v = lds2(P + kp.fr[8][d][kt] * PV + k3 * 64 + col);
          f0 = fma(c, v.x, f0);
          f1 = fma(c, v.y, f1);
        }
        st_cs2(fout + d * (PV * m) + (k3 * 8 + g) * m * 8, f0, f1);
      }
    }
    if (faces) {
      const double bphi0 = (g < 2) ? kp.phi[g][t] : 0.0, bphi1 = (g < 2) ? kp.phi[g][4 + t] : 0.0;
      double xf[1][2] = {{0.0, 0.0}}, yf[1][2] = {{0.0, 0.0}};
      mma_x<1>(xf, P + 8 * PV, k3, g, t, bphi0, bphi1);
      mma_y<1>(yf, P + 8 * PV, k3, g, t, bphi0, bphi1);
      if (t == 0) {
        FQ[0 * FACE + (k3 * 8 + g) * m + 8] = xf[0][0];
        FQ[1 * FACE + (k3 * 8 + g) * m + 8] = xf[0][1];
      }
      if (g < 2) {
        FQ[(2 + g) * FACE + (k3 * 8 + 2 * t) * m + 8] = yf[0][0];
        FQ[(2 + g) * FACE + (k3 * 8 + 2 * t + 1) * m + 8] = yf[0][1];
      }
      if (warp == 0) {
        double z0[2] = {0.0, 0.0}, z1[2] = {0.0, 0.0};
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const double2 v = lds2(P + 8 * PV + kk * 64 + col);
          z0[0] = fma(kp.phi[0][kk], v.x, z0[0]);
          z0[1] = fma(kp.phi[0][kk], v.y, z0[1]);
          z1[0] = fma(kp.phi[1][kk], v.x, z1[0]);
          z1[1] = fma(kp.phi[1][kk], v.y, z1[1]);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          FQ[4 * FACE + (g * 8 + 2 * t + j) * m + 8] = z0[j];
          FQ[5 * FACE + (g * 8 + 2 * t + j) * m + 8] = z1[j];
        }
      }
    }
  }
  if (faces) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();  // FQ complete; qavg (P) no longer read
    const unsigned bytes = 6u * FACE * 8u;
    if (tid == 0 && a.face_q) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                       a.face_q + e * (long long)(6 * FACE)),
                   "r"((unsigned)__cvta_generic_to_shared(FQ)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    double* FF = P;
    if (a.face_f) {  // face_f[f][ab][so] = sum_k fc[so][d][k] face_q[f][ab][fr[so][d][k]], d = f / 2
      for (int i = tid; i < 6 * FA * m; i += THREADS8) {
        const int fa = i / m, so = i - fa * m, f = fa / FA, d = f >> 1;
        const double* src = FQ + fa * m;
        double v = 0.0;
        for (int kt = 0; kt < nt; ++kt) {
          const double c = kp.fc[so][d][kt];
          if (c != 0.0) v = fma(c, src[kp.fr[so][d][kt]], v);
        }
        FF[i] = v;
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncthreads();
      if (tid == 0)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                         a.face_f + e * (long long)(6 * FACE)),
                     "r"((unsigned)__cvta_generic_to_shared(FF)), "r"(bytes)
                     : "memory");
    }
    if (tid == 0) {
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
  }
  if (kp.check && flags) atomicOr(status, flags);
}

}  // namespace

bool dmma8_applicable(const LaunchPlan& p) {
  return p.n == 8 && p.kind == ADERSTP_PDE_ELASTIC && p.src_comp < 0 && p.layout == ADERSTP_LAYOUT_AOSOA &&
         p.out_stride == 9 && p.q_stride >= 9 && p.q_stride <= 64;
}

// the reference's own layout straight into the kernel: ElementTensor AoS rows with the quantity
// padded to 16 (proj/src/layout.cpp:9-21) in and out, 16-byte aligned buffers
bool dmma8_aos_applicable(const LaunchPlan& p, const BatchArgs& a) {
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  return p.n == 8 && p.kind == ADERSTP_PDE_ELASTIC && p.src_comp < 0 && p.layout == ADERSTP_LAYOUT_AOS &&
         p.q_stride == 16 && p.out_stride == 16 && !p.force_generic && !p.no_dmma8 && !p.aos_staged &&
         !a.u_next && al16(a.q) && al16(a.qavg) && al16(a.favg) && al16(a.face_q) && al16(a.face_f);
}

// table PDEs at nDof 8 on the tensor cores: m <= 9, compact AoSoA outputs, no point source
bool dmma8_table_applicable(const LaunchPlan& p, const BatchArgs& a) {
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  return p.n == 8 && p.kind != ADERSTP_PDE_ELASTIC && p.kind != ADERSTP_PDE_ELASTIC_SOURCE && p.src_comp < 0 &&
         p.m >= 1 && p.m <= GM && p.layout == ADERSTP_LAYOUT_AOSOA && p.out_stride == p.m && p.q_stride >= p.m &&
         p.q_stride <= 64 && p.n_terms <= kMaxTerms && !p.force_generic && !p.no_dmma8 && !a.u_next &&
         al16(a.q) && al16(a.qavg) && al16(a.favg) && al16(a.face_q) && al16(a.face_f);
}

cudaError_t launch_dmma8_table(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  ParamsG kp;
  for (int i = 0; i < 64; ++i) kp.d[i] = p.basis.d[i];
  for (int j = 0; j < 8; ++j) {
    kp.phi[0][j] = p.basis.face_left[j];
    kp.phi[1][j] = p.basis.face_right[j];
  }
  {
    double c = a.dt;  // same operation sequence as proj/src/stp_splitck.cpp:45,64
    kp.cf[0] = c;
    for (int o = 1; o < N8; ++o) {
      c *= a.dt / (o + 1);
      kp.cf[o] = c;
    }
  }
  for (int s = 0; s < GM; ++s)
    for (int d = 0; d < 3; ++d)
      for (int k = 0; k < kMaxTerms; ++k) {
        const bool in = s < p.m && k < p.n_terms;
        kp.tr[s][d][k] = in ? p.tr[s][d][k] : 0;
        kp.tc[s][d][k] = in ? p.tc[s][d][k] : 0.0;
        kp.fr[s][d][k] = in ? p.fr[s][d][k] : 0;
        kp.fc[s][d][k] = in ? p.fc[s][d][k] : 0.0;
      }
  kp.m = p.m;
  kp.n_terms = p.n_terms;
  kp.q_stride = p.q_stride;
  kp.check = p.check;
  const int smem = 2 * p.m * PV * 8;
  auto kern = p.m == GM ? stp_dmma8_table_kernel<true> : stp_dmma8_table_kernel<false>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  if (a.n_elem == 0) return cudaSuccess;
  if (a.n_elem > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)a.n_elem, NWARP * 32, smem, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}

cudaError_t init_dmma8(const LaunchPlan& p) {
  return cudaMemcpyToSymbol(aderstp_kD8, p.basis.d, sizeof(double) * 64);
}

cudaError_t launch_dmma8(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  Params8 kp;
  for (int i = 0; i < 64; ++i) kp.d[i] = p.basis.d[i];
  for (int j = 0; j < 8; ++j) {
    kp.phi[0][j] = p.basis.face_left[j];
    kp.phi[1][j] = p.basis.face_right[j];
  }
  kp.check = p.check;
  kp.par_kind = p.par_kind;
  kp.q_stride = p.q_stride;
  kp.prefetch = p.dmma8_prefetch;
  kp.r_src = a.vol_r;
  kp.o_start = a.vol_r ? -1 : N8 - 2;
  {
    double c = a.dt;  // same operation sequence as proj/src/stp_splitck.cpp:45,64
    kp.cf[0] = c;
    for (int o = 1; o < N8; ++o) {
      c *= a.dt / (o + 1);
      kp.cf[o] = c;
    }
  }
  const bool aos = p.layout == ADERSTP_LAYOUT_AOS;  // dmma8_aos_applicable
  auto kern = a.vol_r    ? stp_dmma8_kernel<true, false, true>
              : a.u_next ? stp_dmma8_kernel<true>
              : aos      ? stp_dmma8_kernel<false, true>
                         : stp_dmma8_kernel<false>;
  int smem = aos ? 2 * NV * plane_stride<true>() * 8 : kSmem8;
#ifdef ADERSTP_EXPT_TIMING
  if (const char* x = std::getenv("ADERSTP_EXPT_SMEM")) smem += std::atoi(x);  // occupancy experiments
#endif
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  if (a.n_elem == 0) return cudaSuccess;
  if (a.n_elem > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)a.n_elem, NWARP * 32, smem, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}

}  // namespace aderstp
