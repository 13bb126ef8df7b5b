// nDof = 8 elastic STP kernel on the fp64 tensor cores (sm_100a DMMA, mma.sync m8n8k4 f64).
//
// One CTA = one element, 9 warps, warp w owns output quantity kWarpVar[w] for ALL nodes.
// Lane (g = lane/4, t = lane%4) owns the two z-columns (k2 = g, k1 = 2t, 2t+1): 16 nodes.
// That is exactly the C-fragment of an 8x8 MMA tile C[k2][k1] at fixed k3, so
//   x-contraction  C[k2][k1] += sum_l P[k3][k2][l] * (c D)[k1][l]   A = p slice, B = c*D^T
//   y-contraction  C[k2][k1] += sum_l (c D)[k2][l] * P[k3][l][k1]   A = c*D,     B = p slice
// run as DMMA (16 per field: 8 k3-tiles x 2 k-halves) accumulating straight into the thread's
// t registers, and the z-contraction is register-local DFMA on the thread's own columns with D
// as constant-bank operands:  t[k3] += sum_l D[k3][l] * (c p[l]).
// Flux-first exactly as the reference: t_s = sum_d D_d * F_d(p)_s with the elastic flux
// F_d(p)_s = c(s,d) p_in(s,d) (proj/src/pde.cpp:180-218, proj/src/stp_splitck.cpp:53-55).
//
// Shared memory: the current iterate p, 9 x 8 x 8 x 8 fp64 with an XOR swizzle on the k1 index
// (bit 2 flipped on rows with k2 & 2) so that every fragment load, column load and write-back
// is bank-conflict free; plus face_q / face_f staging.  Warps are ordered so that the three
// light shear warps share SMSP 0 (warp % 4 == 0) and the SMSP loads balance.
// qavg and favg leave straight from registers; the 12 face arrays are computed by DMMA
// (x, y normals) and register DFMA (z normal), staged in shared memory and written coalesced.
#include <cstdint>
#include <utility>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"

namespace aderstp {

namespace {

constexpr int N8 = 8;
constexpr int NV = 9;
constexpr int THREADS8 = NV * 32;
constexpr int PV = N8 * N8 * N8;           // doubles per quantity plane
constexpr int FACE = N8 * N8 * NV;         // doubles per face array (576)
constexpr int SMEM8 = 3 * NV * PV * 8;  // p, p_next, qavg accumulator = 110,592 B (face staging reuses p)

struct Params8 {
  double d[64];      // d[k*8+l] = phi_l'(x_k)
  double phi[2][8];  // phi(0), phi(1)
  int check;
  int par_kind;
  int q_stride;
};

// warp -> output quantity (shear warps on SMSP 0)
__constant__ int kWarpVar[NV] = {3, 0, 1, 2, 4, 6, 7, 8, 5};
// flux table: F_d(q)_s = coef(s,d) * q[in(s,d)]; coef 0: lambda+2mu, 1: lambda, 2: mu, 3: 1/rho, 4: 0
__constant__ int kIn[NV][3] = {{6, 7, 8}, {6, 7, 8}, {6, 7, 8}, {7, 6, 0}, {8, 0, 6},
                               {0, 8, 7}, {0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
__constant__ int kCoef[NV][3] = {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {2, 2, 4}, {2, 4, 2},
                                 {4, 2, 2}, {3, 3, 3}, {3, 3, 3}, {3, 3, 3}};
// outgoing flux entries of each source quantity r: (s, d, coef) with in(s,d) = r, plus the three
// identically-zero entries (coef 4) assigned to the shear warps.  Used for favg and face_f.
__constant__ int kOutN[NV] = {1, 1, 1, 3, 3, 3, 5, 5, 5};
__constant__ int kOut[NV][5][3] = {
    {{6, 0, 3}}, {{7, 1, 3}}, {{8, 2, 3}},
    {{6, 1, 3}, {7, 0, 3}, {3, 2, 4}},
    {{6, 2, 3}, {8, 0, 3}, {4, 1, 4}},
    {{7, 2, 3}, {8, 1, 3}, {5, 0, 4}},
    {{0, 0, 0}, {1, 0, 1}, {2, 0, 1}, {3, 1, 2}, {4, 2, 2}},
    {{0, 1, 1}, {1, 1, 0}, {2, 1, 1}, {3, 0, 2}, {5, 2, 2}},
    {{0, 2, 1}, {1, 2, 1}, {2, 2, 0}, {4, 0, 2}, {5, 1, 2}}};

// D of the nDof = 8 Gauss-Legendre basis (identical for every plan), uploaded once per device;
// read with volatile ld.const so the z-contraction streams it through the constant cache
// instead of pinning 64 doubles in registers.
}  // namespace
}  // namespace aderstp

// D of the nDof = 8 Gauss-Legendre basis (the same for every plan), uploaded once per device.
// The z-contraction reads it at the point of use through volatile ld.const (constant cache,
// broadcast), so ptxas cannot hoist 64 doubles of D into registers and spill.
extern "C" {
__constant__ double aderstp_kD8[64];
}

namespace aderstp {
namespace {

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

__global__ void __maxnreg__(80)
stp_dmma8_kernel(Params8 kp, BatchArgs a, unsigned int* status) {
  extern __shared__ __align__(16) double sm8[];
  double* P = sm8;                  // [9][8][8][8] swizzled: current iterate p
  double* PN = sm8 + NV * PV;       // next iterate (double buffer: one barrier per CK step)
  double* QA = sm8 + 2 * NV * PV;   // [9][8][8][8] swizzled: qavg accumulator
  double* FQ = sm8;                 // epilogue: face_q staging [6][8][8][9] reuses the p buffers
  const long long e = blockIdx.x;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int s = kWarpVar[warp];
  unsigned int flags = 0;
  const double dt = a.dt;

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

  // ---- stage q: AoSoA [k3][k2][s < QS][k1] -> P and QA = dt q -------------------------
  // 64 rows (k3,k2) x 9 quantities x 4 k1-pairs = 2304 pairs = 8 per thread; all loads are
  // issued before the first shared store so their latencies overlap.
  {
    const double* qe = a.q + e * (long long)(PV * kp.q_stride);
    double2 v[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int i = tid + it * THREADS8;
      const int r9 = i >> 2, k32 = r9 / NV, si = r9 - k32 * NV;
      v[it] = ld_nc2(qe + (k32 * kp.q_stride + si) * 8 + 2 * (i & 3));
    }
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int i = tid + it * THREADS8;
      const int r9 = i >> 2, k32 = r9 / NV, si = r9 - k32 * NV;
      if (kp.check && !(isfinite(v[it].x) && isfinite(v[it].y))) flags |= 1u;
      const int j = si * PV + (k32 >> 3) * 64 + phys(k32 & 7, 2 * (i & 3));
      *reinterpret_cast<double2*>(P + j) = v[it];
      *reinterpret_cast<double2*>(QA + j) = make_double2(dt * v[it].x, dt * v[it].y);
    }
  }
  __syncthreads();

  // ---- per-warp constants ---------------------------------------------------------------
  const int in_x = kIn[s][0], in_y = kIn[s][1], in_z = kIn[s][2];
  const double cx = sel4(c4, kCoef[s][0]), cy = sel4(c4, kCoef[s][1]), cz = sel4(c4, kCoef[s][2]);
  const bool has_x = kCoef[s][0] != 4, has_y = kCoef[s][1] != 4, has_z = kCoef[s][2] != 4;
  const double d0 = kp.d[g * 8 + t], d1 = kp.d[g * 8 + 4 + t];  // D[g][kh*4 + t]
  const double bx0 = cx * d0, bx1 = cx * d1;                     // B-fragments of c_x D^T
  const double ay0 = cy * d0, ay1 = cy * d1;                     // A-fragments of c_y D
  const int own = s * PV + phys(g, 2 * t);                       // + k3*64: this lane's node pair

  // ---- Cauchy-Kowalewsky recursion (proj/src/stp_splitck.cpp:46-70) -------------------
  double coeff = dt;
#pragma unroll 1
  for (int o = 1; o < N8; ++o) {
    double tt[8][2];
#pragma unroll
    for (int k3 = 0; k3 < 8; ++k3) tt[k3][0] = tt[k3][1] = 0.0;
    if (has_x) {
      const double* px = P + in_x * PV + phys(g, t);
      const double* px1 = P + in_x * PV + phys(g, 4 + t);
#pragma unroll
      for (int k3 = 0; k3 < 8; ++k3) {
        dmma(tt[k3][0], tt[k3][1], px[k3 * 64], bx0);
        dmma(tt[k3][0], tt[k3][1], px1[k3 * 64], bx1);
      }
    }
    if (has_y) {
      const double* py = P + in_y * PV + phys(t, g);
      const double* py1 = P + in_y * PV + phys(4 + t, g);
#pragma unroll
      for (int k3 = 0; k3 < 8; ++k3) {
        dmma(tt[k3][0], tt[k3][1], ay0, py[k3 * 64]);
        dmma(tt[k3][0], tt[k3][1], ay1, py1[k3 * 64]);
      }
    }
    if (has_z) {
      const double* pz = P + in_z * PV + phys(g, 2 * t);
#pragma unroll
      for (int lq = 0; lq < 4; ++lq) {
        double c0[2], c1[2];
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          const double2 v = *reinterpret_cast<const double2*>(pz + (lq * 2 + l) * 64);
          c0[l] = cz * v.x;
          c1[l] = cz * v.y;
        }
#pragma unroll
        for (int k3 = 0; k3 < 8; ++k3) {
          const double2 dk = ldc2(&aderstp_kD8[k3 * 8 + lq * 2]);
          tt[k3][0] = fma(dk.x, c0[0], tt[k3][0]);
          tt[k3][1] = fma(dk.x, c1[0], tt[k3][1]);
          tt[k3][0] = fma(dk.y, c0[1], tt[k3][0]);
          tt[k3][1] = fma(dk.y, c1[1], tt[k3][1]);
        }
      }
    }
    coeff *= dt / (o + 1);  // dt^(o+1)/(o+1)!
#pragma unroll
    for (int k3 = 0; k3 < 8; ++k3) {  // qavg += c_o t on this lane's own nodes (no race)
      double2* q = reinterpret_cast<double2*>(QA + own + k3 * 64);
      const double2 v = *q;
      *q = make_double2(fma(coeff, tt[k3][0], v.x), fma(coeff, tt[k3][1], v.y));
    }
    if (o + 1 < N8) {
#pragma unroll
      for (int k3 = 0; k3 < 8; ++k3)
        *reinterpret_cast<double2*>(PN + own + k3 * 64) = make_double2(tt[k3][0], tt[k3][1]);
    }
    __syncthreads();  // p_next complete; every warp has finished reading p
    double* sw = P;
    P = PN;
    PN = sw;
  }

  // ---- epilogue ------------------------------------------------------------------------
  double qa[8][2];
#pragma unroll
  for (int k3 = 0; k3 < 8; ++k3) {
    const double2 v = *reinterpret_cast<const double2*>(QA + own + k3 * 64);
    qa[k3][0] = v.x;
    qa[k3][1] = v.y;
  }
  // qavg straight from registers, AoSoA [k3][k2][s][k1]
  {
    double* qout = a.qavg + e * (long long)(PV * NV) + s * 8 + 2 * t;
#pragma unroll
    for (int k3 = 0; k3 < 8; ++k3) st_cs2(qout + (k3 * 8 + g) * NV * 8, qa[k3][0], qa[k3][1]);
  }
  // favg_d[s'] = coef * qavg[s] for every flux entry fed by this warp's quantity
  if (a.favg) {
    double* fout = a.favg + e * (long long)(3 * PV * NV) + 2 * t;
    const int nout = kOutN[s];
#pragma unroll 1
    for (int k = 0; k < nout; ++k) {
      const int so = kOut[s][k][0], d = kOut[s][k][1];
      const double c = sel4(c4, kOut[s][k][2]);
      double* base = fout + d * (PV * NV) + so * 8;
#pragma unroll
      for (int k3 = 0; k3 < 8; ++k3) st_cs2(base + (k3 * 8 + g) * NV * 8, c * qa[k3][0], c * qa[k3][1]);
    }
  }
  if (a.face_q || a.face_f) {
    // z normal (faces 4, 5): register-local columns, (a, b) = (k2, k1)
    // x normal (faces 0, 1): C[k2][side] = sum_l Q[k3][k2][l] phi[side][l]  (B = padded phi^T)
    // y normal (faces 2, 3): C[side][k1] = sum_l phi[side][l] Q[k3][l][k1]  (A = padded phi)
    const double bphi0 = (g < 2) ? kp.phi[g][t] : 0.0;
    const double bphi1 = (g < 2) ? kp.phi[g][4 + t] : 0.0;
    const double* qx = QA + s * PV + phys(g, t);
    const double* qx1 = QA + s * PV + phys(g, 4 + t);
    const double* qy = QA + s * PV + phys(t, g);
    const double* qy1 = QA + s * PV + phys(4 + t, g);
    // the last CK step's write-back was skipped, but p is still being read by no one after the
    // final barrier: reuse it as the face staging area [f][a][b][s]
#pragma unroll
    for (int sd = 0; sd < 2; ++sd)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k3 = 0; k3 < 8; ++k3) acc = fma(kp.phi[sd][k3], qa[k3][j], acc);
        FQ[(4 + sd) * FACE + (g * 8 + 2 * t + j) * NV + s] = acc;
      }
#pragma unroll 2
    for (int k3 = 0; k3 < 8; ++k3) {
      double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
      dmma(x0, x1, qx[k3 * 64], bphi0);
      dmma(x0, x1, qx1[k3 * 64], bphi1);
      dmma(y0, y1, bphi0, qy[k3 * 64]);
      dmma(y0, y1, bphi1, qy1[k3 * 64]);
      if (t == 0) {  // lane (g, 0) holds C[k2 = g][side 0, 1]
        FQ[0 * FACE + (k3 * 8 + g) * NV + s] = x0;
        FQ[1 * FACE + (k3 * 8 + g) * NV + s] = x1;
      }
      if (g < 2) {  // lane (side = g, t) holds C[side][k1 = 2t, 2t+1]
        FQ[(2 + g) * FACE + (k3 * 8 + 2 * t) * NV + s] = y0;
        FQ[(2 + g) * FACE + (k3 * 8 + 2 * t + 1) * NV + s] = y1;
      }
    }
    __syncthreads();
    // coalesced copy-out.  288 threads = 32 in-face nodes x 9 quantities, so thread tid always
    // handles quantity so = tid % 9: face_f[f][ab][so] = coef(so, d) * face_q[f][ab][in(so, d)]
    // (flux linearity), with the coefficients hoisted out of the loop.
    const int so = tid % NV, ab0 = tid / NV;
    double* oq = a.face_q ? a.face_q + e * (long long)(6 * FACE) : nullptr;
    double* of = a.face_f ? a.face_f + e * (long long)(6 * FACE) : nullptr;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double c = sel4(c4, kCoef[so][d]);
      const int src = kIn[so][d];
#pragma unroll
      for (int sd = 0; sd < 2; ++sd)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int base = (2 * d + sd) * FACE + (ab0 + 32 * h) * NV;
          if (oq) __stcs(oq + base + so, FQ[base + so]);
          if (of) __stcs(of + base + so, c * FQ[base + src]);
        }
    }
  }
  if (kp.check && flags) atomicOr(status, flags);
}

}  // namespace

bool dmma8_applicable(const LaunchPlan& p) {
  return p.n == 8 && p.kind == ADERSTP_PDE_ELASTIC && p.src_comp < 0 && p.layout == ADERSTP_LAYOUT_AOSOA &&
         p.out_stride == 9 && p.q_stride >= 9 && p.q_stride <= 64;
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
  cudaError_t err = cudaFuncSetAttribute(stp_dmma8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM8);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(stp_dmma8_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  if (a.n_elem == 0) return cudaSuccess;
  if (a.n_elem > 0x7fffffffLL) return cudaErrorInvalidValue;
  stp_dmma8_kernel<<<(unsigned)a.n_elem, THREADS8, SMEM8, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}

}  // namespace aderstp
