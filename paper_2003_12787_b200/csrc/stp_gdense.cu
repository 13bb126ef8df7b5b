// Dense user LinearPde at nDof 8 on the fp64 tensor cores (sm_100a DMMA, mma.sync m8n8k4 f64).
//
// The systems the term-table kernels cannot take (more than four nonzeros in a row of A_d + B_d,
// or m > 16 -- the paper's application size is m = 21) run the reference's SplitCK
// recursion (proj/src/stp_splitck.cpp:13-81) on a constant-coefficient LinearPde
// (proj/include/ader/pde.hpp:21-46).  For constant coefficients a CK step is
//   L r = sum_d D_d F_d(r) + B_d (D_d r) = sum_d C_d (D_d r),   C_d = A_d + B_d   (x ScaledPde 1/h),
// i.e. three derivative fields per quantity and then, at every node, one dense m x 3m matrix
// [C_x | C_y | C_z] applied to the 3m derivatives: a GEMM of M = m targets, K = 3m, N = nodes.
// The generic kernel (stp_general.cu) does that product with scalar FMAs (fp64 pipe ~10 %); here
// it is a DMMA GEMM per k3 plane with the A operand (the scaled C rows) resident in registers:
//
//   phase Z (once per step): Rn[j][k3] = sum_l D[k3][l] Rc[j][l]   register DFMA per z column,
//            into the buffer that receives the new iterate (a plane's z derivatives are dead once
//            that plane's new iterate is known)
//   per plane k3:
//     XY   : Gx[j], Gy[j] of the plane   two DMMAs per quantity (x: A = Rc slice, B = D^T;
//            y: A = D, B = Rc slice), C fragments to the G rows (double-buffered by plane)
//     GEMM : T[s][node] = c_o q[s][node] + sum_kk Call[s][kk] G[kk][node], kk = d m + j:
//            warp (mt, nq) owns target tile mt (8 quantities) and node tiles nq, nq + 4; the
//            K loop reads the B fragments from G (x, y rows) and Rn (z rows); q from tensor memory
//     the plane's T goes into Rn after the next barrier (one barrier per plane)
//   Horner form r <- c_o q + L r (o = 6 .. 0, from r = c_7 q; stp_dmma8.cu), the last iterate is
//   qavg; favg_d = A_d qavg and face_f = A_d face_q are DMMA GEMMs as well (A_d rows in registers),
//   face_q are line tasks (both sides of a line from one load of it).
//
// Shared memory: Rc, Rn (m x 8 planes x 64, XOR-swizzled rows as stp_dmma8.cu, quantities at qb(j))
// and two G buffers (2 x 4 ceil(m/4) rows of 68 doubles): m = 21 uses 229,888 of 232,448 bytes,
// one CTA of 12 warps per SM.  A 64-bit shared access is served per half-warp
// (lanes g = 0..3 or 4..7, t = 0..3): the B fragments of the GEMMs (4 rows t x 4 columns g) are
// conflict free because the G row stride is 4 mod 16 doubles and qb spreads the z rows (measured
// with strides 72 / 520, 8 mod 16: twice the ideal wavefronts).
#include <cstdint>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"
#include "tmem.cuh"

namespace aderstp {

namespace {

// quantity j starts at qb(j) = 528 j + {0, 8, 4, 12}[j % 4] doubles: four consecutive quantities
// (the rows t of a GEMM B fragment) fall on distinct 4-double bank groups, two consecutive ones
// (the T stores of lanes g, g + 1 in one quarter-warp) 8 doubles apart
constexpr int GD_PS = 528;
__host__ __device__ constexpr int qb(int j) { return j * GD_PS + ((j & 1) << 3) + ((j & 2) << 1); }
__host__ __device__ constexpr int gd_qsz(int m) { return m * GD_PS + 16; }  // one iterate buffer
constexpr int GD_RS = 68;   // doubles per G row (one plane of one derivative field)
constexpr int kGdMaxM = 21;  // the iterate pair and the G buffers fit in 227 KB up to m = 21

struct GdParams {
  double d[64];        // d[k*8+l] = phi_l'(x_k)
  double phi[2][8];    // phi(0), phi(1)
  double cf[8];        // Horner coefficients c_o = dt^(o+1)/(o+1)! (stp_splitck.cpp:45,64)
  const double* c_dense;  // C_d = A_d + B_d, [d][j][s < mp]
  const double* f_dense;  // A_d, [d][j][s < mp]
  double scale;        // ScaledPde gradient scale (1 outside the time loop)
  int m, mp, q_stride, out_stride, layout, check;
};

__device__ __forceinline__ int gphys(int k2, int k1) { return k2 * 8 + (k1 ^ ((k2 & 2) << 1)); }

__device__ __forceinline__ void gdmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ long long glidx(int layout, int stride, int s, int k3, int k2, int k1) {
  return layout == ADERSTP_LAYOUT_AOSOA ? ((long long)(k3 * 8 + k2) * stride + s) * 8 + k1
                                        : ((long long)(k3 * 8 + k2) * 8 + k1) * stride + s;
}

__device__ __forceinline__ double lds_a(uint32_t addr) {  // shared load by 32-bit window address
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double2 glds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void gsts2(double* p, double x, double y) {
  *reinterpret_cast<double2*>(p) = make_double2(x, y);
}

// z derivatives of one quantity, output planes 4H .. 4H+3, on this lane's column pair
template <int H>
__device__ __forceinline__ void z_half(const GdParams& kp, const double* src, double* dst) {
  double2 v[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) v[l] = glds2(src + l * 64);
#pragma unroll
  for (int k = 4 * H; k < 4 * H + 4; ++k) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      a0 = fma(kp.d[k * 8 + l], v[l].x, a0);
      a1 = fma(kp.d[k * 8 + l], v[l].y, a1);
    }
    gsts2(dst + k * 64, a0, a1);
  }
}

// C fragment (row s, nodes (k2, 2t), (k2, 2t+1) of plane k3) to an output array
__device__ __forceinline__ void gst_pair(double* base, const GdParams& kp, int stride, int s, int k3, int k2,
                                         int k1, double x, double y) {
  if (kp.layout == ADERSTP_LAYOUT_AOSOA) {
    double* p = base + glidx(kp.layout, stride, s, k3, k2, k1);
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(x), "d"(y) : "memory");
    } else {
      __stcs(p, x);
      __stcs(p + 1, y);
    }
  } else {
    __stcs(base + glidx(kp.layout, stride, s, k3, k2, k1), x);
    __stcs(base + glidx(kp.layout, stride, s, k3, k2, k1 + 1), y);
  }
}

template <int MT>
constexpr int gd_tcols() { return MT == 1 ? 64 : MT == 2 ? 128 : 256; }

// KPD = ceil(m / 4) k-steps per direction: the K rows of the CK GEMM are [x | y | z] blocks of
// MP4 = 4 KPD rows each (rows j >= m: zero A), so every k-step lies in one direction and all its
// row offsets are compile-time immediates.  MT = ceil(KPD / 2) target tiles of 8 quantities,
// 4 MT warps.
template <int KPD>
__global__ void __launch_bounds__(128 * ((KPD + 1) / 2), 1)
stp_gdense_kernel(GdParams kp, BatchArgs a, unsigned int* status) {
  constexpr int MT = (KPD + 1) / 2, MP4 = 4 * KPD;
  constexpr int W = 4 * MT;
  constexpr int KSMAX = 3 * KPD;
  constexpr int KF = KPD;  // k-steps of the favg / face_f GEMMs
  extern __shared__ __align__(16) double smd[];
  __shared__ uint32_t tmem_base_s;
  const int m = kp.m;
  const long long e = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int mt = warp >> 2, nq = warp & 3;
  const int s = mt * 8 + g;  // this lane's target quantity in the GEMM tiles
  const bool sok = s < m;
  const int nt0 = nq, nt1 = nq + 4;
  double* R0 = smd;
  double* R1 = smd + gd_qsz(m);
  double* GB = smd + 2 * gd_qsz(m);  // two G buffers of 2m rows
  constexpr int gbuf = 2 * MP4 * GD_RS;
  unsigned int flags = 0;

  if (warp == 0) tm_alloc<gd_tcols<MT>()>(&tmem_base_s);

  // A fragments of the CK GEMM: k-step ks = d KPD + i, lane (g, t) holds scale C_d[s][j],
  // j = 4 i + t (the table entry [d m + j][s]); zero for s >= m or j >= m
  double af[KSMAX];
#pragma unroll
  for (int ks = 0; ks < KSMAX; ++ks) {
    const int d = ks / KPD, j = 4 * (ks % KPD) + t;
    af[ks] = (sok && j < m) ? kp.scale * __ldg(kp.c_dense + (d * m + j) * kp.mp + s) : 0.0;
  }
  // the G rows j >= m of both directions and buffers stay zero (finite B for the zero A)
  for (int i = tid; i < 2 * 2 * (MP4 - m) * GD_RS; i += W * 32) {
    const int r = i / GD_RS, c = i - r * GD_RS;  // r = (buffer, direction, pad row)
    const int pr = r % (MP4 - m), bd = r / (MP4 - m);
    GB[(bd * MP4 + m + pr) * GD_RS + c] = 0.0;
  }
  const double d0 = kp.d[g * 8 + t], d1 = kp.d[g * 8 + 4 + t];  // D fragments (XY phase)

  tm_fence_before();
  __syncthreads();  // the TMEM base address is visible
  tm_fence_after();
  // q of this lane's GEMM positions: 8 planes x 2 node tiles x 2 doubles = 64 TMEM columns
  const uint32_t tq = tmem_base_s + ((uint32_t)(32 * nq) << 16) + (uint32_t)(64 * mt);

  // ---- stage q: R0 = c_7 q (every (s < m, node) exactly once over the CTA), TMEM = q ----------
  {
    const double* qe = a.q + e * (512ll * kp.q_stride);
    const double c7 = kp.cf[7];
#pragma unroll
    for (int k3 = 0; k3 < 8; ++k3) {
      uint32_t r[8];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int nt = i ? nt1 : nt0;
        double v0 = 0.0, v1 = 0.0;
        if (sok) {
          v0 = __ldcs(qe + glidx(kp.layout, kp.q_stride, s, k3, nt, 2 * t));
          v1 = __ldcs(qe + glidx(kp.layout, kp.q_stride, s, k3, nt, 2 * t + 1));
          if (kp.check && !(isfinite(v0) && isfinite(v1))) flags |= 1u;
          gsts2(R0 + qb(s) + k3 * 64 + gphys(nt, 2 * t), c7 * v0, c7 * v1);
        }
        tm_split(v0, r, 2 * i);
        tm_split(v1, r, 2 * i + 1);
      }
      tm_st8(tq + 8 * k3, r);
    }
    tm_wait_st();
  }
  __syncthreads();

  // ---- CK series, Horner form --------------------------------------------------------------
  double* Rc = R0;
  double* Rn = R1;
  const int zcol = gphys(lane >> 2, 2 * (lane & 3));  // phase Z: this lane's column pair
#pragma unroll 1
  for (int o = 6; o >= 0; --o) {
    const double co = kp.cf[o];
    // phase Z: tasks (quantity j, half h of the output planes)
#pragma unroll 1
    for (int task = warp; task < 2 * m; task += W) {
      const int j = task >> 1;
      if (task & 1)
        z_half<1>(kp, Rc + qb(j) + zcol, Rn + qb(j) + zcol);
      else
        z_half<0>(kp, Rc + qb(j) + zcol, Rn + qb(j) + zcol);
    }
    __syncthreads();
    double tp[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // T of the previous plane
#pragma unroll 1
    for (int k3 = 0; k3 < 8; ++k3) {
      double* G = GB + (k3 & 1) * gbuf;
      // XY: G[d m + j] = D_d Rc[j] on plane k3
#pragma unroll 1
      for (int task = warp; task < 2 * m; task += W) {
        const bool y = task >= m;
        const double* pl = Rc + qb(task - (y ? m : 0)) + k3 * 64;
        double c0 = 0.0, c1 = 0.0;
        if (!y) {
          gdmma(c0, c1, pl[gphys(g, t)], d0);
          gdmma(c0, c1, pl[gphys(g, 4 + t)], d1);
        } else {
          gdmma(c0, c1, d0, pl[gphys(t, g)]);
          gdmma(c0, c1, d1, pl[gphys(4 + t, g)]);
        }
        gsts2(G + (task + (y ? MP4 - m : 0)) * GD_RS + g * 8 + 2 * t, c0, c1);
      }
      __syncthreads();  // G of plane k3 complete; every read of plane k3-1's z rows is done
      if (k3 > 0 && sok) {
        double* dst = Rn + qb(s) + (k3 - 1) * 64;
        gsts2(dst + gphys(nt0, 2 * t), tp[0][0], tp[0][1]);
        gsts2(dst + gphys(nt1, 2 * t), tp[1][0], tp[1][1]);
      }
      double acc[2][2];
      {
        uint32_t r[8];
        tm_ld8(tq + 8 * k3, r);
        tm_wait_ld();
        acc[0][0] = co * tm_double(r, 0);
        acc[0][1] = co * tm_double(r, 1);
        acc[1][0] = co * tm_double(r, 2);
        acc[1][1] = co * tm_double(r, 3);
      }
      // B operand: k-step ks = d KPD + i reads row 4 i + t of direction d -- G rows (x, y) or the
      // z rows in Rn; every offset is a compile-time immediate on three per-lane bases (the z
      // padding rows j >= m, only in the last k-step, read row t instead: A is zero there)
      const uint32_t gx0 = (uint32_t)__cvta_generic_to_shared(G + t * GD_RS + nt0 * 8 + g);
      const uint32_t rz0 = (uint32_t)__cvta_generic_to_shared(Rn + qb(t) + k3 * 64 + gphys(nt0, g));
      const uint32_t rz1 = (uint32_t)__cvta_generic_to_shared(Rn + qb(t) + k3 * 64 + gphys(nt1, g));
      const bool zpad = 4 * (KPD - 1) + t >= m;
#pragma unroll
      for (int ks = 0; ks < KSMAX; ++ks) {
        const int d = ks / KPD, i = ks % KPD;
        uint32_t a0, a1;
        if (d < 2) {
          a0 = gx0 + 8u * (uint32_t)((d * MP4 + 4 * i) * GD_RS);
          a1 = a0 + 8u * 32u;  // node tile nt0 + 4: 32 doubles on
        } else {
          const uint32_t oz = 8u * (uint32_t)(4 * i * GD_PS);
          const bool pad = i == KPD - 1 && zpad;  // z padding row: row t instead (A is zero)
          a0 = pad ? rz0 : rz0 + oz;
          a1 = pad ? rz1 : rz1 + oz;
        }
        gdmma(acc[0][0], acc[0][1], af[ks], lds_a(a0));
        gdmma(acc[1][0], acc[1][1], af[ks], lds_a(a1));
      }
      tp[0][0] = acc[0][0];
      tp[0][1] = acc[0][1];
      tp[1][0] = acc[1][0];
      tp[1][1] = acc[1][1];
    }
    __syncthreads();  // every read of plane 7's z rows is done
    if (sok) {
      double* dst = Rn + qb(s) + 7 * 64;
      gsts2(dst + gphys(nt0, 2 * t), tp[0][0], tp[0][1]);
      gsts2(dst + gphys(nt1, 2 * t), tp[1][0], tp[1][1]);
    }
    __syncthreads();  // the new iterate is complete
    double* sw = Rc;
    Rc = Rn;
    Rn = sw;
  }
  // every TMEM read has completed (tcgen05.wait::ld); the allocating warp frees the columns
  tm_fence_before();
  __syncthreads();
  if (warp == 0) {
    tm_fence_after();
    tm_dealloc<gd_tcols<MT>()>(tmem_base_s);
  }

  // ---- epilogue: Rc = qavg ---------------------------------------------------------------
  const int os = kp.out_stride;
  {  // qavg in output order (padding slots s >= m as zeros, like the reference's PredictorOutput)
    double* qo = a.qavg + e * (512ll * os);
    for (int i = tid; i < 512 * os; i += W * 32) {
      int so, k3, k2, k1;
      if (kp.layout == ADERSTP_LAYOUT_AOSOA) {
        k1 = i & 7;
        const int r = i >> 3;
        so = r % os;
        const int k32 = r / os;
        k3 = k32 >> 3;
        k2 = k32 & 7;
      } else {
        so = i % os;
        const int node = i / os;
        k3 = node >> 6;
        k2 = (node >> 3) & 7;
        k1 = node & 7;
      }
      __stcs(qo + i, so < m ? Rc[qb(so) + k3 * 64 + gphys(k2, k1)] : 0.0);
    }
  }
  // A_d fragments (scaled): lane (g, t) holds A_d[s][j = 4 ks + t]
  auto load_fd = [&](int d, double (&fa)[KF]) {
#pragma unroll
    for (int ks = 0; ks < KF; ++ks) {
      const int j = 4 * ks + t;
      fa[ks] = (sok && j < m) ? kp.scale * __ldg(kp.f_dense + (d * m + j) * kp.mp + s) : 0.0;
    }
  };
  if (a.favg) {  // favg_d = A_d qavg (stp_splitck.cpp:72-78): per plane, tiles (mt, nq / nq + 4)
    double* fo = a.favg + e * (3 * 512ll * os);
#pragma unroll 1
    for (int d = 0; d < 3; ++d) {
      double fa[KF];
      load_fd(d, fa);
#pragma unroll 1
      for (int k3 = 0; k3 < 8; ++k3) {
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        const double* b0p = Rc + k3 * 64 + gphys(nt0, g);
        const double* b1p = Rc + k3 * 64 + gphys(nt1, g);
#pragma unroll
        for (int ks = 0; ks < KF; ++ks) {
          const int j = 4 * ks + t < m ? 4 * ks + t : t < m ? t : 0;  // padding: a real row
          gdmma(acc[0][0], acc[0][1], fa[ks], b0p[qb(j)]);
          gdmma(acc[1][0], acc[1][1], fa[ks], b1p[qb(j)]);
        }
        if (sok) {
          gst_pair(fo + d * (512ll * os), kp, os, s, k3, nt0, 2 * t, acc[0][0], acc[0][1]);
          gst_pair(fo + d * (512ll * os), kp, os, s, k3, nt1, 2 * t, acc[1][0], acc[1][1]);
        }
      }
    }
    if (os > m)  // padding slots
      for (int i = tid; i < 3 * 512 * (os - m); i += W * 32) {
        const int per = 512 * (os - m), d = i / per, r = i - d * per;
        const int node = r / (os - m), so = m + r % (os - m);
        fo[d * (512ll * os) + glidx(kp.layout, os, so, node >> 6, (node >> 3) & 7, node & 7)] = 0.0;
      }
  }
  if (a.face_q || a.face_f) {
    // face_q (predictor_common.cpp:311-341), staged as rows F[f m + s][ab] over the dead Rn:
    // task (s, k3) contracts plane k3 of quantity s against phi by DMMA for the x normal
    // (C[k2][side], B = phi^T zero-padded to 8 columns) and the y normal (C[side][k1], A = phi);
    // task (s, z) the z normal by FMAs on the lane's own column pair.
    double* F = Rn;
    const int FACE = 64 * m;
    double* fq = a.face_q ? a.face_q + e * 6ll * FACE : nullptr;
    const double ph0 = g < 2 ? kp.phi[g][t] : 0.0, ph1 = g < 2 ? kp.phi[g][4 + t] : 0.0;
#pragma unroll 1
    for (int task = warp; task < 9 * m; task += W) {
      if (task < 8 * m) {
        const int so = task >> 3, k3 = task & 7;
        const double* pl = Rc + qb(so) + k3 * 64;
        double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
        gdmma(x0, x1, pl[gphys(g, t)], ph0);
        gdmma(x0, x1, pl[gphys(g, 4 + t)], ph1);
        gdmma(y0, y1, ph0, pl[gphys(t, g)]);
        gdmma(y0, y1, ph1, pl[gphys(4 + t, g)]);
        if (t == 0) {  // x faces: lane (g, 0) holds sides 0, 1 at (k3, k2 = g)
          const int line = k3 * 8 + g;
          F[(0 * m + so) * GD_RS + line] = x0;
          F[(1 * m + so) * GD_RS + line] = x1;
          if (fq) {
            __stcs(fq + 0 * FACE + line * m + so, x0);
            __stcs(fq + 1 * FACE + line * m + so, x1);
          }
        }
        if (g < 2) {  // y faces: lane (g < 2, t) holds side g at (k3, k1 = 2t, 2t + 1)
          const int f = 2 + g, line = k3 * 8 + 2 * t;
          gsts2(F + (f * m + so) * GD_RS + line, y0, y1);
          if (fq) {
            __stcs(fq + f * FACE + line * m + so, y0);
            __stcs(fq + f * FACE + (line + 1) * m + so, y1);
          }
        }
      } else {
        const int so = task - 8 * m;
        const double* col = Rc + qb(so) + zcol;
        double f0a = 0.0, f0b = 0.0, f1a = 0.0, f1b = 0.0;
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const double2 v = glds2(col + l * 64);
          f0a = fma(kp.phi[0][l], v.x, f0a);
          f0b = fma(kp.phi[0][l], v.y, f0b);
          f1a = fma(kp.phi[1][l], v.x, f1a);
          f1b = fma(kp.phi[1][l], v.y, f1b);
        }
        const int line = (lane >> 2) * 8 + 2 * (lane & 3);  // (k2, k1) of the column pair
        gsts2(F + (4 * m + so) * GD_RS + line, f0a, f0b);
        gsts2(F + (5 * m + so) * GD_RS + line, f1a, f1b);
        if (fq) {
          __stcs(fq + 4 * FACE + line * m + so, f0a);
          __stcs(fq + 4 * FACE + (line + 1) * m + so, f0b);
          __stcs(fq + 5 * FACE + line * m + so, f1a);
          __stcs(fq + 5 * FACE + (line + 1) * m + so, f1b);
        }
      }
    }
    if (a.face_f) {
      __syncthreads();
      // face_f[f] = A_d face_q[f] (d = f / 2): tiles (s, ab) from the staged rows
      double* ff = a.face_f + e * 6ll * FACE;
#pragma unroll 1
      for (int d = 0; d < 3; ++d) {
        double fa[KF];
        load_fd(d, fa);
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
          const int f = 2 * d + side;
          double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
          const double* b0p = F + f * m * GD_RS + nt0 * 8 + g;
          const double* b1p = F + f * m * GD_RS + nt1 * 8 + g;
#pragma unroll
          for (int ks = 0; ks < KF; ++ks) {
            const int j = 4 * ks + t < m ? 4 * ks + t : t < m ? t : 0;  // padding: a real row
            gdmma(acc[0][0], acc[0][1], fa[ks], b0p[j * GD_RS]);
            gdmma(acc[1][0], acc[1][1], fa[ks], b1p[j * GD_RS]);
          }
          if (sok) {
            double* base = ff + f * FACE + s;
            __stcs(base + (nt0 * 8 + 2 * t) * m, acc[0][0]);
            __stcs(base + (nt0 * 8 + 2 * t + 1) * m, acc[0][1]);
            __stcs(base + (nt1 * 8 + 2 * t) * m, acc[1][0]);
            __stcs(base + (nt1 * 8 + 2 * t + 1) * m, acc[1][1]);
          }
        }
      }
    }
  }
  if (kp.check && flags) atomicOr(status, flags);
}

template <int KPD>
cudaError_t launch_gd(const GdParams& kp, const BatchArgs& a, unsigned int* status, cudaStream_t stream) {
  const size_t smem = sizeof(double) * (2 * (size_t)gd_qsz(kp.m) + 4 * (size_t)(4 * KPD) * GD_RS);
  cudaError_t err = cudaFuncSetAttribute(stp_gdense_kernel<KPD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  stp_gdense_kernel<KPD><<<(unsigned)a.n_elem, 128 * ((KPD + 1) / 2), smem, stream>>>(kp, a, status);
  return cudaGetLastError();
}

}  // namespace

bool gdense_applicable(const LaunchPlan& p, const BatchArgs& a) {
  return p.n == 8 && !p.no_gdense && !p.force_generic && p.gen.t_dense && p.gen.f_dense && p.m >= 1 &&
         p.m <= kGdMaxM && p.src_comp < 0 && a.u_next == nullptr && a.vol_r == nullptr && a.qavg != nullptr;
}

cudaError_t launch_gdense(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  GdParams kp;
  for (int i = 0; i < 64; ++i) kp.d[i] = p.basis.d[i];
  for (int j = 0; j < 8; ++j) {
    kp.phi[0][j] = p.basis.face_left[j];
    kp.phi[1][j] = p.basis.face_right[j];
  }
  {
    double c = a.dt;  // the reference's sequence (stp_splitck.cpp:45,64)
    kp.cf[0] = c;
    for (int o = 1; o < 8; ++o) {
      c *= a.dt / (o + 1);
      kp.cf[o] = c;
    }
  }
  kp.c_dense = p.gen.t_dense;
  kp.f_dense = p.gen.f_dense;
  kp.scale = p.gen.scale;
  kp.m = p.m;
  kp.mp = (p.m + 7) / 8 * 8;
  kp.q_stride = p.q_stride;
  kp.out_stride = p.out_stride;
  kp.layout = p.layout;
  kp.check = p.check;
  if (a.n_elem == 0) return cudaSuccess;
  if (a.n_elem > 0x7fffffffLL) return cudaErrorInvalidValue;
  switch ((p.m + 3) / 4) {
    case 1: return launch_gd<1>(kp, a, p.d_status, stream);
    case 2: return launch_gd<2>(kp, a, p.d_status, stream);
    case 3: return launch_gd<3>(kp, a, p.d_status, stream);
    case 4: return launch_gd<4>(kp, a, p.d_status, stream);
    case 5: return launch_gd<5>(kp, a, p.d_status, stream);
    case 6: return launch_gd<6>(kp, a, p.d_status, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace aderstp
