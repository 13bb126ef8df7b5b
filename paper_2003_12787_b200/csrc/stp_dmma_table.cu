// Table PDEs (the user-LinearPde path: any constant-coefficient system given as term tables,
// m <= 9, at most four nonzeros per (row, dim) of A_d + B_d) on the fp64 tensor cores at
// nDof 5..7: the nDof-8 table kernel of stp_dmma8.cu on zero-padded 8 x 8 (k2, k1) planes, the
// padding scheme of the elastic stp_dmmap kernel (stp_dma.cu).
//
// One CTA per element, 8 warps; warp s owns output quantity s (s < 8), a ninth quantity is split
// over the warps by k3 plane (HAS9).  Lane (g, t) owns nodes (k2 = g, k1 = 2t, 2t+1) of every
// plane -- the C fragment of an 8x8 DMMA tile -- and a CK step in Horner form (r <- c_o q + L r,
// stp_dmma8.cu) is
//   t_s = c_o q_s + sum_d sum_k tc[s][d][k] D_d r_{tr[s][d][k]}
// (build_terms folds the ncp matrices in: D_d (A_d + B_d) p for constant coefficients,
// proj/src/stp_splitck.cpp:53-61), every term a pair of DMMAs (x, y; the coefficient folded into
// the D fragments) or register DFMAs (z, D from the constant bank).  Rows / columns k2, k1 >= N of
// the planes and of D are exact zeros, so the padded lanes stay zero and the real nodes see
// exactly the N-term sums; N <= 4 needs one k-step.  favg_d = A_d qavg and face_f = A_d face_q from
// the favg tables; x / y faces by DMMA against the padded phi, z faces by DFMA; face_q and face_f
// leave as TMA bulk stores.
#include <cstdint>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"

extern "C" {
// zero-padded 8 x 8 D per order (row k = node, col l) at offset 64 n, uploaded at plan creation
__constant__ __align__(16) double aderstp_kDT[11 * 64];
}

namespace aderstp {

namespace {

constexpr int TW = 8;              // warps
constexpr int TTHREADS = TW * 32;
constexpr int TGM = 9;             // max quantities

struct ParamsT {
  double d[64];       // zero-padded D (fragments)
  double phi[2][8];   // zero-padded phi(0), phi(1)
  double cf[8];       // cf[o] = dt^(o+1)/(o+1)!
  double tc[TGM][3][kMaxTerms];
  double fc[TGM][3][kMaxTerms];
  signed char tr[TGM][3][kMaxTerms];
  signed char fr[TGM][3][kMaxTerms];
  int m, n_terms, q_stride, check;
};

__device__ __forceinline__ int tphys(int k2, int k1) { return k2 * 8 + (k1 ^ ((k2 & 2) << 1)); }
__device__ __forceinline__ void tdmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 tlds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void tsts2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
__device__ __forceinline__ double tldc(const double* p) {  // constant cache at the point of use
  double v;
  asm volatile("{\n .reg .u64 ca;\n cvta.to.const.u64 ca, %1;\n ld.const.f64 %0, [ca];\n}\n" : "=d"(v) : "l"(p));
  return v;
}

// output node pair (k1 = 2t, 2t+1) of a row: one 16-byte streaming store for even N
template <int N>
__device__ __forceinline__ void tst_pair(double* p, double x, double y, bool ok0, bool ok1) {
  if (N % 2 == 0) {
    if (ok0) asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(x), "d"(y) : "memory");
  } else {
    if (ok0) __stcs(p, x);
    if (ok1) __stcs(p + 1, y);
  }
}

template <int N, int NT>
__device__ __forceinline__ void tmma_x(double (&acc)[NT][2], const double* f, int K0, int g, int t, double b0,
                                       double b1) {
  const double* p0 = f + K0 * 64 + tphys(g, t);
  const double* p1 = f + K0 * 64 + tphys(g, 4 + t);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    tdmma(acc[k][0], acc[k][1], p0[k * 64], b0);
    if (N > 4) tdmma(acc[k][0], acc[k][1], p1[k * 64], b1);
  }
}

template <int N, int NT>
__device__ __forceinline__ void tmma_y(double (&acc)[NT][2], const double* f, int K0, int g, int t, double a0,
                                       double a1) {
  const double* p0 = f + K0 * 64 + tphys(t, g);
  const double* p1 = f + K0 * 64 + tphys(4 + t, g);
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    tdmma(acc[k][0], acc[k][1], a0, p0[k * 64]);
    if (N > 4) tdmma(acc[k][0], acc[k][1], a1, p1[k * 64]);
  }
}

// acc[k][j] += c sum_{l < N} D[K0 + k][l] f[l] on the lane's two columns
template <int N, int NT>
__device__ __forceinline__ void tdfma_z(double (&acc)[NT][2], const double* f, int K0, int col, double c) {
  const double* dz = &aderstp_kDT[N * 64];
#pragma unroll
  for (int l = 0; l < N; ++l) {
    const double2 v = tlds2(f + l * 64 + col);
    const double c0 = c * v.x, c1 = c * v.y;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const double dk = tldc(dz + (K0 + k) * 8 + l);
      acc[k][0] = fma(dk, c0, acc[k][0]);
      acc[k][1] = fma(dk, c1, acc[k][1]);
    }
  }
}

template <int N, bool HAS9>
__global__ void __maxnreg__(N <= 6 ? 64 : 80) stp_dmmat_kernel(ParamsT kp, BatchArgs a, unsigned int* status) {
  constexpr int PL = N * 64;  // one quantity: N planes of 8 x 8
  extern __shared__ __align__(16) double smt[];
  const int m = kp.m, nt = kp.n_terms;
  double* P = smt;           // iterate r [m][N][8][8] swizzled; qavg at the end
  double* Q = smt + m * PL;  // q
  const long long e = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int col = tphys(g, 2 * t);
  unsigned int flags = 0;
  // ---- stage q (AoSoA [k3][k2][s < q_stride][k1]) -> Q = q, P = c_(N-1) q, padding = 0 -------
  {
    const double* qe = a.q + e * (long long)(N * N * N * kp.q_stride);
    const double c0 = kp.cf[N - 1];
    for (int i = tid; i < m * PL; i += TTHREADS) {
      const int s = i / PL, r = i - s * PL, k3 = r >> 6, k2 = (r >> 3) & 7, k1 = r & 7;
      double v = 0.0;
      if (k2 < N && k1 < N) {
        v = __ldcs(qe + ((k3 * N + k2) * kp.q_stride + s) * N + k1);
        if (kp.check && !isfinite(v)) flags |= 1u;
      }
      const int j = s * PL + k3 * 64 + tphys(k2, k1);
      Q[j] = v;
      P[j] = c0 * v;
    }
  }
  __syncthreads();
  const double d0 = kp.d[g * 8 + t], d1 = kp.d[g * 8 + 4 + t];
  const int s = warp;
  const bool own = s < m && s < 8;
  double tt[N][2];
  double t8[1][2] = {{0.0, 0.0}};
  const bool plane8 = HAS9 && warp < N;  // quantity 8: warp w takes plane k3 = w
  // ---- Horner form of the CK series ------------------------------------------------------------
#pragma unroll 1
  for (int o = N - 2; o >= 0; --o) {
    const double co = kp.cf[o];
    if (own) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double2 v = tlds2(Q + s * PL + k * 64 + col);
        tt[k][0] = co * v.x;
        tt[k][1] = co * v.y;
      }
#pragma unroll 1
      for (int k = 0; k < nt; ++k) {
        const double cx = kp.tc[s][0][k], cy = kp.tc[s][1][k], cz = kp.tc[s][2][k];
        if (cx != 0.0) tmma_x<N, N>(tt, P + kp.tr[s][0][k] * PL, 0, g, t, cx * d0, cx * d1);
        if (cy != 0.0) tmma_y<N, N>(tt, P + kp.tr[s][1][k] * PL, 0, g, t, cy * d0, cy * d1);
        if (cz != 0.0) tdfma_z<N, N>(tt, P + kp.tr[s][2][k] * PL, 0, col, cz);
      }
    }
    if (plane8) {
      const double2 v = tlds2(Q + 8 * PL + warp * 64 + col);
      t8[0][0] = co * v.x;
      t8[0][1] = co * v.y;
#pragma unroll 1
      for (int k = 0; k < nt; ++k) {
        const double cx = kp.tc[8][0][k], cy = kp.tc[8][1][k], cz = kp.tc[8][2][k];
        if (cx != 0.0) tmma_x<N, 1>(t8, P + kp.tr[8][0][k] * PL, warp, g, t, cx * d0, cx * d1);
        if (cy != 0.0) tmma_y<N, 1>(t8, P + kp.tr[8][1][k] * PL, warp, g, t, cy * d0, cy * d1);
        if (cz != 0.0) tdfma_z<N, 1>(t8, P + kp.tr[8][2][k] * PL, warp, col, cz);
      }
    }
    __syncthreads();  // every warp has finished reading r
    if (own) {
#pragma unroll
      for (int k = 0; k < N; ++k) tsts2(P + s * PL + k * 64 + col, tt[k][0], tt[k][1]);
    }
    if (plane8) tsts2(P + 8 * PL + warp * 64 + col, t8[0][0], t8[0][1]);
    __syncthreads();  // new r (qavg after the last step) complete
  }
  // ---- epilogue ---------------------------------------------------------------------------
  double* FQ = Q;                  // face_q staging [6][N][N][m] (q is dead)
  const int FACE = N * N * m;
  const bool faces = a.face_q || a.face_f;
  const bool rowok = g < N, k1a = 2 * t < N, k1b = 2 * t + 1 < N;
  const long long vol = (long long)N * N * N * m;
  // qavg and favg of quantity s (compact AoSoA [k3][k2][s][k1]); favg_d[s] = sum fc A_d terms
  auto emit_q = [&](int sq, int k3, double v0, double v1) {
    if (!rowok) return;
    double* qo = a.qavg + e * vol + ((k3 * N + g) * m + sq) * N + 2 * t;
    tst_pair<N>(qo, v0, v1, k1a, k1b);
  };
  if (own) {
#pragma unroll
    for (int k = 0; k < N; ++k) emit_q(s, k, tt[k][0], tt[k][1]);
  }
  if (plane8) emit_q(8, warp, t8[0][0], t8[0][1]);
  if (a.favg) {
    // unit (quantity so, plane k3) over the warps: favg_d[so] = sum_k fc[so][d][k] qavg[fr]
    for (int u = warp; u < m * N; u += TW) {
      const int so = u / N, k3 = u - so * N;
#pragma unroll 1
      for (int d = 0; d < 3; ++d) {
        double f0 = 0.0, f1 = 0.0;
#pragma unroll 1
        for (int kt = 0; kt < nt; ++kt) {
          const double c = kp.fc[so][d][kt];
          if (c == 0.0) continue;
          const double2 v = tlds2(P + kp.fr[so][d][kt] * PL + k3 * 64 + col);
          f0 = fma(c, v.x, f0);
          f1 = fma(c, v.y, f1);
        }
        if (rowok)
          tst_pair<N>(a.favg + e * 3 * vol + d * vol + ((k3 * N + g) * m + so) * N + 2 * t, f0, f1, k1a, k1b);
      }
    }
  }
  if (faces) {
    // x / y faces of (quantity so, plane k3) by DMMA against the padded phi; z faces of quantity
    // so (whole columns) by DFMA
    const double bphi0 = (g < 2) ? kp.phi[g][t] : 0.0, bphi1 = (g < 2) ? kp.phi[g][4 + t] : 0.0;
    for (int u = warp; u < m * N; u += TW) {
      const int so = u / N, k3 = u - so * N;
      const double* qs = P + so * PL;
      double xf[1][2] = {{0.0, 0.0}}, yf[1][2] = {{0.0, 0.0}};
      tmma_x<N, 1>(xf, qs, k3, g, t, bphi0, bphi1);
      tmma_y<N, 1>(yf, qs, k3, g, t, bphi0, bphi1);
      if (t == 0 && g < N) {  // lane (g, 0): C[k2 = g][side]
        FQ[0 * FACE + (k3 * N + g) * m + so] = xf[0][0];
        FQ[1 * FACE + (k3 * N + g) * m + so] = xf[0][1];
      }
      if (g < 2) {  // lane (side = g, t): C[side][k1 = 2t, 2t+1]
        if (k1a) FQ[(2 + g) * FACE + (k3 * N + 2 * t) * m + so] = yf[0][0];
        if (k1b) FQ[(2 + g) * FACE + (k3 * N + 2 * t + 1) * m + so] = yf[0][1];
      }
    }
    for (int so = warp; so < m; so += TW) {
      if (!rowok) continue;
      double z0[2] = {0.0, 0.0}, z1[2] = {0.0, 0.0};
#pragma unroll
      for (int k3 = 0; k3 < N; ++k3) {
        const double2 v = tlds2(P + so * PL + k3 * 64 + col);
        z0[0] = fma(kp.phi[0][k3], v.x, z0[0]);
        z0[1] = fma(kp.phi[0][k3], v.y, z0[1]);
        z1[0] = fma(kp.phi[1][k3], v.x, z1[0]);
        z1[1] = fma(kp.phi[1][k3], v.y, z1[1]);
      }
      if (k1a) {
        FQ[4 * FACE + (g * N + 2 * t) * m + so] = z0[0];
        FQ[5 * FACE + (g * N + 2 * t) * m + so] = z1[0];
      }
      if (k1b) {
        FQ[4 * FACE + (g * N + 2 * t + 1) * m + so] = z0[1];
        FQ[5 * FACE + (g * N + 2 * t + 1) * m + so] = z1[1];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();  // FQ complete; qavg (P) no longer read
    const unsigned bytes = 6u * FACE * 8u;  // 48 N^2 m: a multiple of 16
    if (tid == 0 && a.face_q) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                       a.face_q + e * (long long)(6 * FACE)),
                   "r"((unsigned)__cvta_generic_to_shared(FQ)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    double* FF = P;
    if (a.face_f) {  // face_f[f][ab][so] = sum_k fc[so][d][k] face_q[f][ab][fr[so][d][k]], d = f / 2
      for (int i = tid; i < 6 * FACE; i += TTHREADS) {
        const int fa = i / m, so = i - fa * m, f = fa / (N * N), d = f >> 1;
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

template <int N>
cudaError_t launch_dmmat_n(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  ParamsT kp;
  for (int i = 0; i < 64; ++i) kp.d[i] = 0.0;
  for (int k = 0; k < N; ++k)
    for (int l = 0; l < N; ++l) kp.d[k * 8 + l] = p.basis.d[k * N + l];
  for (int j = 0; j < 8; ++j) {
    kp.phi[0][j] = j < N ? p.basis.face_left[j] : 0.0;
    kp.phi[1][j] = j < N ? p.basis.face_right[j] : 0.0;
  }
  {
    double c = a.dt;  // same operation sequence as proj/src/stp_splitck.cpp:45,64
    for (int o = 0; o < 8; ++o) kp.cf[o] = 0.0;
    kp.cf[0] = c;
    for (int o = 1; o < N; ++o) {
      c *= a.dt / (o + 1);
      kp.cf[o] = c;
    }
  }
  for (int s = 0; s < TGM; ++s)
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
  // the iterate and q (2 m N 64 doubles) hold the face staging too (6 N^2 m <= m N 64)
  const int smem = 2 * p.m * N * 64 * 8;
  auto kern = p.m == TGM ? stp_dmmat_kernel<N, true> : stp_dmmat_kernel<N, false>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  if (a.n_elem == 0) return cudaSuccess;
  if (a.n_elem > 0x7fffffffLL) return cudaErrorInvalidValue;
  kern<<<(unsigned)a.n_elem, TTHREADS, smem, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}

}  // namespace

// table PDEs at nDof 5..7 on the tensor cores: m <= 9, compact AoSoA outputs, no point source
bool dmmat_applicable(const LaunchPlan& p, const BatchArgs& a) {
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  const bool vec = p.n % 2 ? true : (al16(a.q) && al16(a.qavg) && al16(a.favg));  // 16-byte pairs
  // nDof 4 stays on the generic table kernel (measured: it is as fast or faster there, the padded
  // 8 x 8 tiles carry 4x the useful fragment traffic at nDof 4)
  return p.n >= 5 && p.n <= 7 && p.kind != ADERSTP_PDE_ELASTIC && p.kind != ADERSTP_PDE_ELASTIC_SOURCE &&
         p.src_comp < 0 && p.gen.t_ptr == nullptr && p.m >= 1 && p.m <= TGM &&
         p.layout == ADERSTP_LAYOUT_AOSOA && p.out_stride == p.m && p.q_stride >= p.m && p.q_stride <= 64 &&
         p.n_terms <= kMaxTerms && !p.force_generic && !a.u_next && vec && al16(a.face_q) && al16(a.face_f);
}

cudaError_t init_dmmat(const LaunchPlan& p) {
  double buf[64] = {0};
  for (int k = 0; k < p.n; ++k)
    for (int l = 0; l < p.n; ++l) buf[k * 8 + l] = p.basis.d[k * p.n + l];
  return cudaMemcpyToSymbol(aderstp_kDT, buf, sizeof(buf), sizeof(double) * 64 * p.n);
}

cudaError_t launch_dmmat(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  switch (p.n) {
    case 5: return launch_dmmat_n<5>(p, a, stream);
    case 6: return launch_dmmat_n<6>(p, a, stream);
    case 7: return launch_dmmat_n<7>(p, a, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace aderstp
