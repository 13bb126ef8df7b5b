// GPU corrector step and the small device helpers of the GPU time loop.
//
// The reference advances its periodic Cartesian mesh (proj/include/ader/solver.hpp:16-32) after
// the predictor with corrector_step (proj/src/solver.cpp:257-311), one correct_cell per element
// (:184-253):
//   u += V(qavg)                          volume term: one application of the element operator
//                                         Σ_d D_d F_d + B_d D_d (apply_volume_once,
//                                         proj/src/predictor_common.cpp:243-259) on the scaled PDE
//   for d, side:  fhat = ½(f⁺ + f⁻) − ½ smax (q⁻ − q⁺)          (the plus side is the element in
//                 u[line j] += sign φ_side[j] / w_j · (fhat − f_self)   the +d direction)
// with the ScaledPde of an element of size h (flux and ncp × 1/h, smax = max_wavespeed / h,
// solver.cpp:111-156).  Here one CTA corrects one element: qavg is staged in shared memory for the
// volume contraction, the 6 face fluctuations (fhat − f_self) are formed once per face node from
// the element's and its neighbours' predictor faces (L2-resident: every face array is read by its
// owner and one neighbour), and every state entry is updated by one coalesced read-modify-write in
// the state's own layout.  Per-element elastic material (the reference has one material per mesh)
// is supported; smax is then max(cp) of the two elements of a face unless the caller passes one.
// A point source adds its projection times the time integral of its amplitude to its component
// (solver.cpp:206-216), between the volume and the surface terms like the reference.
#include <cstdint>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"

namespace aderstp {

namespace {

constexpr int NVC = 9;

struct CorrParams {
  double d[kMaxOrder * kMaxOrder];
  double phi[2][kMaxOrder];
  double inv_w[kMaxOrder];
  signed char tr[kMaxM][3][kMaxTerms];
  double tc[kMaxM][3][kMaxTerms];
  int m, q_stride, out_stride, layout, par_kind, n_terms;
  int e;         // elements per dimension
  double inv_h;  // grad scale 1 / h
  double smax;   // scaled max wave speed; < 0: elastic, per face from the material
};

// elastic flux table (proj/src/pde.cpp:180-218): F_d(q)_s = coef(s,d) q[in(s,d)]
__constant__ int8_t kInC[NVC][3] = {{6, 7, 8}, {6, 7, 8}, {6, 7, 8}, {7, 6, 0}, {8, 0, 6},
                                    {0, 8, 7}, {0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
__constant__ int8_t kCoefC[NVC][3] = {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {2, 2, 4}, {2, 4, 2},
                                      {4, 2, 2}, {3, 3, 3}, {3, 3, 3}, {3, 3, 3}};

struct Material {
  double c4[5];  // lambda+2mu, lambda, mu, 1/rho, 0
  double cp;
};

__device__ __forceinline__ Material material(const double* pr, int par_kind) {
  double lam, mu, rho;
  if (par_kind == ADERSTP_PAR_RHO_CP_CS) {
    rho = pr[0];
    mu = __dmul_rn(__dmul_rn(pr[0], pr[2]), pr[2]);
    lam = __dsub_rn(__dmul_rn(__dmul_rn(pr[0], pr[1]), pr[1]), __dmul_rn(2.0, mu));
  } else {
    lam = pr[0];
    mu = pr[1];
    rho = pr[2];
  }
  Material mt;
  mt.c4[0] = lam + 2.0 * mu;
  mt.c4[1] = lam;
  mt.c4[2] = mu;
  mt.c4[3] = 1.0 / rho;
  mt.c4[4] = 0.0;
  mt.cp = sqrt((lam + 2.0 * mu) / rho);  // ElasticPde::cp_ (pde.cpp:177)
  return mt;
}

constexpr int kCorrThreads = 512;

// VOL = false: the volume term was already applied by the fused predictor (BatchArgs::u_next),
// only the surface fluctuations remain.
template <int N, bool ELASTIC, bool VOL>
__global__ void __launch_bounds__(kCorrThreads) correct_kernel(CorrParams kp, CorrArgs ca, unsigned int* status) {
  double* __restrict__ u = ca.u;
  const double* __restrict__ par = ca.par;
  const double* __restrict__ qavg = ca.qavg;
  const double* __restrict__ face_q = ca.face_q;
  const double* __restrict__ face_f = ca.face_f;
  constexpr int N2 = N * N, N3 = N * N * N;
  const int m = ELASTIC ? NVC : kp.m;
  extern __shared__ __align__(16) double smc[];
  double* QA = smc;           // qavg [s][k3][k2][k1]
  // quantity planes of QA padded by 8 doubles (different source fields of one warp's rows fall
  // on different bank halves); rows of D padded to N + 1 (per-lane rows k1: conflict free)
  constexpr int QP = N3 + 8, DR = N + 1;
  double* DL = smc + (VOL ? m * QP : 0);  // fhat - f_self  [f][a][b][s]
  __shared__ double Ds[N * DR];     // D (per-thread row indices: shared, not the constant bank)
  __shared__ double SC[2][N];      // sign * phi_side[j] / w_j
  __shared__ double SMAX[6];       // per face
  const int e = kp.e;
  const long long c = blockIdx.x;  // element of this slab
  const int ix = (int)(c % e), iy = (int)((c / e) % e), iz = ca.z0 + (int)(c / ((long long)e * e));
  const int nz = ca.nz > 0 ? ca.nz : e;
  const int tid = threadIdx.x;
  // the neighbour across face (d, step): local, or in the slab below / above (peer memory)
  struct Nb {
    const double* fq;
    const double* ff;
    const double* pr;
    long long idx;
  };
  auto neighbour = [&](int d, int step) -> Nb {
    const int ixn = ((ix + (d == 0 ? step : 0)) % e + e) % e;
    const int iyn = ((iy + (d == 1 ? step : 0)) % e + e) % e;
    const int izn = ((iz + (d == 2 ? step : 0)) % e + e) % e;
    if (izn >= ca.z0 && izn < ca.z0 + nz)
      return {face_q, face_f, par, ((long long)(izn - ca.z0) * e + iyn) * e + ixn};
    const HaloRef& hr = step < 0 ? ca.lo : ca.hi;
    const int lz = ((izn - hr.z_base) % e + e) % e;
    return {hr.face_q, hr.face_f, hr.par, ((long long)lz * e + iyn) * e + ixn};
  };

  Material mine;
  if (ELASTIC) {
    mine = material(par + 3 * c, kp.par_kind);
#pragma unroll
    for (int i = 0; i < 4; ++i) mine.c4[i] *= kp.inv_h;  // ScaledPde: flux x 1/h
  }
  for (int i = tid; i < N * N; i += blockDim.x) Ds[(i / N) * DR + i % N] = kp.d[i];
  if (tid < 2 * N) {
    const int side = tid / N, j = tid - side * N;
    SC[side][j] = (side == 0 ? -1.0 : 1.0) * kp.phi[side][j] * kp.inv_w[j];
  }
  if (tid < 6) {
    const int d = tid >> 1, step = (tid & 1) ? 1 : -1;
    double smax = kp.smax;
    if (ELASTIC && smax < 0.0) {
      const Nb nb = neighbour(d, step);
      smax = fmax(material(par + 3 * c, kp.par_kind).cp, material(nb.pr + 3 * nb.idx, kp.par_kind).cp) * kp.inv_h;
    }
    SMAX[tid] = smax;
  }
  __syncthreads();

  // ---- qavg -> shared (flat over the output layout: coalesced) ----------------------------
  if (VOL) {
    const int os = kp.out_stride;
    const double* qa = qavg + c * (long long)(N3 * os);
    for (int j = tid; j < N3 * os; j += blockDim.x) {
      int s, node;
      if (kp.layout == ADERSTP_LAYOUT_AOSOA) {
        const int k1 = j % N, r = j / N;
        s = r % os;
        node = (r / os) * N + k1;
      } else {
        s = j % os;
        node = j / os;
      }
      if (s < m) QA[s * QP + node] = qa[j];
    }
  }
  // ---- face fluctuations (solver.cpp:218-226) --------------------------------------------
  {
    const int FV = N2 * m;
    const double* mq = face_q + c * 6LL * FV;
    const double* mf = face_f + c * 6LL * FV;
    for (int i = tid; i < 6 * FV; i += blockDim.x) {
      const int f = i / FV, r = i - f * FV;
      const int d = f >> 1, side = f & 1, step = side ? 1 : -1;
      const Nb nb = neighbour(d, step);
      const double* tq = nb.fq + nb.idx * 6LL * FV;
      const double* tf = nb.ff + nb.idx * 6LL * FV;
      double q_plus, q_minus, f_plus, f_minus;
      if (side == 1) {
        q_plus = tq[(2 * d) * FV + r];
        q_minus = mq[(2 * d + 1) * FV + r];
        f_plus = tf[(2 * d) * FV + r];
        f_minus = mf[(2 * d + 1) * FV + r];
      } else {
        q_plus = mq[(2 * d) * FV + r];
        q_minus = tq[(2 * d + 1) * FV + r];
        f_plus = mf[(2 * d) * FV + r];
        f_minus = tf[(2 * d + 1) * FV + r];
      }
      const double fh = 0.5 * (f_plus + f_minus) - 0.5 * SMAX[f] * (q_minus - q_plus);
      DL[i] = fh - mf[f * FV + r];
    }
  }
  __syncthreads();

  // ---- u += V(qavg) + surface terms, in the state's layout ---------------------------------
  unsigned int flags = 0;
  const int qs = kp.q_stride;
  double* ue = u + c * (long long)(N3 * qs);
  for (int j = tid; j < N3 * qs; j += blockDim.x) {
    int s, k1, k2, k3;
    if (kp.layout == ADERSTP_LAYOUT_AOSOA) {
      k1 = j % N;
      const int r = j / N;
      s = r % qs;
      const int k32 = r / qs;
      k2 = k32 % N;
      k3 = k32 / N;
    } else {
      s = j % qs;
      const int node = j / qs;
      k1 = node % N;
      k2 = (node / N) % N;
      k3 = node / N2;
    }
    if (s >= m) continue;
    // volume (apply_volume_once): sum over d of D_d applied to the scaled flux / ncp terms
    double vol = 0.0;
#pragma unroll
    for (int d = 0; d < 3 && VOL; ++d) {
      const int kd = d == 0 ? k1 : d == 1 ? k2 : k3;
      const int stride = d == 0 ? 1 : d == 1 ? N : N2;
      const int base = k3 * N2 + k2 * N + k1 - kd * stride;
      if (ELASTIC) {
        const int cf = kCoefC[s][d];
        if (cf == 4) continue;
        const double cc = cf == 0 ? mine.c4[0] : cf == 1 ? mine.c4[1] : cf == 2 ? mine.c4[2] : mine.c4[3];
        const double* src = QA + kInC[s][d] * QP + base;
        double acc = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) acc = fma(Ds[kd * DR + l], cc * src[l * stride], acc);
        vol += acc;
      } else {
        for (int k = 0; k < kp.n_terms; ++k) {
          const double cc = kp.tc[s][d][k] * kp.inv_h;
          if (cc == 0.0) continue;
          const double* src = QA + kp.tr[s][d][k] * QP + base;
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = fma(Ds[kd * DR + l], cc * src[l * stride], acc);
          vol += acc;
        }
      }
    }
    double val = ue[j] + vol;
    // point source: projection x time integral of the amplitude (solver.cpp:206-216)
    if (s == ca.src_comp) val += ca.src_proj[(k3 * N + k2) * N + k1] * ca.src_sint;
    // surface (solver.cpp:228-249): in-face (a, b) in (z, y, x) order without dimension d
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int kd = d == 0 ? k1 : d == 1 ? k2 : k3;
      const int ab = d == 0 ? k3 * N + k2 : d == 1 ? k3 * N + k1 : k2 * N + k1;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        val += SC[side][kd] * DL[((2 * d + side) * N2 + ab) * m + s];
      }
    }
    if (!isfinite(val)) flags |= 1u;
    ue[j] = val;
  }
  if (flags) atomicOr(status, flags);
}

// Surface-only corrector of the fused time step (elastic, AoSoA state with quantity stride QS,
// even N): the volume term was applied by the fused predictor, so per element only the six face
// fluctuations fhat - f_self (solver.cpp:218-226) and their lifting onto every node
// (solver.cpp:228-249) remain.  HBM-bound (u read + written, every face array read by its owner
// and its neighbour): the neighbour face blocks are resolved once per CTA, the fluctuations are
// formed from 16-byte loads, and the state is updated as k1 pairs with compile-time indexing.
constexpr int kSurfThreads = 256;
// V entries per thread and step: 2 (16-byte pairs) for even N, 1 for odd N
template <int V>
struct VecT;
template <>
struct VecT<1> {
  using T = double;
  __device__ static double& at(T& v, int) { return v; }
};
template <>
struct VecT<2> {
  using T = double2;
  __device__ static double& at(T& v, int i) { return i ? v.y : v.x; }
};

// VOL: also the volume term V(qavg) (the public corrector_step, solver.cpp:257-311): qavg is
// staged in shared memory and the state is walked quantity-major, so that the quantity (and with
// it the flux table entries) is uniform across a warp.
template <int N, bool VOL>
constexpr int surf_threads() { return VOL && N >= 9 ? 512 : kSurfThreads; }  // 1 CTA/SM at N >= 9

// SRC: a point source (compiled only into the instances that need it: the branch alone costs the
// common instance 8 registers and a spill)
template <int N, int QS, bool VOL, bool SRC>
__global__ void __launch_bounds__(surf_threads<N, VOL>()) surface_kernel(CorrParams kp, CorrArgs ca, unsigned int* status) {
  constexpr int NT = surf_threads<N, VOL>();
  constexpr int V = N % 2 == 0 ? 2 : 1;
  using VT = typename VecT<V>::T;
  constexpr int N2 = N * N, N3 = N * N * N, FV = N2 * NVC;
  constexpr int QP = N3 + 8, DR = N + 1;  // padded quantity planes of qavg, padded rows of D
  extern __shared__ __align__(16) double sms[];
  double* DL = sms;            // fhat - f_self  [f][a][b][s]
  double* QA = sms + 6 * FV;   // VOL: qavg [s][k3][k2][k1]
  __shared__ double Ds[VOL ? N * DR : 1];
  __shared__ double SC[2][N];
  __shared__ double SMAX[6];
  __shared__ const double* NBQ[6];
  __shared__ const double* NBF[6];
  const int e = kp.e;
  const long long c = blockIdx.x;
  const int ix = (int)(c % e), iy = (int)((c / e) % e), iz = ca.z0 + (int)(c / ((long long)e * e));
  const int nz = ca.nz > 0 ? ca.nz : e;
  const int tid = threadIdx.x;
  if (tid < 6) {
    const int d = tid >> 1, step = (tid & 1) ? 1 : -1;
    const int ixn = ((ix + (d == 0 ? step : 0)) % e + e) % e;
    const int iyn = ((iy + (d == 1 ? step : 0)) % e + e) % e;
    const int izn = ((iz + (d == 2 ? step : 0)) % e + e) % e;
    const double *fq, *ff, *pr;
    long long idx;
    if (izn >= ca.z0 && izn < ca.z0 + nz) {
      fq = ca.face_q; ff = ca.face_f; pr = ca.par;
      idx = ((long long)(izn - ca.z0) * e + iyn) * e + ixn;
    } else {
      const HaloRef& hr = step < 0 ? ca.lo : ca.hi;
      fq = hr.face_q; ff = hr.face_f; pr = hr.par;
      idx = ((long long)(((izn - hr.z_base) % e + e) % e) * e + iyn) * e + ixn;
    }
    NBQ[tid] = fq + idx * 6LL * FV;
    NBF[tid] = ff + idx * 6LL * FV;
    double smax = kp.smax;
    if (smax < 0.0)
      smax = fmax(material(ca.par + 3 * c, kp.par_kind).cp, material(pr + 3 * idx, kp.par_kind).cp) * kp.inv_h;
    SMAX[tid] = smax;
  }
  if (tid < 2 * N) {
    const int side = tid / N, j = tid - side * N;
    SC[side][j] = (side == 0 ? -1.0 : 1.0) * kp.phi[side][j] * kp.inv_w[j];
  }
  Material mine;
  if (VOL) {
    mine = material(ca.par + 3 * c, kp.par_kind);
#pragma unroll
    for (int i = 0; i < 4; ++i) mine.c4[i] *= kp.inv_h;  // ScaledPde: flux x 1/h
    for (int i = tid; i < N2; i += NT) Ds[(i / N) * DR + i % N] = kp.d[i];
    const double* qa = ca.qavg + c * (long long)(N3 * NVC);
    for (int iv = tid; iv < N3 * NVC / V; iv += NT) {  // [k3][k2][s][k1] -> [s][k3][k2][k1]
      const int k1 = V * (iv % (N / V)), r = iv / (N / V), sq = r % NVC, k32 = r / NVC;
      *reinterpret_cast<VT*>(QA + sq * QP + k32 * N + k1) = *reinterpret_cast<const VT*>(qa + V * iv);
    }
  }
  __syncthreads();
  {  // fluctuations, V face entries per thread and step (V divides FV)
    const double* mq = ca.face_q + c * 6LL * FV;
    const double* mf = ca.face_f + c * 6LL * FV;
    for (int i = V * tid; i < 6 * FV; i += V * NT) {
      const int f = i / FV, r = i - f * FV;
      VT qo = *reinterpret_cast<const VT*>(mq + i), fo = *reinterpret_cast<const VT*>(mf + i);
      VT qn = *reinterpret_cast<const VT*>(NBQ[f] + (f ^ 1) * FV + r);
      VT fn = *reinterpret_cast<const VT*>(NBF[f] + (f ^ 1) * FV + r);
      const double sm = SMAX[f];
      VT dl;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const double a_o = VecT<V>::at(qo, k), a_n = VecT<V>::at(qn, k);
        const double b_o = VecT<V>::at(fo, k), b_n = VecT<V>::at(fn, k);
        // + side: the element is the minus state; - side: the plus state (solver.cpp:218-226)
        VecT<V>::at(dl, k) = (f & 1) ? (0.5 * (b_n + b_o) - 0.5 * sm * (a_o - a_n)) - b_o
                                     : (0.5 * (b_o + b_n) - 0.5 * sm * (a_n - a_o)) - b_o;
      }
      *reinterpret_cast<VT*>(DL + i) = dl;
    }
  }
  __syncthreads();
  unsigned int flags = 0;
  const int qs = QS ? QS : kp.q_stride;  // QS = 0: run-time quantity stride of the state
  double* ue = ca.u + c * (long long)(N3 * qs);
  for (int jv = tid; jv < N3 * NVC / V; jv += NT) {
    // VOL: quantity-major walk (s = jv / (N^3 / V) uniform over runs of N^3 / V threads, so the
    // flux table lookups are warp-uniform); surface only: the state's own order (contiguous)
    int s, k1, k32;
    if (VOL) {
      s = jv / (N3 / V);
      const int rem = jv - s * (N3 / V);
      k1 = V * (rem % (N / V));
      k32 = rem / (N / V);
    } else {
      k1 = V * (jv % (N / V));
      const int r = jv / (N / V);
      s = r % NVC;
      k32 = r / NVC;
    }
    const int k2 = k32 % N, k3 = k32 / N;
    double* up = ue + (k32 * qs + s) * N + k1;
    VT v = *reinterpret_cast<const VT*>(up);
    if (VOL) {  // apply_volume_once (predictor_common.cpp:243-259) on the scaled elastic flux
      double vol[V];
#pragma unroll
      for (int k = 0; k < V; ++k) vol[k] = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int cf = kCoefC[s][d];
        if (cf == 4) continue;
        const double cc = cf == 0 ? mine.c4[0] : cf == 1 ? mine.c4[1] : cf == 2 ? mine.c4[2] : mine.c4[3];
        const double* src = QA + kInC[s][d] * QP;
        double acc[V];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = 0.0;
        if (d == 0) {  // x: the row (k3, k2) is shared by the k1 run
          const double* row = src + k32 * N;
#pragma unroll
          for (int l = 0; l < N; ++l) {
            const double x = cc * row[l];
#pragma unroll
            for (int k = 0; k < V; ++k) acc[k] = fma(Ds[(k1 + k) * DR + l], x, acc[k]);
          }
        } else {       // y (stride N, D row k2) and z (stride N^2, D row k3): k1 runs are contiguous
          const int kd = d == 1 ? k2 : k3, stride = d == 1 ? N : N2;
          const double* col = src + k3 * N2 + k2 * N + k1 - kd * stride;
#pragma unroll
          for (int l = 0; l < N; ++l) {
            VT x = *reinterpret_cast<const VT*>(col + l * stride);
            const double dl = Ds[kd * DR + l];
#pragma unroll
            for (int k = 0; k < V; ++k) acc[k] = fma(dl, cc * VecT<V>::at(x, k), acc[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < V; ++k) vol[k] += acc[k];
      }
#pragma unroll
      for (int k = 0; k < V; ++k) VecT<V>::at(v, k) += vol[k];
    }
    if (SRC && s == ca.src_comp) {  // point source (solver.cpp:206-216), after the volume term
#pragma unroll
      for (int k = 0; k < V; ++k) VecT<V>::at(v, k) += ca.src_proj[k32 * N + k1 + k] * ca.src_sint;
    }
    // x faces: the in-face node (k3, k2) is shared by the k1 run, the lifting differs; y faces
    // (k3, k1) and z faces (k2, k1): per-node fluctuations, shared lifting
    const double dxm = DL[(k3 * N + k2) * NVC + s], dxp = DL[(N2 + k3 * N + k2) * NVC + s];
    const int iy0 = (2 * N2 + k3 * N + k1) * NVC + s, iz0 = (4 * N2 + k2 * N + k1) * NVC + s;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double x = VecT<V>::at(v, k);
      x += SC[0][k1 + k] * dxm;
      x += SC[1][k1 + k] * dxp;
      x += SC[0][k2] * DL[iy0 + k * NVC];
      x += SC[1][k2] * DL[iy0 + N2 * NVC + k * NVC];
      x += SC[0][k3] * DL[iz0 + k * NVC];
      x += SC[1][k3] * DL[iz0 + N2 * NVC + k * NVC];
      if (!isfinite(x)) flags |= 1u;
      VecT<V>::at(v, k) = x;
    }
    *reinterpret_cast<VT*>(up) = v;
  }
  if (flags) atomicOr(status, flags);
}

// (lambda, mu, rho) scaled like ScaledPde(1/h): every flux coefficient x s  ->  (s lambda, s mu, rho / s)
__global__ void scale_par_kernel(const double* __restrict__ in, int par_kind, double s, long long n,
                                 double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double* pr = in + 3 * i;
    double lam, mu, rho;
    if (par_kind == ADERSTP_PAR_RHO_CP_CS) {
      rho = pr[0];
      mu = __dmul_rn(__dmul_rn(pr[0], pr[2]), pr[2]);
      lam = __dsub_rn(__dmul_rn(__dmul_rn(pr[0], pr[1]), pr[1]), __dmul_rn(2.0, mu));
    } else {
      lam = pr[0];
      mu = pr[1];
      rho = pr[2];
    }
    out[3 * i] = lam * s;
    out[3 * i + 1] = mu * s;
    out[3 * i + 2] = rho / s;
  }
}

// max over elements of the P-wave speed, for the time step (stable_dt, solver.cpp:170-174)
__global__ void max_cp_kernel(const double* __restrict__ par, int par_kind, long long n, unsigned long long* out) {
  double best = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    best = fmax(best, material(par + 3 * i, par_kind).cp);
  // non-negative doubles order like their bit patterns
  atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

template <int N>
cudaError_t launch_correct_n(const LaunchPlan& p, const CorrArgs& a, cudaStream_t stream) {
  CorrParams kp;
  const int n = p.n;
  for (int i = 0; i < n * n; ++i) kp.d[i] = p.basis.d[i];
  for (int j = 0; j < n; ++j) {
    kp.phi[0][j] = p.basis.face_left[j];
    kp.phi[1][j] = p.basis.face_right[j];
    kp.inv_w[j] = 1.0 / p.basis.weights[j];
  }
  for (int s = 0; s < kMaxM; ++s)
    for (int d = 0; d < 3; ++d)
      for (int k = 0; k < kMaxTerms; ++k) {
        kp.tr[s][d][k] = p.tr[s][d][k];
        kp.tc[s][d][k] = p.tc[s][d][k];
      }
  kp.m = p.m;
  kp.q_stride = p.q_stride;
  kp.out_stride = p.out_stride;
  kp.layout = p.layout;
  kp.par_kind = p.par_kind;
  kp.n_terms = p.n_terms;
  kp.e = a.e;
  kp.inv_h = a.inv_h;
  kp.smax = a.smax;
  const bool elastic = p.kind == ADERSTP_PDE_ELASTIC;
  const bool vol = a.qavg != nullptr;
  if (elastic && p.layout == ADERSTP_LAYOUT_AOSOA && p.m == NVC && (!vol || p.out_stride == NVC)) {
    // tuned elastic path (any q stride; qavg in the compact AoSoA output layout)
    const size_t ssm = sizeof(double) * (6 * N * N * NVC + (vol ? NVC * (N * N * N + 8) : 0));
    auto sk = vol ? surface_kernel<N, 0, true, false> : surface_kernel<N, 0, false, false>;
    if (p.q_stride == NVC) sk = vol ? surface_kernel<N, NVC, true, false> : surface_kernel<N, NVC, false, false>;
    if (a.src_comp >= 0)  // elastic point source: the volume term is never fused (generic predictor)
      sk = p.q_stride == NVC ? surface_kernel<N, NVC, true, true> : surface_kernel<N, 0, true, true>;
    if (a.src_comp >= 0 && !vol) return cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
    if (err != cudaSuccess) return err;
    const long long cells = (long long)a.e * a.e * (a.nz > 0 ? a.nz : a.e);
    if (cells == 0) return cudaSuccess;
    sk<<<(unsigned)cells, vol ? surf_threads<N, true>() : surf_threads<N, false>(), ssm, stream>>>(kp, a, p.d_status);
    return cudaGetLastError();
  }
  const size_t smem = sizeof(double) * (size_t)p.m * ((vol ? N * N * N + 8 : 0) + 6 * N * N);
  auto kern = elastic ? (vol ? correct_kernel<N, true, true> : correct_kernel<N, true, false>)
                      : (vol ? correct_kernel<N, false, true> : correct_kernel<N, false, false>);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  const long long cells = (long long)a.e * a.e * (a.nz > 0 ? a.nz : a.e);
  kern<<<(unsigned)cells, kCorrThreads, smem, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_correct(const LaunchPlan& p, const CorrArgs& a, cudaStream_t stream) {
  switch (p.n) {
    case 2: return launch_correct_n<2>(p, a, stream);
    case 3: return launch_correct_n<3>(p, a, stream);
    case 4: return launch_correct_n<4>(p, a, stream);
    case 5: return launch_correct_n<5>(p, a, stream);
    case 6: return launch_correct_n<6>(p, a, stream);
    case 7: return launch_correct_n<7>(p, a, stream);
    case 8: return launch_correct_n<8>(p, a, stream);
    case 9: return launch_correct_n<9>(p, a, stream);
    case 10: return launch_correct_n<10>(p, a, stream);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_scale_par(const double* in, int par_kind, double s, long long n, double* out,
                             cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const long long blocks = (n + 255) / 256;
  scale_par_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, stream>>>(in, par_kind, s, n, out);
  return cudaGetLastError();
}

cudaError_t launch_max_cp(const double* par, int par_kind, long long n, unsigned long long* out,
                          cudaStream_t stream) {
  cudaError_t err = cudaMemsetAsync(out, 0, sizeof(unsigned long long), stream);
  if (err != cudaSuccess || n == 0) return err;
  const long long blocks = (n + 255) / 256;
  max_cp_kernel<<<(unsigned)(blocks < 1024 ? blocks : 1024), 256, 0, stream>>>(par, par_kind, n, out);
  return cudaGetLastError();
}

}  // namespace aderstp
