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

// Even/odd derivative operator per order (uploaded once per device at plan creation):
// [A: h x (h+1)][B: h x h][M: h+1] with h = n/2, stored at offset order*64.
extern "C" {
__constant__ double aderstp_kEO[11 * 64];
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
// flux table for favg / face_f: F_d(q)_s = coef(s,d) q[in(s,d)], coef 4 = 0
__constant__ int8_t kInE[NVE][3] = {{6, 7, 8}, {6, 7, 8}, {6, 7, 8}, {7, 6, 0}, {8, 0, 6},
                                    {0, 8, 7}, {0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
__constant__ int8_t kCoefE[NVE][3] = {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {2, 2, 4}, {2, 4, 2},
                                      {4, 2, 2}, {3, 3, 3}, {3, 3, 3}, {3, 3, 3}};

template <int N>
struct Geo {
  static constexpr int H = N / 2;
  static constexpr int RS = (N % 2 == 0) ? N + 1 : N;  // odd row stride: conflict-free lines
  static constexpr int PL = N * RS;                    // k3 plane
  static constexpr int VS = N * PL;                    // one quantity
  static constexpr int ES = NVE * VS;                  // one tensor
  static constexpr int LINES = N * N;
  static constexpr int TASKS = 6 * LINES;              // per element per pass
  static constexpr int EPB = N <= 2 ? 16 : N == 3 ? 8 : N <= 4 ? 4 : N <= 6 ? 2 : 1;
  static constexpr int THREADS = ((TASKS * EPB + 31) / 32) * 32;
  static constexpr int OUTV = NVE * N * N * N;         // qavg values per element
  static constexpr int QPT = (OUTV * EPB + THREADS - 1) / THREADS;  // qavg values per thread
  static constexpr int FQV = 6 * N * N * NVE;                        // face staging
  static constexpr int EB = ES + (ES > FQV ? ES : FQV);             // per-element doubles
  static constexpr int SMEM = EB * EPB * 8;
  static constexpr int MINB = N >= 10 ? 1 : 2;
};

__device__ __forceinline__ double ceo(int i) {
  double v;
  asm volatile("{\n .reg .u64 ca;\n cvta.to.const.u64 ca, %1;\n ld.const.f64 %0, [ca];\n}\n"
               : "=d"(v)
               : "l"(&aderstp_kEO[i]));
  return v;
}

__device__ __forceinline__ double pick4(const double c[4], int i) {
  return i == 0 ? c[0] : i == 1 ? c[1] : i == 2 ? c[2] : c[3];
}

// out[k] = sum_l D[k][l] p[l] via the even/odd split; p is overwritten.
template <int N>
__device__ __forceinline__ void eo_apply(double (&p)[N], double (&out)[N]) {
  constexpr int H = N / 2;
  const int base = N * 64;
  double e[H + 1], o[H];
#pragma unroll
  for (int l = 0; l < H; ++l) {
    e[l] = p[l] + p[N - 1 - l];
    o[l] = p[l] - p[N - 1 - l];
  }
  if (N % 2) e[H] = p[H];
#pragma unroll
  for (int k = 0; k < H; ++k) {
    double al = 0.0, be = 0.0;
#pragma unroll
    for (int l = 0; l < H + (N % 2); ++l) al = fma(ceo(base + k * (H + 1) + l), e[l], al);
#pragma unroll
    for (int l = 0; l < H; ++l) be = fma(ceo(base + H * (H + 1) + k * H + l), o[l], be);
    out[k] = al + be;
    out[N - 1 - k] = be - al;
  }
  if (N % 2) {
    double mid = 0.0;
#pragma unroll
    for (int l = 0; l < H; ++l) mid = fma(ceo(base + H * (H + 1) + H * H + l), o[l], mid);
    out[H] = fma(ceo(base + H * (H + 1) + H * H + H), e[H], mid);
  }
}

template <int N>
struct PassParams {
  double phi[2][N];
  int check, par_kind, q_stride;
};

template <int N>
__global__ void __launch_bounds__(Geo<N>::THREADS, Geo<N>::MINB)
stp_pass_kernel(PassParams<N> kp, BatchArgs a, unsigned int* status) {
  using G = Geo<N>;
  extern __shared__ __align__(16) double smp[];
  const int tid = threadIdx.x;
  unsigned int flags = 0;
  const double dt = a.dt;
  const long long e0 = (long long)blockIdx.x * G::EPB;

  // task of this thread in every pass: element el, source slot, line index
  const int task = tid;
  const int el = task / G::TASKS;
  const int slot = (task - el * G::TASKS) / G::LINES;
  const int line = task - el * G::TASKS - slot * G::LINES;
  const bool active = el < G::EPB && e0 + el < a.n_elem;
  const int la = line / N, lb = line - la * N;  // line = la * N + lb

  // material of the task's element (proj/src/pde.cpp:171-178)
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

  // ---- stage q (AoSoA [k3][k2][s < QS][k1]) -> P, qavg registers = dt q ----------------
  // flat qavg ownership in output order [e][k3][k2][s][k1]: entry i = tid + j * THREADS
  double qa[G::QPT];
  {
    const int qs = kp.q_stride;
    for (int i = tid; i < G::EPB * N * N * qs * N; i += G::THREADS) {
      const int ee = i / (N * N * qs * N);
      int r = i - ee * (N * N * qs * N);
      const int k1 = r % N;
      r /= N;
      const int s = r % qs;
      r /= qs;
      if (s >= NVE || e0 + ee >= a.n_elem) continue;
      const double v = __ldcs(a.q + (e0 + ee) * (long long)(N * N * qs * N) + (i - ee * (N * N * qs * N)));
      if (kp.check && !isfinite(v)) flags |= 1u;
      smp[ee * G::EB + s * G::VS + (r / N) * G::PL + (r % N) * G::RS + k1] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < G::QPT; ++j) {
    const int i = tid + j * G::THREADS;
    double v = 0.0;
    if (i < G::EPB * G::OUTV) {
      const int ee = i / G::OUTV;
      int r = i - ee * G::OUTV;
      const int k1 = r % N;
      r /= N;
      const int s = r % NVE;
      r /= NVE;
      v = dt * smp[ee * G::EB + s * G::VS + (r / N) * G::PL + (r % N) * G::RS + k1];
    }
    qa[j] = v;
  }

  // buffers of element ee: B(ee, 0) holds p, B(ee, 1) the next iterate; they alternate
  auto buf = [&](int ee, int which) { return smp + ee * G::EB + which * G::ES; };
  double coeff = dt;
  int cur = 0;  // buffer holding the current iterate p
#pragma unroll 1
  for (int o = 1; o < N; ++o) {
    const double* P = buf(el < G::EPB ? el : 0, cur);
    double* T = buf(el < G::EPB ? el : 0, cur ^ 1);
#pragma unroll 1
    for (int d = 0; d < 3; ++d) {
      if (active) {
        const PassSlot ps = kPass[d][slot];
        int start, stride;  // line start and stride along direction d
        if (d == 0) {
          start = la * G::PL + lb * G::RS;  // x-line (k3, k2)
          stride = 1;
        } else if (d == 1) {
          start = la * G::PL + lb;  // y-line (k3, k1)
          stride = G::RS;
        } else {
          start = la * G::RS + lb;  // z-line (k2, k1)
          stride = G::PL;
        }
        double p[N], out[N];
        const double* src = P + ps.src * G::VS + start;
#pragma unroll
        for (int l = 0; l < N; ++l) p[l] = src[l * stride];
        eo_apply<N>(p, out);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          if (k < ps.nt) {
            const double c = pick4(c4, ps.coef[k]);
            double* dst = T + ps.tgt[k] * G::VS + start;
            // pass x writes every target but syz; pass y writes syz (its first touch)
            if (d == 0 || (d == 1 && ps.tgt[k] == 5)) {
#pragma unroll
              for (int l = 0; l < N; ++l) dst[l * stride] = c * out[l];
            } else {
#pragma unroll
              for (int l = 0; l < N; ++l) dst[l * stride] = fma(c, out[l], dst[l * stride]);
            }
          }
        }
      }
      __syncthreads();
    }
    // T = sum_d D_d F_d(p) is the next iterate: qavg += c_o T  (stp_splitck.cpp:64-69)
    coeff *= dt / (o + 1);
    cur ^= 1;
#pragma unroll
    for (int j = 0; j < G::QPT; ++j) {
      const int i = tid + j * G::THREADS;
      if (i < G::EPB * G::OUTV) {
        const int ee = i / G::OUTV;
        int r = i - ee * G::OUTV;
        const int k1 = r % N;
        r /= N;
        const int s = r % NVE;
        r /= NVE;
        qa[j] = fma(coeff, buf(ee, cur)[s * G::VS + (r / N) * G::PL + (r % N) * G::RS + k1], qa[j]);
      }
    }
    // no barrier needed: the next pass x reads buf(cur) (read-only) and writes buf(cur ^ 1),
    // whose last readers were this step's passes, all behind the pass-z barrier
  }
  __syncthreads();  // every qavg read of the last iterate is done

  // ---- epilogue --------------------------------------------------------------------------
  // qavg: registers -> global (flat, coalesced) and -> buffer 0 for favg / faces
#pragma unroll
  for (int j = 0; j < G::QPT; ++j) {
    const int i = tid + j * G::THREADS;
    if (i < G::EPB * G::OUTV) {
      const int ee = i / G::OUTV;
      int r = i - ee * G::OUTV;
      if (e0 + ee < a.n_elem) __stcs(a.qavg + (e0 + ee) * (long long)G::OUTV + r, qa[j]);
      const int k1 = r % N;
      r /= N;
      const int s = r % NVE;
      r /= NVE;
      buf(ee, 0)[s * G::VS + (r / N) * G::PL + (r % N) * G::RS + k1] = qa[j];
    }
  }
  __syncthreads();
  // favg_d[s] = coef(s,d) qavg[in(s,d)]  (proj/src/stp_splitck.cpp:72-78), flat over
  // [e][d][k3][k2][s][k1]; the element's material is recomputed per entry's element
  if (a.favg) {
    for (int i = tid; i < G::EPB * 3 * G::OUTV; i += G::THREADS) {
      const int ee = i / (3 * G::OUTV);
      if (e0 + ee >= a.n_elem) continue;
      int r = i - ee * 3 * G::OUTV;
      const int d = r / G::OUTV;
      r -= d * G::OUTV;
      const int k1 = r % N;
      int rr = r / N;
      const int s = rr % NVE;
      rr /= NVE;
      const int ci = kCoefE[s][d];
      double v = 0.0;
      if (ci != 4) {
        const double* pr = a.par + 3 * (e0 + ee);
        double cc;
        if (kp.par_kind == ADERSTP_PAR_RHO_CP_CS) {
          const double mu = __dmul_rn(__dmul_rn(pr[0], pr[2]), pr[2]);
          const double lam = __dsub_rn(__dmul_rn(__dmul_rn(pr[0], pr[1]), pr[1]), __dmul_rn(2.0, mu));
          cc = ci == 0 ? lam + 2.0 * mu : ci == 1 ? lam : ci == 2 ? mu : 1.0 / pr[0];
        } else {
          cc = ci == 0 ? pr[0] + 2.0 * pr[1] : ci == 1 ? pr[0] : ci == 2 ? pr[1] : 1.0 / pr[2];
        }
        v = cc * buf(ee, 0)[kInE[s][d] * G::VS + (rr / N) * G::PL + (rr % N) * G::RS + k1];
      }
      __stcs(a.favg + (e0 + ee) * 3LL * G::OUTV + d * G::OUTV + r, v);
    }
  }
  if (a.face_q || a.face_f) {
    // face_q: task (normal d, a, b, s) contracts one line with phi(0) and phi(1) into the
    // staging buffer 1 laid out as the reference's [f][a][b][s]
    constexpr int FV = N * N * NVE;  // one face array
    for (int i = tid; i < G::EPB * 3 * FV; i += G::THREADS) {
      const int ee = i / (3 * FV);
      int r = i - ee * 3 * FV;
      const int d = r / FV;
      r -= d * FV;
      const int s = r % NVE;
      const int ab = r / NVE;
      const int aa = ab / N, bb = ab - aa * N;
      int start, stride;
      if (d == 0) {
        start = aa * G::PL + bb * G::RS;
        stride = 1;
      } else if (d == 1) {
        start = aa * G::PL + bb;
        stride = G::RS;
      } else {
        start = aa * G::RS + bb;
        stride = G::PL;
      }
      const double* ln = buf(ee, 0) + s * G::VS + start;
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double x = ln[j * stride];
        v0 = fma(kp.phi[0][j], x, v0);
        v1 = fma(kp.phi[1][j], x, v1);
      }
      double* fq = buf(ee, 1);
      fq[(2 * d) * FV + ab * NVE + s] = v0;
      fq[(2 * d + 1) * FV + ab * NVE + s] = v1;
    }
    __syncthreads();
    for (int i = tid; i < G::EPB * 6 * FV; i += G::THREADS) {
      const int ee = i / (6 * FV);
      if (e0 + ee >= a.n_elem) continue;
      const int r = i - ee * 6 * FV;
      const double* fq = buf(ee, 1);
      if (a.face_q) __stcs(a.face_q + (e0 + ee) * 6LL * FV + r, fq[r]);
      if (a.face_f) {
        const int f = r / FV, d = f >> 1;
        const int s = r % NVE;
        const int ci = kCoefE[s][d];
        double v = 0.0;
        if (ci != 4) {
          const double* pr = a.par + 3 * (e0 + ee);
          double cc;
          if (kp.par_kind == ADERSTP_PAR_RHO_CP_CS) {
            const double mu = __dmul_rn(__dmul_rn(pr[0], pr[2]), pr[2]);
            const double lam = __dsub_rn(__dmul_rn(__dmul_rn(pr[0], pr[1]), pr[1]), __dmul_rn(2.0, mu));
            cc = ci == 0 ? lam + 2.0 * mu : ci == 1 ? lam : ci == 2 ? mu : 1.0 / pr[0];
          } else {
            cc = ci == 0 ? pr[0] + 2.0 * pr[1] : ci == 1 ? pr[0] : ci == 2 ? pr[1] : 1.0 / pr[2];
          }
          v = cc * fq[r - s + kInE[s][d]];
        }
        __stcs(a.face_f + (e0 + ee) * 6LL * FV + r, v);
      }
    }
  }
  if (kp.check && flags) atomicOr(status, flags);
}

template <int N>
cudaError_t launch_pass_n(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  using G = Geo<N>;
  PassParams<N> kp;
  for (int j = 0; j < N; ++j) {
    kp.phi[0][j] = p.basis.face_left[j];
    kp.phi[1][j] = p.basis.face_right[j];
  }
  kp.check = p.check;
  kp.par_kind = p.par_kind;
  kp.q_stride = p.q_stride;
  cudaError_t err = cudaFuncSetAttribute(stp_pass_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  if (err == cudaSuccess)
    err = cudaFuncSetAttribute(stp_pass_kernel<N>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  const long long blocks = (a.n_elem + G::EPB - 1) / G::EPB;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  stp_pass_kernel<N><<<(unsigned)blocks, G::THREADS, G::SMEM, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}

}  // namespace

bool pass_applicable(const LaunchPlan& p) {
  return p.n >= 2 && p.n <= 10 && p.kind == ADERSTP_PDE_ELASTIC && p.src_comp < 0 &&
         p.layout == ADERSTP_LAYOUT_AOSOA && p.out_stride == 9 && p.q_stride >= 9 && p.q_stride <= 64;
}

// Even/odd split of D (see the file comment), per order, into aderstp_kEO[n*64 ...].
cudaError_t init_pass(const LaunchPlan& p) {
  const int n = p.n, h = n / 2;
  double buf[64] = {0};
  const double* D = p.basis.d;
  for (int k = 0; k < h; ++k) {
    for (int l = 0; l < h; ++l) {
      buf[k * (h + 1) + l] = 0.5 * (D[k * n + l] + D[k * n + (n - 1 - l)]);          // A
      buf[h * (h + 1) + k * h + l] = 0.5 * (D[k * n + l] - D[k * n + (n - 1 - l)]);  // B
    }
    if (n % 2) buf[k * (h + 1) + h] = D[k * n + h];  // middle column acts on e[h] = p[h]
  }
  if (n % 2) {
    for (int l = 0; l < h; ++l) buf[h * (h + 1) + h * h + l] = 0.5 * (D[h * n + l] - D[h * n + (n - 1 - l)]);
    buf[h * (h + 1) + h * h + h] = D[h * n + h];
  }
  return cudaMemcpyToSymbol(aderstp_kEO, buf, sizeof(buf), sizeof(double) * 64 * n);
}

cudaError_t launch_pass(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  switch (p.n) {
    case 2: return launch_pass_n<2>(p, a, stream);
    case 3: return launch_pass_n<3>(p, a, stream);
    case 4: return launch_pass_n<4>(p, a, stream);
    case 5: return launch_pass_n<5>(p, a, stream);
    case 6: return launch_pass_n<6>(p, a, stream);
    case 7: return launch_pass_n<7>(p, a, stream);
    case 8: return launch_pass_n<8>(p, a, stream);
    case 9: return launch_pass_n<9>(p, a, stream);
    case 10: return launch_pass_n<10>(p, a, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace aderstp
