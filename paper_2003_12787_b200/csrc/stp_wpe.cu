// Elastic STP for nDof 4..6: one WARP per element, no CTA barrier.  The default for large nDof 4
// and nDof 5 batches (kWpeMinElems4 / 5: 104 vs 78 M and 40.9 vs 37.7 M elem/s for stp_dmmap); at
// nDof 6 opt-in (ADERSTP_WPE=1: 21.4 vs 30.4 M).
//
// The padded-DMMA kernel (stp_dmma.cu) carries (8/N)^2 of the useful fragment traffic and fp64
// work at nDof <= 6 and spends its largest stall on CTA barriers.  Here every warp owns an element
// from load to store (persistent warps, 7 / 8 / 12 per SM at nDof 6 / 5 / 4, each with 2 x 9
// fields of shared memory), and a CK step r <- c_o q + L r (Horner form, see stp_dmma8.cu; proj/src/stp_splitck.cpp:46-70) is two
// warp-synchronous phases of TILE tasks: a lane owns an N x N tile (a, b) of one target field at a
// fixed third index, keeps its N^2 accumulators in registers and contracts
//   term A: acc[ia][ib] += D[ia][l] srcA(l, ib)      (derivative along a)
//   term B: acc[ia][ib] += D[ib][l] srcB(ia, l)      (derivative along b)
// so every value loaded from shared memory feeds N FMAs.  The tile orientation is chosen per
// target so that both in-tile directions carry a flux term (proj/src/pde.cpp:180-218):
//   phase A  sxy' (x,y), sxz' (x,z), syz' (y,z) from the old velocities, and the four z
//            derivatives that have no in-tile home (d_z sxz, d_z syz, d_z szz, d_z w), two per
//            lane, stored raw in the slots of the fields they complete (u', v', w', szz');
//   phase B  u', v', w' (x,y tiles: two in-tile terms + the stored z term) and the normal
//            stresses (one lane per k3 plane: a = d_x u, b = d_y v in-tile, c = d_z w stored;
//            s_ii' = lambda (a+b+c) + 2 mu {a,b,c}_i).
// Tile strides are per-lane run-time values, so all orientations run the same instruction stream.
// The Horner term c_o q comes from tensor memory (thread-private columns, filled once per
// element), the iterate ping-pongs between the warp's two buffers.  Epilogue: face extrapolations
// as line tasks into the dead buffer, leaving as TMA bulk stores (face_f formed in place once the
// face_q copy has been read); qavg / favg are written in output order (coalesced 16-byte stores,
// 8-byte at the odd nDof 5).  No CTA-wide barrier after the TMEM allocation.
#include <cstdint>
#include <type_traits>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"
#include "tmem.cuh"

namespace aderstp {

namespace {

// A/B knobs (make variant EXTRA=-D...): warps per SM at nDof 4 / 5, branching stores at nDof 5
#ifndef WPE_WPC4
#define WPE_WPC4 12
#endif
#ifndef WPE_WPC5
#define WPE_WPC5 8
#endif
#ifndef WPE_PRED5
#define WPE_PRED5 0
#endif
constexpr int NVW = 9;
enum { MODE_IDLE = 0, MODE_SUM = 1, MODE_NORMAL = 2, MODE_PAIR = 3 };

template <int N>
struct GeoW {
  static constexpr int N2 = N * N, N3 = N * N * N;
  // warps (= elements in flight) per CTA, one CTA per SM.  nDof 6: as many as the shared memory
  // holds.  nDof 4 / 5: a multiple of the 4 SM sub-partitions whose register budget leaves the
  // tile accumulators unspilled -- measured nDof 4: 8 / 12 / 16 warps 95.6 / 104.1 / 99.4 M elem/s;
  // nDof 5: 4 / 8 / 10 warps 33.1 / 40.7 / 36.6 M (10 warps = 3 + 3 + 2 + 2 per sub-partition at 168
  // registers with spills)
  static constexpr int WPC = N == 6 ? 7 : N == 5 ? WPE_WPC5 : WPE_WPC4;
  // compute layout [field][k3][k2][k1]: strides in doubles (bank model: tools/wpe_bank_model.py)
  static constexpr int S2 = N == 6 ? 6 : 5;
  static constexpr int S3 = N == 6 ? 37 : N == 5 ? 25 : 21;
  static constexpr int FS = N == 6 ? 223 : N == 5 ? 125 : 94;
  // idle lanes / absent outputs: skipped by one branch per row and output set (N = 4: whole
  // half-warps fall idle and cost no wavefront, +14 %) or sent to the dummy slot with plain stores
  // (N = 5, 6: the branching form measured -5 %, -6 %; an inline-asm predicated store -6 %, -10 %)
  static constexpr bool PRED = N == 4 || (N == 5 && WPE_PRED5);
  static constexpr int FACE = N2 * NVW;                       // one face array
  static constexpr int BUF = ((NVW * FS > 6 * FACE ? NVW * FS : 6 * FACE) + 2) & ~1;  // doubles, even, >= fields + 1
  static constexpr int DUMMY = NVW * FS;                      // a slot no field uses (write-only sink)
  static constexpr int WARP_DOUBLES = 2 * BUF;
  static constexpr int QC = 2 * N2;                           // TMEM columns of one q tile
  static constexpr int TCW = 3 * QC;                          // TMEM columns per warp
  static constexpr int SMEM = WPC * WARP_DOUBLES * 8;
};

struct TaskW {
  int srcA, saA, sbA;  // term A: source tile origin and strides (doubles) along a, b
  int srcB, saB, sbB;  // term B
  int dst1, dst2, dst3, part;  // idle lanes and unused outputs point at the buffer's dummy slot
  int s2a, s2b;        // strides of dst2 / dst3 (0 where they are the dummy slot)
  int mode, coef;
};

struct ParamsW {
  double d[36];        // D[k][l], row-major N x N
  double phi[2][6];    // phi(0), phi(1)
  double cf[8];        // cf[o] = dt^(o+1)/(o+1)!
  int check, par_kind, q_stride, prefetch;
};

__constant__ TaskW kTaskW[3][2][32];  // [N - 4][phase][lane]

template <int N>
__device__ __forceinline__ void tm_ld_row(uint32_t ta, uint32_t* r) {
  tm_ld8(ta, r);
  if constexpr (N == 6) tm_ld4(ta + 8, r + 8);
  if constexpr (N == 5) tm_ld2(ta + 8, r + 8);
}
template <int N>
__device__ __forceinline__ void tm_st_row(uint32_t ta, const uint32_t* r) {
  tm_st8(ta, r);
  if constexpr (N == 6) tm_st4(ta + 8, r + 8);
  if constexpr (N == 5) tm_st2(ta + 8, r + 8);
}

// e_in(s, d) / e_coef(s, d) of the 9 output quantities packed 4 bits each
constexpr unsigned long long pack_flux_w(int d, bool coef) {
  unsigned long long v = 0;
  for (int s = 0; s < NVW; ++s) v |= (unsigned long long)(coef ? e_coef(s, d) : e_in(s, d)) << (4 * s);
  return v;
}

// One phase of a CK step for the calling lane's task: R (source iterate), W (destination).
// Every lane runs every load and FMA; idle lanes and unused outputs have zero strides and the
// buffer's dummy slot as destination (their stores are skipped in the PRED instance).  out1 = co q1 + c1 (a + b + p) + c2 a; the
// normal-stress lanes (phase B) also write out2 = co q2 + c1 S + c2 b and out3 = co q3 + c1 S +
// c2 p; the raw-derivative lanes (phase A: co = c1 = 0, c2 = 1) write a to dst1 and b to dst2.
template <int N, bool PHASEB>
__device__ __forceinline__ void run_phase(const ParamsW& kp, TaskW t, const double* __restrict__ R,
                                          double* __restrict__ W, uint32_t tq, double co, double c1, double c2) {
  using G = GeoW<N>;
  // the strides are opaque per call: ptxas would otherwise hoist all 2 N^2 tile offsets out of the
  // CK loop and spill them
  asm volatile("" : "+r"(t.saA), "+r"(t.sbA), "+r"(t.saB), "+r"(t.sbB));
  // idle lanes and absent outputs are predicated off (no wavefront for a half-warp without a
  // live lane): the second / third outputs sit in one half-warp (build_tasks)
  const bool act = !G::PRED || t.mode != MODE_IDLE;
  const bool has2 = !G::PRED || (PHASEB ? t.mode == MODE_NORMAL : t.mode == MODE_PAIR);
  double accA[N][N], accB[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) accA[i][j] = accB[i][j] = 0.0;
  {  // term A: derivative along a, one line (fixed ib) at a time
    const double* p = R + t.srcA;
#pragma unroll
    for (int ib = 0; ib < N; ++ib) {
      double v[N];
#pragma unroll
      for (int l = 0; l < N; ++l) v[l] = act ? p[l * t.saA] : 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l)
#pragma unroll
        for (int ia = 0; ia < N; ++ia) accA[ia][ib] = fma(kp.d[ia * N + l], v[l], accA[ia][ib]);
      p += t.sbA;
    }
  }
  {  // term B: derivative along b, one line (fixed ia) at a time
    const double* p = R + t.srcB;
#pragma unroll
    for (int ia = 0; ia < N; ++ia) {
      double v[N];
#pragma unroll
      for (int l = 0; l < N; ++l) v[l] = act ? p[l * t.sbB] : 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l)
#pragma unroll
        for (int ib = 0; ib < N; ++ib) accB[ia][ib] = fma(kp.d[ib * N + l], v[l], accB[ia][ib]);
      p += t.saB;
    }
  }
  double* w1 = W + t.dst1;
  double* w2 = W + t.dst2;
  double* w3 = W + t.dst3;
  const double* wp = W + t.part;
#pragma unroll
  for (int ia = 0; ia < N; ++ia) {
    uint32_t r1[2 * N], r2[2 * N], r3[2 * N];
    tm_ld_row<N>(tq + (PHASEB ? G::QC : 0) + 2 * N * ia, r1);
    if (PHASEB) {
      tm_ld_row<N>(tq + 2 * N * ia, r2);
      tm_ld_row<N>(tq + 2 * G::QC + 2 * N * ia, r3);
    }
    tm_wait_ld();
    double o1[N], o2[N], o3[N];
#pragma unroll
    for (int ib = 0; ib < N; ++ib) {
      const double a = accA[ia][ib], b = accB[ia][ib];
      if (PHASEB) {
        const double p = act ? wp[ib * t.sbA] : 0.0;
        const double S = a + b + p, cS = c1 * S;
        o1[ib] = fma(co, tm_double(r1, ib), fma(c2, a, cS));
        o2[ib] = fma(co, tm_double(r2, ib), fma(c2, b, cS));
        o3[ib] = fma(co, tm_double(r3, ib), fma(c2, p, cS));
      } else {
        o1[ib] = fma(co, tm_double(r1, ib), fma(c2, a, c1 * (a + b)));
        o2[ib] = b;
      }
    }
    // PRED: one branch per row and output set (a branch per store made ptxas emit BSSY / BSYNC
    // around each; an inline-asm predicated store serialised the schedule): lanes without the
    // output skip its stores, so a half-warp without a live lane costs no wavefront
    if (act) {
#pragma unroll
      for (int ib = 0; ib < N; ++ib) w1[ib * t.sbA] = o1[ib];
    }
    if (has2) {
#pragma unroll
      for (int ib = 0; ib < N; ++ib) {
        w2[ib * t.s2b] = o2[ib];
        if (PHASEB) w3[ib * t.s2b] = o3[ib];
      }
    }
    w1 += t.saA;
    w2 += t.s2a;
    w3 += t.s2a;
    wp += t.saA;
  }
}

// copy the N x N tile at off (strides sa, sb) of the q buffer into TMEM columns [col, col + QC)
template <int N>
__device__ __forceinline__ unsigned fill_tile(const double* q, int off, int sa, int sb, uint32_t ta, bool check) {
  unsigned bad = 0;
#pragma unroll
  for (int ia = 0; ia < N; ++ia) {
    uint32_t r[2 * N];
#pragma unroll
    for (int ib = 0; ib < N; ++ib) {
      const double v = q[off + ia * sa + ib * sb];
      if (check && !isfinite(v)) bad = 1u;
      tm_split(v, r, ib);
    }
    tm_st_row<N>(ta + 2 * N * ia, r);
  }
  return bad;
}

template <int N>
__global__ void __launch_bounds__(GeoW<N>::WPC * 32, 1) stp_wpe_kernel(ParamsW kp, BatchArgs a, unsigned int* status) {
  using G = GeoW<N>;
  constexpr int N2 = G::N2, N3 = G::N3, S2 = G::S2, S3 = G::S3, FS = G::FS, FACE = G::FACE, WPC = G::WPC;
  extern __shared__ __align__(16) double smw[];
  __shared__ uint32_t tmem_base_s;
  __shared__ TaskW task_s[2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 64) task_s[threadIdx.x >> 5][lane] = kTaskW[N - 4][threadIdx.x >> 5][lane];
  if (warp == 0) tm_alloc<512>(&tmem_base_s);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tq = tmem_base_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * G::TCW);
  double* B0 = smw + warp * G::WARP_DOUBLES;
  double* B1 = B0 + G::BUF;
  unsigned int flags = 0;
  const int qs = kp.q_stride;
  const long long estride = (long long)gridDim.x * WPC;

  // element = CTA + grid * (warp + WPC * round): a small batch spreads over the SMs first
  for (long long e = blockIdx.x + (long long)gridDim.x * warp; e < a.n_elem; e += estride) {
    // ---- material -----------------------------------------------------------------------------
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
    // ---- q: HBM -> registers -> B0 in the compute layout -----------------------------------------
    const double* qe = a.q + e * (long long)(N3 * qs);
    if (kp.prefetch && lane == 0 && e + estride < a.n_elem) {
      const unsigned long long pa = reinterpret_cast<unsigned long long>(a.q + (e + estride) * (long long)(N3 * qs));
      const unsigned long long p0 = pa & ~15ull, p1 = (pa + 8ull * N3 * qs + 15ull) & ~15ull;  // 16-byte bounds
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p0), "r"((unsigned)(p1 - p0)) : "memory");
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // B0 was the face staging
    __syncwarp();
    if constexpr (N % 2 != 0) {  // rows of N doubles are 8-byte aligned only: scalar loads
      if (qs == NVW) {
        constexpr int ND = N3 * NVW, IT = (ND + 31) / 32;
        double v[IT];
#pragma unroll
        for (int i = 0; i < IT; ++i) {
          const int p = lane + 32 * i;
          v[i] = p < ND ? __ldcs(qe + p) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < IT; ++i) {
          const int p = lane + 32 * i;
          if (p < ND) {
            const int k1 = p % N, r1 = p / N, s = r1 % NVW, k32 = r1 / NVW;
            B0[s * FS + (k32 / N) * S3 + (k32 % N) * S2 + k1] = v[i];
          }
        }
      } else {
        const int rowd = qs * N;
        for (int p = lane; p < N2 * rowd; p += 32) {
          const int k32 = p / rowd, rem = p - k32 * rowd, s = rem / N, k1 = rem - s * N;
          if (s < NVW) B0[s * FS + (k32 / N) * S3 + (k32 % N) * S2 + k1] = __ldcs(qe + p);
        }
      }
    } else
    if (qs == NVW) {
      constexpr int NP = N3 * NVW / 2, IT = (NP + 31) / 32;
      double2 v[IT];
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        const int p = lane + 32 * i;
        v[i] = p < NP ? __ldcs(reinterpret_cast<const double2*>(qe) + p) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int i = 0; i < IT; ++i) {
        const int p = lane + 32 * i;
        if (p < NP) {
          const int kp1 = p % (N / 2), r1 = p / (N / 2), s = r1 % NVW, k32 = r1 / NVW;
          double* dst = B0 + s * FS + (k32 / N) * S3 + (k32 % N) * S2 + 2 * kp1;
          dst[0] = v[i].x;
          dst[1] = v[i].y;
        }
      }
    } else {
      const int rowp = qs * (N / 2);  // pairs per (k3, k2) row group
      for (int p = lane; p < N2 * rowp; p += 32) {
        const int k32 = p / rowp, rem = p - k32 * rowp, s = rem / (N / 2), kp1 = rem - s * (N / 2);
        if (s < NVW) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(qe) + p);
          double* dst = B0 + s * FS + (k32 / N) * S3 + (k32 % N) * S2 + 2 * kp1;
          dst[0] = v.x;
          dst[1] = v.y;
        }
      }
    }
    __syncwarp();
    // ---- q tiles -> tensor memory (the Horner term of every task of this lane) ----------------
    {
      unsigned bad = 0;
      const TaskW tA = task_s[0][lane], tB = task_s[1][lane];
      const bool nB = tB.mode == MODE_NORMAL;
      // lanes without a tile in a region copy field 0 (any finite-or-not value: never used, never checked)
      const bool r0 = nB || tA.mode == MODE_SUM, r1 = tB.mode != MODE_IDLE;
      bad |= fill_tile<N>(B0, nB ? tB.dst2 : r0 ? tA.dst1 : 0, nB ? tB.saA : tA.saA, nB ? tB.sbA : tA.sbA, tq,
                          kp.check && r0);
      bad |= fill_tile<N>(B0, r1 ? tB.dst1 : 0, tB.saA, tB.sbA, tq + G::QC, kp.check && r1);
      bad |= fill_tile<N>(B0, nB ? tB.dst3 : 0, tB.saA, tB.sbA, tq + 2 * G::QC, kp.check && nB);
      tm_wait_st();
      if (bad) flags |= 1u;
    }
    // ---- CK series in Horner form: r <- c_o q + L r, o = N-2 .. 0; the first iterate is
    // c_(N-1) q, folded into the coefficients of the first step --------------------------------
#pragma unroll 1
    for (int it = 0; it < N - 1; ++it) {
      const double co = kp.cf[N - 2 - it];
      const double sc = it == 0 ? kp.cf[N - 1] : 1.0;
      const double* R = (it & 1) ? B1 : B0;
      double* W = (it & 1) ? B0 : B1;
      {
        const TaskW tA = task_s[0][lane];
        const double cc = tA.coef == 0 ? c4[0] : tA.coef == 1 ? c4[1] : tA.coef == 2 ? c4[2] : c4[3];
        const bool pair = tA.mode == MODE_PAIR;
        run_phase<N, false>(kp, tA, R, W, tq, pair ? 0.0 : co, pair ? 0.0 : cc * sc, pair ? 1.0 : 0.0);
      }
      __syncwarp();
      {
        const TaskW tB = task_s[1][lane];
        const bool nrm = tB.mode == MODE_NORMAL;
        const double cc = tB.coef == 0 ? c4[0] : tB.coef == 1 ? c4[1] : tB.coef == 2 ? c4[2] : c4[3];
        run_phase<N, true>(kp, tB, R, W, tq, co, nrm ? c4[1] * sc : cc * sc, nrm ? 2.0 * c4[2] * sc : 0.0);
      }
      __syncwarp();
    }
    const double* Y = ((N - 1) & 1) ? B1 : B0;  // qavg: the last iterate (B1: N - 1 is odd)
    double* X = ((N - 1) & 1) ? B0 : B1;        // free: the face staging buffer
    const bool faces = a.face_q || a.face_f;
    // ---- faces: line tasks (in-face node, quantity) per direction -> X [6][N][N][9]; the line
    // strides are compile-time constants per direction (immediate offsets) -----------------------
    if (faces) {
      constexpr int TD = N2 * NVW;
      auto face_dir = [&](auto dd) {
        constexpr int D = decltype(dd)::value;
        constexpr int SA = D == 2 ? S2 : S3, SB = D == 0 ? S2 : 1, SL = D == 0 ? 1 : D == 1 ? S2 : S3;
#pragma unroll 2
        for (int i = lane; i < TD; i += 32) {
          const int ab = i / NVW, s = i - ab * NVW, a0 = ab / N, b0 = ab - a0 * N;
          const double* line = Y + s * FS + a0 * SA + b0 * SB;
          double f0 = 0.0, f1 = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            const double v = line[k * SL];
            f0 = fma(kp.phi[0][k], v, f0);
            f1 = fma(kp.phi[1][k], v, f1);
          }
          X[(2 * D) * FACE + i] = f0;
          X[(2 * D + 1) * FACE + i] = f1;
        }
      };
      face_dir(std::integral_constant<int, 0>{});
      face_dir(std::integral_constant<int, 1>{});
      face_dir(std::integral_constant<int, 2>{});
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0 && a.face_q) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                         a.face_q + e * (long long)(6 * FACE)),
                     "r"((unsigned)__cvta_generic_to_shared(X)), "r"((unsigned)(6 * FACE * 8))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    }
    // ---- qavg / favg in output order: lane = (quantity s, k1 pair) of a (k3, k2) row group, so a
    // warp store covers the row group's 9 N contiguous doubles; per-lane flux sources and
    // coefficients are loop constants and every shared / global offset is an immediate ----------
    if constexpr (N % 2 != 0) {
      // odd N: rows of N doubles are 8-byte aligned only; lane = (quantity s, k1) of a row group in
      // passes of 32 lanes, 8-byte stores of consecutive doubles
      constexpr int RD = NVW * N;  // doubles per row group
      constexpr unsigned long long IN[3] = {pack_flux_w(0, false), pack_flux_w(1, false), pack_flux_w(2, false)};
      constexpr unsigned long long CO[3] = {pack_flux_w(0, true), pack_flux_w(1, true), pack_flux_w(2, true)};
      double* qo = a.qavg + e * (long long)(N3 * NVW);
      double* fo = a.favg ? a.favg + e * (long long)(3 * N3 * NVW) : nullptr;
#pragma unroll
      for (int base = 0; base < RD; base += 32) {
        const int idx = base + lane;
        if (idx < RD) {
          const int s = idx / N, k1 = idx - s * N;
          const double* sq = Y + s * FS + k1;
          const double* sf[3];
          double cf3[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const int si = (int)((IN[d] >> (4 * s)) & 15), ci = (int)((CO[d] >> (4 * s)) & 15);
            sf[d] = Y + si * FS + k1;
            cf3[d] = ci == 0 ? c4[0] : ci == 1 ? c4[1] : ci == 2 ? c4[2] : ci == 3 ? c4[3] : 0.0;
          }
#pragma unroll
          for (int k3 = 0; k3 < N; ++k3)
#pragma unroll
            for (int k2 = 0; k2 < N; ++k2) {
              const int node = k3 * S3 + k2 * S2, o = (k3 * N + k2) * RD + idx;
              __stcs(qo + o, sq[node]);
              if (fo) {
#pragma unroll
                for (int d = 0; d < 3; ++d) __stcs(fo + d * (N3 * NVW) + o, cf3[d] * sf[d][node]);
              }
            }
        }
      }
    } else
    {
      constexpr int PR = NVW * N / 2;  // 16-byte pairs per row group
      constexpr unsigned long long IN[3] = {pack_flux_w(0, false), pack_flux_w(1, false), pack_flux_w(2, false)};
      constexpr unsigned long long CO[3] = {pack_flux_w(0, true), pack_flux_w(1, true), pack_flux_w(2, true)};
      if (lane < PR) {
        const int s = lane / (N / 2), kp1 = lane - s * (N / 2);
        const double* sq = Y + s * FS + 2 * kp1;
        const double* sf[3];
        double cf3[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const int si = (int)((IN[d] >> (4 * s)) & 15), ci = (int)((CO[d] >> (4 * s)) & 15);
          sf[d] = Y + si * FS + 2 * kp1;
          cf3[d] = ci == 0 ? c4[0] : ci == 1 ? c4[1] : ci == 2 ? c4[2] : ci == 3 ? c4[3] : 0.0;
        }
        double2* qo = reinterpret_cast<double2*>(a.qavg + e * (long long)(N3 * NVW)) + lane;
        double2* fo = a.favg ? reinterpret_cast<double2*>(a.favg + e * (long long)(3 * N3 * NVW)) + lane : nullptr;
#pragma unroll
        for (int k3 = 0; k3 < N; ++k3)
#pragma unroll
          for (int k2 = 0; k2 < N; ++k2) {
            const int node = k3 * S3 + k2 * S2, rg = k3 * N + k2;
            __stcs(qo + rg * PR, make_double2(sq[node], sq[node + 1]));
            if (fo) {
#pragma unroll
              for (int d = 0; d < 3; ++d)
                __stcs(fo + d * (N3 * NVW / 2) + rg * PR,
                       make_double2(cf3[d] * sf[d][node], cf3[d] * sf[d][node + 1]));
            }
          }
      }
    }
    // ---- face_f = F_d(face_q) in place, once the face_q copy has read the staging buffer ---------
    if (faces) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      __syncwarp();
      if (a.face_f) {
#pragma unroll 1
        for (int i = lane; i < 6 * N2; i += 32) {
          const int d = i / (2 * N2);
          double* node = X + i * NVW;
          double v[NVW];
#pragma unroll
          for (int s = 0; s < NVW; ++s) v[s] = node[s];
          auto emit = [&](auto dd) {
            constexpr int D = decltype(dd)::value;
#pragma unroll
            for (int so = 0; so < NVW; ++so) {
              const int ci = e_coef(so, D);
              node[so] = ci == 4 ? 0.0 : c4[ci & 3] * v[e_in(so, D)];
            }
          };
          if (d == 0) emit(std::integral_constant<int, 0>{});
          else if (d == 1) emit(std::integral_constant<int, 1>{});
          else emit(std::integral_constant<int, 2>{});
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                           a.face_f + e * (long long)(6 * FACE)),
                       "r"((unsigned)__cvta_generic_to_shared(X)), "r"((unsigned)(6 * FACE * 8))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
  if (kp.check && flags) atomicOr(status, flags);
  tm_fence_before();
  __syncthreads();
  if (warp == 0) {
    tm_fence_after();
    tm_dealloc<512>(tmem_base_s);
  }
}

// ---- host: the lane -> task tables ------------------------------------------------------------------
template <int N>
void build_tasks(TaskW (&tab)[2][32]) {
  using G = GeoW<N>;
  constexpr int FS = G::FS;
  const int st[3] = {1, G::S2, G::S3};  // strides of x, y, z
  enum { SXX, SYY, SZZ, SXY, SXZ, SYZ, U, V, Wq };
  for (int ph = 0; ph < 2; ++ph)
    for (int l = 0; l < 32; ++l) {
      TaskW t{};  // idle: zero strides, every access at offset 0 / the dummy slot
      t.mode = MODE_IDLE;
      t.dst1 = t.dst2 = t.dst3 = t.part = G::DUMMY;
      tab[ph][l] = t;
    }
  // tile (a, b) at fixed third direction c = k; sources fA (derivative along a), fB (along b)
  auto tile = [&](int da, int db, int dc, int k, int fA, int fB, int dst, int coef, int part) {
    TaskW t{};
    t.saA = t.saB = st[da];
    t.sbA = t.sbB = st[db];
    t.srcA = fA * FS + k * st[dc];
    t.srcB = fB * FS + k * st[dc];
    t.dst1 = dst * FS + k * st[dc];
    t.dst2 = t.dst3 = G::DUMMY;
    t.s2a = t.s2b = 0;
    t.part = part < 0 ? G::DUMMY : part * FS + k * st[dc];
    t.mode = MODE_SUM;
    t.coef = coef;
    return t;
  };
  int lane = 0;
  // phase A: shear stresses (coef 2 = mu)
  for (int k = 0; k < N; ++k) tab[0][lane++] = tile(0, 1, 2, k, V, U, SXY, 2, -1);
  for (int k = 0; k < N; ++k) tab[0][lane++] = tile(0, 2, 1, k, Wq, U, SXZ, 2, -1);
  for (int k = 0; k < N; ++k) tab[0][lane++] = tile(1, 2, 0, k, Wq, V, SYZ, 2, -1);
  // phase A: raw z derivatives, two per lane: d_z sxz -> u', d_z syz -> v' | d_z szz -> w', d_z w -> szz'
  const int psrc[4] = {SXZ, SYZ, SZZ, Wq}, pdst[4] = {U, V, Wq, SZZ};
  if (lane < 16 && 16 + 2 * N <= 32) lane = 16;  // the raw-derivative lanes share one half-warp
  for (int i = 0; i < 2 * N; ++i) {
    const int u1 = i / N, u2 = 2 + i / N, k = i % N;  // tiles at fixed k2 = k
    TaskW t{};
    t.mode = MODE_PAIR;
    t.part = t.dst3 = G::DUMMY;
    t.coef = 0;
    t.saA = st[2];  // term A: a = z, b = x
    t.sbA = st[0];
    t.srcA = psrc[u1] * FS + k * st[1];
    t.dst1 = pdst[u1] * FS + k * st[1];
    t.saB = st[0];  // term B: a = x, b = z
    t.sbB = st[2];
    t.srcB = psrc[u2] * FS + k * st[1];
    t.dst2 = pdst[u2] * FS + k * st[1];
    t.s2a = t.saB;
    t.s2b = t.sbB;
    tab[0][lane++] = t;
  }
  // phase B: velocities (coef 3 = 1/rho) on x,y tiles + the stored z term; normal stresses
  lane = 0;
  for (int k = 0; k < N; ++k) tab[1][lane++] = tile(0, 1, 2, k, SXX, SXY, U, 3, U);
  for (int k = 0; k < N; ++k) tab[1][lane++] = tile(0, 1, 2, k, SXY, SYY, V, 3, V);
  for (int k = 0; k < N; ++k) tab[1][lane++] = tile(0, 1, 2, k, SXZ, SYZ, Wq, 3, Wq);
  if (lane < 16 && lane + N > 16) lane = 16;  // the normal-stress lanes share one half-warp
  for (int k = 0; k < N; ++k) {
    TaskW t = tile(0, 1, 2, k, U, V, SXX, 1, SZZ);
    t.mode = MODE_NORMAL;
    t.dst2 = SYY * FS + k * st[2];
    t.dst3 = SZZ * FS + k * st[2];
    t.s2a = t.saA;
    t.s2b = t.sbA;
    tab[1][lane++] = t;
  }
}

template <int N>
cudaError_t launch_wpe_n(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  using G = GeoW<N>;
  ParamsW kp;
  for (int i = 0; i < 36; ++i) kp.d[i] = 0.0;
  for (int k = 0; k < N; ++k)
    for (int l = 0; l < N; ++l) kp.d[k * N + l] = p.basis.d[k * N + l];
  for (int j = 0; j < 6; ++j) {
    kp.phi[0][j] = j < N ? p.basis.face_left[j] : 0.0;
    kp.phi[1][j] = j < N ? p.basis.face_right[j] : 0.0;
  }
  kp.check = p.check;
  kp.par_kind = p.par_kind;
  kp.q_stride = p.q_stride;
  kp.prefetch = p.dmma8_prefetch ? 1 : 0;
  {
    double c = a.dt;  // same operation sequence as proj/src/stp_splitck.cpp:45,64
    kp.cf[0] = c;
    for (int o = 1; o < 8; ++o) {
      c *= a.dt / (o + 1);
      kp.cf[o] = c;
    }
  }
  auto kern = stp_wpe_kernel<N>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  if (err != cudaSuccess) return err;
  if (a.n_elem == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(a.n_elem < sms ? a.n_elem : sms);
  kern<<<grid, G::WPC * 32, G::SMEM, stream>>>(kp, a, p.d_status);
  return cudaGetLastError();
}

}  // namespace

bool wpe_applicable(const LaunchPlan& p, const BatchArgs& a) {
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  const bool sel = p.wpe == 1 ? (p.n >= 4 && p.n <= 6) : p.wpe == 2 && ((p.n == 4 && a.n_elem >= kWpeMinElems4) || (p.n == 5 && a.n_elem >= kWpeMinElems5));
  return sel && p.kind == ADERSTP_PDE_ELASTIC && p.src_comp < 0 &&
         p.layout == ADERSTP_LAYOUT_AOSOA && p.out_stride == 9 && p.q_stride >= 9 && p.q_stride <= 64 &&
         !p.force_generic && !a.u_next && a.qavg && al16(a.q) && al16(a.qavg) && al16(a.favg) && al16(a.face_q) &&
         al16(a.face_f);
}

cudaError_t init_wpe(const LaunchPlan& p) {
  if (p.n < 4 || p.n > 6) return cudaSuccess;
  TaskW tab[2][32];
  if (p.n == 6) build_tasks<6>(tab);
  else if (p.n == 5) build_tasks<5>(tab);
  else build_tasks<4>(tab);
  return cudaMemcpyToSymbol(kTaskW, tab, sizeof(tab), sizeof(tab) * (p.n - 4));
}

cudaError_t launch_wpe(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream) {
  if (p.n == 6) return launch_wpe_n<6>(p, a, stream);
  if (p.n == 5) return launch_wpe_n<5>(p, a, stream);
  if (p.n == 4) return launch_wpe_n<4>(p, a, stream);
  return cudaErrorInvalidValue;
}

}  // namespace aderstp
