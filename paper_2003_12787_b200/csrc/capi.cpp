// Host side of the C ABI (include/aderstp.h): plans, argument validation with the reference's
// validate_stp semantics (proj/src/predictor_common.cpp:129-146), PDE term tables from the
// reference's LinearPde factories (proj/src/pde.cpp), and the pipelined host-buffer path.
#include <algorithm>
#include <cmath>
#include <limits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <new>
#include <string>

#include "../../include/aderstp.h"
#include "aderstp_internal.h"

using aderstp::HostBasis;
using aderstp::LaunchPlan;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(ADERSTP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr int kHostStreams = 3;
// per-call device scratch of the AoS staged path
constexpr long long kStageBytes = 512ll << 20;

// the reference layout through device transposes to a tuned AoSoA kernel: the elastic PDE, and
// table PDEs with m <= 9 at nDof 8 (stp_dmma8_table)
bool aos_staged(const aderstp::LaunchPlan& lp) {
  const bool tuned = lp.kind == ADERSTP_PDE_ELASTIC || (lp.kind != ADERSTP_PDE_ELASTIC_SOURCE && lp.n == 8 && lp.m <= 9);
  return tuned && lp.src_comp < 0 && lp.layout == ADERSTP_LAYOUT_AOS && !lp.force_generic &&
         lp.gen.t_ptr == nullptr;  // the general kernel reads and writes the AoS rows itself
}

cudaMemPoolProps& pool_props_of(int device) {
  static thread_local cudaMemPoolProps props;
  std::memset(&props, 0, sizeof props);
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  return props;
}

}  // namespace

struct aderstp_plan {
  LaunchPlan lp;
  int device = 0;
  // host-buffer path scratch (allocated on first use or by aderstp_plan_reserve_host_path)
  int64_t chunk = 0;
  double* buf[kHostStreams] = {nullptr, nullptr, nullptr};
  cudaStream_t streams[kHostStreams] = {nullptr, nullptr, nullptr};
  // stream-ordered scratch (AoS staging, time-loop buffers): a plan-owned pool that keeps its
  // memory between calls (no re-mapping per call) until aderstp_plan_trim / destroy
  cudaMemPool_t pool = nullptr;
  // general kernel tables (CSR rows of C_d and A_d; one cudaMalloc) and the corrector's point
  // source projection (n^3 doubles)
  void* gen_buf = nullptr;
  double* src_proj = nullptr;
};

namespace {

// Build the per-(s,d) term tables from flux Jacobians A_d and ncp matrices B_d (row-major
// m x m): t-terms from A_d + B_d (the CK step applies D_d F_d(p) + B_d D_d p, equal to
// D_d (A_d + B_d) p for constant coefficients), favg terms from A_d alone.
int build_terms(LaunchPlan& lp, const double* A[3], const double* B[3]) {
  const int m = lp.m;
  std::memset(lp.tr, 0, sizeof lp.tr);
  std::memset(lp.fr, 0, sizeof lp.fr);
  for (int s = 0; s < aderstp::kMaxM; ++s)
    for (int d = 0; d < 3; ++d)
      for (int k = 0; k < aderstp::kMaxTerms; ++k) lp.tc[s][d][k] = lp.fc[s][d][k] = 0.0;
  int max_terms = 1;
  for (int s = 0; s < m; ++s)
    for (int d = 0; d < 3; ++d) {
      int nt = 0, nf = 0;
      for (int r = 0; r < m; ++r) {
        const double a = A[d] ? A[d][s * m + r] : 0.0;
        const double b = B[d] ? B[d][s * m + r] : 0.0;
        if (!std::isfinite(a) || !std::isfinite(b))
          return fail(ADERSTP_ERR_INVALID_ARG, "linear pde: non-finite coefficient");
        const double c = a + b;
        if (c != 0.0) {
          if (nt == aderstp::kMaxTerms)
            return fail(ADERSTP_ERR_UNSUPPORTED, "linear pde: more than 4 nonzeros in a row of A_d+B_d");
          lp.tr[s][d][nt] = (signed char)r;
          lp.tc[s][d][nt] = c;
          ++nt;
        }
        if (a != 0.0) {
          if (nf == aderstp::kMaxTerms)
            return fail(ADERSTP_ERR_UNSUPPORTED, "linear pde: more than 4 nonzeros in a row of A_d");
          lp.fr[s][d][nf] = (signed char)r;
          lp.fc[s][d][nf] = a;
          ++nf;
        }
      }
      if (nt > max_terms) max_terms = nt;
      if (nf > max_terms) max_terms = nf;
    }
  lp.n_terms = max_terms;
  return ADERSTP_OK;
}

// The general kernel's tables: CSR rows (s, d) of C_d = A_d + B_d (the CK step) and of A_d
// (favg, face_f), zeros dropped, in one device allocation owned by the plan.
cudaError_t upload_general(aderstp_plan* p, const std::vector<double>& A, const std::vector<double>& B) {
  const int m = p->lp.m;
  std::vector<int> tp(3 * m + 1, 0), fp(3 * m + 1, 0), tc, fc;
  std::vector<double> tv, fv;
  for (int s = 0; s < m; ++s)
    for (int d = 0; d < 3; ++d) {
      for (int j = 0; j < m; ++j) {
        const double a = A[(size_t)d * m * m + s * m + j], c = a + B[(size_t)d * m * m + s * m + j];
        if (c != 0.0) {
          tc.push_back(j);
          tv.push_back(c);
        }
        if (a != 0.0) {
          fc.push_back(j);
          fv.push_back(a);
        }
      }
      tp[3 * s + d + 1] = (int)tc.size();
      fp[3 * s + d + 1] = (int)fc.size();
    }
  // dense C_d [d][j][s < mp] (mp = m rounded up to 8: whole target blocks of the dense phase 2)
  // and dense A_d in the same layout (stp_gdense's favg / face_f GEMMs)
  const int mp = (m + 7) / 8 * 8;
  std::vector<double> cd(6 * (size_t)m * mp, 0.0);
  for (int d = 0; d < 3; ++d)
    for (int s = 0; s < m; ++s)
      for (int j = 0; j < m; ++j) {
        cd[((size_t)d * m + j) * mp + s] = A[(size_t)d * m * m + s * m + j] + B[(size_t)d * m * m + s * m + j];
        cd[((size_t)(3 + d) * m + j) * mp + s] = A[(size_t)d * m * m + s * m + j];
      }
  // layout: [cd][t_val][f_val][t_ptr][f_ptr][t_col][f_col] (doubles first: 16-byte alignment)
  const size_t bytes = sizeof(double) * (cd.size() + tv.size() + fv.size()) +
                       sizeof(int) * (tp.size() + fp.size() + tc.size() + fc.size());
  std::vector<char> host(bytes > 0 ? bytes : 8);
  char* h = host.data();
  size_t off = 0;
  auto put = [&](const void* src, size_t n) {
    if (n) std::memcpy(h + off, src, n);
    const size_t at = off;
    off += n;
    return at;
  };
  const size_t o_cd = put(cd.data(), sizeof(double) * cd.size());
  const size_t o_tv = put(tv.data(), sizeof(double) * tv.size());
  const size_t o_fv = put(fv.data(), sizeof(double) * fv.size());
  const size_t o_tp = put(tp.data(), sizeof(int) * tp.size());
  const size_t o_fp = put(fp.data(), sizeof(int) * fp.size());
  const size_t o_tc = put(tc.data(), sizeof(int) * tc.size());
  const size_t o_fc = put(fc.data(), sizeof(int) * fc.size());
  cudaError_t e = cudaMalloc(&p->gen_buf, host.size());
  if (e == cudaSuccess) e = cudaMemcpy(p->gen_buf, h, host.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  char* dv = static_cast<char*>(p->gen_buf);
  aderstp::LaunchPlan::GeneralTables& g = p->lp.gen;
  g.t_dense = reinterpret_cast<const double*>(dv + o_cd);
  g.f_dense = g.t_dense + 3 * (size_t)m * mp;
  g.t_val = reinterpret_cast<const double*>(dv + o_tv);
  g.f_val = reinterpret_cast<const double*>(dv + o_fv);
  g.t_ptr = reinterpret_cast<const int*>(dv + o_tp);
  g.f_ptr = reinterpret_cast<const int*>(dv + o_fp);
  g.t_col = reinterpret_cast<const int*>(dv + o_tc);
  g.f_col = reinterpret_cast<const int*>(dv + o_fc);
  g.scale = 1.0;
  g.t_nnz = (int)tv.size();
  return cudaSuccess;
}

// point_source_projection (proj/src/basis.cpp:124-142) with the reference's operation order:
// phi_x phi_y phi_z / (w_x w_y w_z) at node (k3, k2, k1), for the corrector's source term
cudaError_t upload_source_projection(aderstp_plan* p) {
  const aderstp::LaunchPlan& lp = p->lp;
  const int n = lp.n;
  double phi[3][aderstp::kMaxOrder];
  for (int d = 0; d < 3; ++d) aderstp::lagrange_values(n, lp.basis.nodes, lp.src_pos[d], phi[d]);
  std::vector<double> proj((size_t)n * n * n);
  for (int k3 = 0; k3 < n; ++k3)
    for (int k2 = 0; k2 < n; ++k2)
      for (int k1 = 0; k1 < n; ++k1) {
        const double num = phi[0][k1] * phi[1][k2] * phi[2][k3];
        const double mass = lp.basis.weights[k1] * lp.basis.weights[k2] * lp.basis.weights[k3];
        proj[(k3 * n + k2) * n + k1] = num / mass;
      }
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p->src_proj), sizeof(double) * proj.size());
  if (e == cudaSuccess) e = cudaMemcpy(p->src_proj, proj.data(), sizeof(double) * proj.size(), cudaMemcpyHostToDevice);
  return e;
}

// time integral of the source amplitude over [t, t + dt], truncated like the predictor
// (corrector_step, proj/src/solver.cpp:266-278), on the source-scaled PDE
double source_integral(const aderstp::LaunchPlan& lp, double dt, double t) {
  double amp[aderstp::kMaxOrder];
  aderstp::source_amplitudes(lp, t, lp.n, amp);
  double sint = 0.0, coeff = dt;
  for (int o = 0; o < lp.n; ++o) {
    sint += coeff * amp[o];
    coeff *= dt / (o + 2);
  }
  return sint;
}

}  // namespace

extern "C" {

const char* aderstp_last_error(void) { return g_last_error.c_str(); }
int aderstp_abi_version(void) { return ADERSTP_ABI_VERSION; }
int aderstp_supported_order(int order) { return aderstp::kernel_available(order) ? 1 : 0; }

int aderstp_basis(int order, double* nodes, double* weights, double* d, double* face_left,
                  double* face_right) {
  HostBasis b;
  if (aderstp::make_host_basis(order, &b) != 0)
    return fail(ADERSTP_ERR_INVALID_ARG, "basis: order out of range");
  const int n = order;
  if (nodes) std::memcpy(nodes, b.nodes, sizeof(double) * n);
  if (weights) std::memcpy(weights, b.weights, sizeof(double) * n);
  if (d) std::memcpy(d, b.d, sizeof(double) * n * n);
  if (face_left) std::memcpy(face_left, b.face_left, sizeof(double) * n);
  if (face_right) std::memcpy(face_right, b.face_right, sizeof(double) * n);
  return ADERSTP_OK;
}

double aderstp_flop_count(int order, int quantities) {
  const double n = order, m = quantities;
  return m * n * n * n * ((n - 1.0) * (6.0 * n + 8.0) + 28.0);
}

double aderstp_byte_count(int order, int quantities, int with_favg) {
  const double n = order, m = quantities;
  return 8.0 * m * ((with_favg ? 5.0 : 2.0) * n * n * n + 12.0 * n * n) + 24.0;
}

int aderstp_plan_create(const aderstp_config* cfg, aderstp_plan** out) {
  if (!cfg || !out) return fail(ADERSTP_ERR_INVALID_ARG, "plan_create: null argument");
  *out = nullptr;
  const int n = cfg->order, m = cfg->quantities;
  if (!aderstp::kernel_available(n))
    return fail(ADERSTP_ERR_UNSUPPORTED, "plan_create: order " + std::to_string(n) +
                                             " has no compiled kernel (2..10)");
  if (m < 1 || m > ADERSTP_MAX_QUANTITIES)
    return fail(ADERSTP_ERR_UNSUPPORTED, "plan_create: quantity count out of range (1.." +
                                             std::to_string(ADERSTP_MAX_QUANTITIES) + ")");
  if (cfg->layout != ADERSTP_LAYOUT_AOSOA && cfg->layout != ADERSTP_LAYOUT_AOS)
    return fail(ADERSTP_ERR_INVALID_ARG, "plan_create: unknown layout");
  const int qs = cfg->q_stride ? cfg->q_stride : m;
  const int os = cfg->out_stride ? cfg->out_stride : m;
  if (qs < m || os < m || qs > 64 || os > 64)
    return fail(ADERSTP_ERR_INVALID_ARG, "plan_create: quantity strides must be in [m, 64]");
  const int kind = cfg->pde_kind;
  const bool elastic = kind == ADERSTP_PDE_ELASTIC || kind == ADERSTP_PDE_ELASTIC_SOURCE;
  if (elastic && m != 9)
    return fail(ADERSTP_ERR_INVALID_ARG, "stp: pde/tensor quantity mismatch (elastic has m = 9)");
  if (kind == ADERSTP_PDE_DEMO && m != 6)
    return fail(ADERSTP_ERR_INVALID_ARG, "stp: pde/tensor quantity mismatch (demo has m = 6)");
  if (kind < ADERSTP_PDE_ELASTIC || kind > ADERSTP_PDE_LINEAR)
    return fail(ADERSTP_ERR_INVALID_ARG, "plan_create: unknown pde kind");
  if (elastic && cfg->par_kind != ADERSTP_PAR_LAMBDA_MU_RHO && cfg->par_kind != ADERSTP_PAR_RHO_CP_CS)
    return fail(ADERSTP_ERR_INVALID_ARG, "plan_create: unknown parameter kind");

  aderstp_plan* p = new (std::nothrow) aderstp_plan();
  if (!p) return fail(ADERSTP_ERR_INVALID_ARG, "plan_create: out of host memory");
  LaunchPlan& lp = p->lp;
  lp.n = n;
  lp.m = m;
  lp.kind = elastic ? ADERSTP_PDE_ELASTIC : ADERSTP_PDE_LINEAR;
  lp.layout = cfg->layout;
  lp.q_stride = qs;
  lp.out_stride = os;
  lp.par_kind = cfg->par_kind;
  lp.check = cfg->check_inputs ? 1 : 0;
  {
    const char* env = std::getenv("ADERSTP_FORCE_GENERIC");
    lp.force_generic = (env && env[0] == '1') ? 1 : 0;
    const char* nd = std::getenv("ADERSTP_NO_DMMA8");
    lp.no_dmma8 = (nd && nd[0] == '1') ? 1 : 0;
    // L2 prefetch distance of the tensor-core kernels: one wave of SMs ahead (measured: C3 +5 %)
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* pf = std::getenv("ADERSTP_PREFETCH");
    lp.dmma8_prefetch = pf ? std::atoi(pf) : sms;
    const char* as = std::getenv("ADERSTP_AOS_STAGED");
    lp.aos_staged = (as && as[0] == '1') ? 1 : 0;
    const char* nq = std::getenv("ADERSTP_NO_DMMAP");
    lp.no_dmmap = (nq && nq[0] == '1') ? 1 : 0;
    const char* wp = std::getenv("ADERSTP_WPE");
    lp.wpe = wp ? (wp[0] == '1' ? 1 : 0) : 2;  // 2: automatic (large nDof 4 batches)
    const char* ng = std::getenv("ADERSTP_NO_GDENSE");
    lp.no_gdense = (ng && ng[0] == '1') ? 1 : 0;
    const char* ac = std::getenv("ADERSTP_AOS_CHUNK");
    lp.aos_chunk = ac ? std::atoi(ac) : 0;
    const char* ps = std::getenv("ADERSTP_PASS_SLOTS");
    lp.pass_slots = !ps ? 0 : (ps[0] == '6') ? 6 : (ps[0] == '1' && ps[1] == '2') ? 12 : 0;
  }
  aderstp::make_host_basis(n, &lp.basis);

  // PDE terms (proj/src/pde.cpp): advection :61-85, ncp-advection :87-117, demo :119-146
  int rc = ADERSTP_OK;
  bool general = false;
  std::vector<double> Av, Bv;  // dense A_d, B_d (3 x m x m) of the non-elastic kinds
  if (!elastic) {
    Av.assign(3 * (size_t)m * m, 0.0);
    Bv.assign(3 * (size_t)m * m, 0.0);
    double* A[3] = {Av.data(), Av.data() + m * m, Av.data() + 2 * m * m};
    double* B[3] = {Bv.data(), Bv.data() + m * m, Bv.data() + 2 * m * m};
    const double* pa[3] = {A[0], A[1], A[2]};
    const double* pb[3] = {B[0], B[1], B[2]};
    const double* v = cfg->pde_args;
    if (kind == ADERSTP_PDE_ADVECTION) {
      for (int d = 0; d < 3; ++d)
        for (int s = 0; s < m; ++s) A[d][s * m + s] = -v[d];
    } else if (kind == ADERSTP_PDE_NCP_ADVECTION) {
      for (int d = 0; d < 3; ++d)
        for (int s = 0; s < m; ++s) B[d][s * m + s] = -v[d];
    } else if (kind == ADERSTP_PDE_DEMO) {
      // x-flux rows F0 = -(Q0+Q3+Q4), F1 = -(Q1+Q3+Q5), F2 = -(Q2+Q4+Q5); y/z rotate the
      // quantity indices by (0 1 2)(3 4 5) (pde.hpp:66-70)
      const int rot[6] = {1, 2, 0, 4, 5, 3};
      int rows[3][3] = {{0, 3, 4}, {1, 3, 5}, {2, 4, 5}};
      int outs[3] = {0, 1, 2};
      for (int d = 0; d < 3; ++d) {
        for (int r = 0; r < 3; ++r)
          for (int j = 0; j < 3; ++j) A[d][outs[r] * m + rows[r][j]] = -1.0;
        for (int r = 0; r < 3; ++r) {
          outs[r] = rot[outs[r]];
          for (int j = 0; j < 3; ++j) rows[r][j] = rot[rows[r][j]];
        }
      }
    } else if (kind == ADERSTP_PDE_LINEAR) {
      for (int d = 0; d < 3; ++d) {
        if (cfg->linear[d]) std::memcpy(A[d], cfg->linear[d], sizeof(double) * m * m);
        if (cfg->linear[3 + d]) std::memcpy(B[d], cfg->linear[3 + d], sizeof(double) * m * m);
      }
    }
    for (double v : Av)
      if (!std::isfinite(v)) {
        delete p;
        return fail(ADERSTP_ERR_INVALID_ARG, "linear pde: non-finite coefficient");
      }
    for (double v : Bv)
      if (!std::isfinite(v)) {
        delete p;
        return fail(ADERSTP_ERR_INVALID_ARG, "linear pde: non-finite coefficient");
      }
    // the term-table kernels take m <= 16 and <= 4 nonzeros per (row, dim); everything else
    // (and ADERSTP_GENERAL=1) runs on the general kernel
    const char* ge = std::getenv("ADERSTP_GENERAL");
    general = (ge && ge[0] == '1') || m > aderstp::kMaxM;
    if (!general) {
      rc = build_terms(lp, pa, pb);
      if (rc == ADERSTP_ERR_UNSUPPORTED) general = true;
      else if (rc != ADERSTP_OK) {
        delete p;
        return rc;
      }
    }
    if (general) {
      std::memset(lp.tr, 0, sizeof lp.tr);
      std::memset(lp.fr, 0, sizeof lp.fr);
      for (int q = 0; q < aderstp::kMaxM; ++q)
        for (int d = 0; d < 3; ++d)
          for (int k = 0; k < aderstp::kMaxTerms; ++k) lp.tc[q][d][k] = lp.fc[q][d][k] = 0.0;
      lp.n_terms = 1;
    }
  } else {
    lp.n_terms = 1;
  }
  // point source (pde.hpp:47-56; weak Dirac projection predictor_common.cpp:261-283)
  if (kind == ADERSTP_PDE_ELASTIC_SOURCE || kind == ADERSTP_PDE_SOURCE_ONLY ||
      (kind == ADERSTP_PDE_LINEAR && cfg->pde_args[7] != 0.0)) {
    const double* a = cfg->pde_args;
    const int comp = (int)a[3];
    if (comp < 0 || comp >= m || (kind == ADERSTP_PDE_ELASTIC_SOURCE && (comp < 6 || comp > 8))) {
      delete p;
      return fail(ADERSTP_ERR_INVALID_ARG, "point source: component out of range");
    }
    if (!(a[6] > 0.0)) {
      delete p;
      return fail(ADERSTP_ERR_INVALID_ARG, "point source: width must be positive");
    }
    lp.src_comp = comp;
    lp.src_amp = a[4];
    lp.src_center = a[5];
    lp.src_width = a[6];
    for (int d = 0; d < 3; ++d) {
      lp.src_pos[d] = a[d];
      double phi[aderstp::kMaxOrder];
      aderstp::lagrange_values(n, lp.basis.nodes, a[d], phi);
      for (int j = 0; j < n; ++j) lp.src_proj[d][j] = phi[j] / lp.basis.weights[j];
    }
  } else {
    lp.src_comp = -1;
    for (int d = 0; d < 3; ++d)
      for (int j = 0; j < aderstp::kMaxOrder; ++j) lp.src_proj[d][j] = 0.0;
  }

  cudaError_t e = cudaGetDevice(&p->device);
  if (e == cudaSuccess) e = cudaMalloc(&lp.d_status, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(lp.d_status, 0, sizeof(unsigned int));
  if (e == cudaSuccess && general) e = upload_general(p, Av, Bv);
  if (e == cudaSuccess && lp.src_comp >= 0) e = upload_source_projection(p);
  // device constants of the tuned kernels this plan can dispatch to -- for the reference AoS
  // layout those of its AoSoA staging (predict_aos_staged)
  aderstp::LaunchPlan kl = lp;
  if (aos_staged(lp)) {
    kl.layout = ADERSTP_LAYOUT_AOSOA;
    kl.q_stride = kl.out_stride = lp.m;
  }
  // plan-owned stream-ordered pool (AoS staging, time-loop faces): keeps its memory between
  // calls, returned when the plan is destroyed
  if (e == cudaSuccess) e = cudaMemPoolCreate(&p->pool, &pool_props_of(p->device));
  // keep what the plan's calls allocated (a time loop re-maps GBs of face buffers otherwise);
  // the AoS staging is capped at kStageBytes per call, and aderstp_plan_trim returns the rest
  const uint64_t keep = UINT64_MAX;
  if (e == cudaSuccess) e = cudaMemPoolSetAttribute(p->pool, cudaMemPoolAttrReleaseThreshold, (void*)&keep);
  // D of nDof 8 in the constant bank: the elastic and the table-PDE tensor-core kernels
  if (e == cudaSuccess && kl.n == 8) e = aderstp::init_dmma8(kl);
  if (e == cudaSuccess && (aderstp::pass_applicable(kl) || (kl.kind != ADERSTP_PDE_ELASTIC && kl.n >= 9)))
    e = aderstp::init_pass(kl);  // the even/odd D of the line-pass kernels (stp_pass, stp_bip, stp_tlp)
  if (e == cudaSuccess && aderstp::dmmap_applicable(kl)) e = aderstp::init_dmmap(kl);
  if (e == cudaSuccess && kl.wpe && kl.kind == ADERSTP_PDE_ELASTIC) e = aderstp::init_wpe(kl);
  if (e == cudaSuccess && kl.kind != ADERSTP_PDE_ELASTIC && kl.n >= 5 && kl.n <= 7) e = aderstp::init_dmmat(kl);
  if (e == cudaSuccess) lp.gen.pool = p->pool;
  if (e != cudaSuccess) {
    aderstp_plan_destroy(p);
    return cuda_fail(e, "plan_create");
  }
  *out = p;
  return ADERSTP_OK;
}

void aderstp_plan_destroy(aderstp_plan* p) {
  if (!p) return;
  for (int i = 0; i < kHostStreams; ++i) {
    if (p->buf[i]) cudaFree(p->buf[i]);
    if (p->streams[i]) cudaStreamDestroy(p->streams[i]);
  }
  if (p->lp.d_status) cudaFree(p->lp.d_status);
  if (p->gen_buf) cudaFree(p->gen_buf);
  if (p->src_proj) cudaFree(p->src_proj);
  if (p->pool) cudaMemPoolDestroy(p->pool);
  delete p;
}

namespace {

int validate_batch(const aderstp_plan* p, int64_t n_elem, const double* q, const double* par,
                   double dt, const double* qavg, const double* favg, const double* face_f) {
  if (!p) return fail(ADERSTP_ERR_INVALID_ARG, "stp: null plan");
  if (n_elem < 0) return fail(ADERSTP_ERR_INVALID_ARG, "stp: negative element count");
  if (!(dt > 0.0)) return fail(ADERSTP_ERR_INVALID_ARG, "stp: dt must be positive");
  if (n_elem > 0 && !q) return fail(ADERSTP_ERR_INVALID_ARG, "stp: null input tensor");
  if (n_elem > 0 && !qavg) return fail(ADERSTP_ERR_INVALID_ARG, "stp: null qavg output");
  if (n_elem > 0 && p->lp.kind == ADERSTP_PDE_ELASTIC && !par)
    return fail(ADERSTP_ERR_INVALID_ARG, "stp: elastic kinds need per-element parameters");
  (void)favg;
  (void)face_f;
  return ADERSTP_OK;
}

}  // namespace

namespace {

// The reference's own layout (AoS ElementTensor, m_pad = 16) for the elastic PDE: the element
// tensors are transposed to the native AoSoA layout on the device (aderstp_convert_layout's
// kernel) in chunks through stream-ordered scratch (cudaMallocAsync: no shared plan state, so
// calls stay thread-safe), the tuned kernel runs, and qavg / favg are transposed back; the face
// arrays have the same layout in both and are written directly.  3-8x faster than running the
// generic kernel on AoS data.

cudaError_t predict_aos_staged(const aderstp_plan* plan, const aderstp::BatchArgs& a, cudaStream_t st) {
  const aderstp::LaunchPlan& lp = plan->lp;
  aderstp::LaunchPlan sp = lp;
  sp.layout = ADERSTP_LAYOUT_AOSOA;
  const int n = lp.n, m = lp.m;  // compact AoSoA staging: quantity stride m
  sp.q_stride = m;
  sp.out_stride = m;
  const size_t t9 = (size_t)n * n * n * m;  // one AoSoA tensor (doubles)
  const size_t per = t9 * (a.favg ? 5 : 2);  // q, qavg (+ favg[3])
  // staging capped at kStageBytes per call (a few waves of CTAs at every order)
  long long chunk = std::max<long long>(1, std::min<long long>(a.n_elem, kStageBytes / (long long)(per * 8)));
  if (lp.aos_chunk > 0) chunk = std::min<long long>(chunk, lp.aos_chunk);  // tests: force several chunks
  double* buf = nullptr;
  cudaError_t err = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&buf), sizeof(double) * per * chunk, plan->pool, st);
  if (err != cudaSuccess) return err;
  double* sq = buf;
  double* sqa = buf + t9 * chunk;
  double* sfa = a.favg ? buf + 2 * t9 * chunk : nullptr;
  const size_t face = 6 * (size_t)n * n * lp.m;
  const size_t qin = (size_t)n * n * n * lp.q_stride, qout = (size_t)n * n * n * lp.out_stride;
  for (long long e0 = 0; e0 < a.n_elem && err == cudaSuccess; e0 += chunk) {
    const long long c = std::min(chunk, a.n_elem - e0);
    err = aderstp::launch_convert(n, m, c, ADERSTP_LAYOUT_AOS, lp.q_stride, a.q + e0 * qin, ADERSTP_LAYOUT_AOSOA, m,
                                  sq, st);
    aderstp::BatchArgs b{sq, a.par ? a.par + 3 * e0 : nullptr, sqa, sfa, a.face_q ? a.face_q + e0 * face : nullptr,
                         a.face_f ? a.face_f + e0 * face : nullptr, c, a.dt, a.t_start};
    if (err == cudaSuccess) err = aderstp::launch_stp(sp, b, st);
    if (err == cudaSuccess)
      err = aderstp::launch_convert(n, m, c, ADERSTP_LAYOUT_AOSOA, m, sqa, ADERSTP_LAYOUT_AOS, lp.out_stride,
                                    a.qavg + e0 * qout, st);
    if (sfa && err == cudaSuccess)  // favg[e][d][...]: three consecutive tensors per element in both layouts
      err = aderstp::launch_convert(n, m, 3 * c, ADERSTP_LAYOUT_AOSOA, m, sfa, ADERSTP_LAYOUT_AOS, lp.out_stride,
                                    a.favg + e0 * 3 * qout, st);
  }
  cudaFreeAsync(buf, st);
  return err;
}

}  // namespace

// the device-side dispatch of one batch: the reference layout straight into the nDof 8 kernel,
// through the device transposes for the other orders, every other case to launch_stp
cudaError_t predict_device(const aderstp_plan* p, const aderstp::BatchArgs& a, cudaStream_t st) {
  if (aderstp::dmma8_aos_applicable(p->lp, a)) return aderstp::launch_dmma8(p->lp, a, st);
  if (aderstp::bip_aos_applicable(p->lp, a)) return aderstp::launch_bip(p->lp, a, st);
  if (aderstp::dmmap_aos_applicable(p->lp, a)) return aderstp::launch_dmmap(p->lp, a, st);
  if (aos_staged(p->lp) && p->pool) return predict_aos_staged(p, a, st);
  return aderstp::launch_stp(p->lp, a, st);
}

int aderstp_predict_batch(const aderstp_plan* p, int64_t n_elem, const double* q,
                          const double* par, double dt, double t_start, double* qavg,
                          double* favg, double* face_q, double* face_f, void* stream) {
  int rc = validate_batch(p, n_elem, q, par, dt, qavg, favg, face_f);
  if (rc != ADERSTP_OK) return rc;
  if (n_elem == 0) return ADERSTP_OK;
  aderstp::BatchArgs a{q, par, qavg, favg, face_q, face_f, (long long)n_elem, dt, t_start};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = predict_device(p, a, st);
  if (e != cudaSuccess) return cuda_fail(e, "predict_batch launch");
  return ADERSTP_OK;
}

int aderstp_plan_trim(aderstp_plan* p) {
  if (!p) return fail(ADERSTP_ERR_INVALID_ARG, "plan_trim: null plan");
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess && p->pool) e = cudaMemPoolTrimTo(p->pool, 0);
  if (e != cudaSuccess) return cuda_fail(e, "plan_trim");
  return ADERSTP_OK;
}

int aderstp_plan_status(aderstp_plan* p, void* stream) {
  if (!p) return fail(ADERSTP_ERR_INVALID_ARG, "plan_status: null plan");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned int flags = 0;
  cudaError_t e = cudaMemcpyAsync(&flags, p->lp.d_status, sizeof flags, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p->lp.d_status, 0, sizeof flags, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "plan_status");
  if (flags & 1u) return fail(ADERSTP_ERR_NONFINITE, "stp: non-finite input DOFs");
  if (flags & 2u)
    return fail(ADERSTP_ERR_MATERIAL, "elastic_pde: need rho > 0, mu >= 0, lambda + 2mu > 0");
  return ADERSTP_OK;
}

namespace {

struct ChunkLayout {
  size_t q, par, qavg, favg, face;  // doubles per element
};

ChunkLayout chunk_layout(const LaunchPlan& lp) {
  const size_t n3 = (size_t)lp.n * lp.n * lp.n;
  ChunkLayout c;
  c.q = n3 * lp.q_stride;
  c.par = 3;
  c.qavg = n3 * lp.out_stride;
  c.favg = 3 * c.qavg;
  c.face = 6 * (size_t)lp.n * lp.n * lp.m;
  return c;
}

// device sub-buffers of one chunk slot, each starting on a 256-byte boundary
size_t round256(size_t doubles) { return (doubles + 31) / 32 * 32; }
size_t chunk_doubles(const ChunkLayout& c, int64_t chunk) {
  return round256(c.q * chunk) + round256(c.par * chunk) + round256(c.qavg * chunk) +
         round256(c.favg * chunk) + 2 * round256(c.face * chunk);
}

}  // namespace

int aderstp_plan_reserve_host_path(aderstp_plan* p, int64_t chunk_elems) {
  if (!p || chunk_elems <= 0) return fail(ADERSTP_ERR_INVALID_ARG, "reserve_host_path: bad argument");
  if (p->chunk >= chunk_elems) return ADERSTP_OK;
  for (int i = 0; i < kHostStreams; ++i) {
    if (p->buf[i]) cudaFree(p->buf[i]);
    p->buf[i] = nullptr;
  }
  const ChunkLayout c = chunk_layout(p->lp);
  for (int i = 0; i < kHostStreams; ++i) {
    cudaError_t e = cudaSuccess;
    if (!p->streams[i]) e = cudaStreamCreateWithFlags(&p->streams[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&p->buf[i], sizeof(double) * chunk_doubles(c, chunk_elems));
    if (e != cudaSuccess) {
      p->chunk = 0;
      return cuda_fail(e, "reserve_host_path");
    }
  }
  p->chunk = chunk_elems;
  return ADERSTP_OK;
}

int aderstp_predict_batch_host(aderstp_plan* p, int64_t n_elem, const double* q,
                               const double* par, double dt, double t_start, double* qavg,
                               double* favg, double* face_q, double* face_f) {
  int rc = validate_batch(p, n_elem, q, par, dt, qavg, favg, face_f);
  if (rc != ADERSTP_OK) return rc;
  if (n_elem == 0) return ADERSTP_OK;
  const ChunkLayout c = chunk_layout(p->lp);
  if (p->chunk == 0) {
    // ~256 MiB of device traffic per chunk
    const size_t per = c.q + c.par + c.qavg + c.favg + 2 * c.face;
    int64_t ch = (int64_t)((256u << 20) / (per * sizeof(double)));
    if (ch < 1) ch = 1;
    rc = aderstp_plan_reserve_host_path(p, ch);
    if (rc != ADERSTP_OK) return rc;
  }
  const int64_t chunk = p->chunk;
  const bool elastic = p->lp.kind == ADERSTP_PDE_ELASTIC;
  int64_t done = 0;
  int slot = 0;
  cudaError_t e = cudaSuccess;
  while (done < n_elem && e == cudaSuccess) {
    const int64_t cnt = (n_elem - done < chunk) ? n_elem - done : chunk;
    cudaStream_t st = p->streams[slot];
    double* b = p->buf[slot];
    double* dq = b;
    double* dpar = dq + round256(c.q * chunk);
    double* dqa = dpar + round256(c.par * chunk);
    double* dfa = dqa + round256(c.qavg * chunk);
    double* dfq = dfa + round256(c.favg * chunk);
    double* dff = dfq + round256(c.face * chunk);
    e = cudaMemcpyAsync(dq, q + done * c.q, sizeof(double) * c.q * cnt, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && elastic)
      e = cudaMemcpyAsync(dpar, par + done * 3, sizeof(double) * 3 * cnt, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      aderstp::BatchArgs a{dq, elastic ? dpar : nullptr, dqa, favg ? dfa : nullptr,
                           face_q ? dfq : nullptr, face_f ? dff : nullptr, (long long)cnt, dt, t_start};
      e = predict_device(p, a, st);
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(qavg + done * c.qavg, dqa, sizeof(double) * c.qavg * cnt, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && favg)
      e = cudaMemcpyAsync(favg + done * c.favg, dfa, sizeof(double) * c.favg * cnt, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && face_q)
      e = cudaMemcpyAsync(face_q + done * c.face, dfq, sizeof(double) * c.face * cnt, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && face_f)
      e = cudaMemcpyAsync(face_f + done * c.face, dff, sizeof(double) * c.face * cnt, cudaMemcpyDeviceToHost, st);
    done += cnt;
    slot = (slot + 1) % kHostStreams;
  }
  for (int i = 0; i < kHostStreams; ++i) {
    cudaError_t e2 = cudaStreamSynchronize(p->streams[i]);
    if (e == cudaSuccess) e = e2;
  }
  if (e != cudaSuccess) return cuda_fail(e, "predict_batch_host");
  return p->lp.check ? aderstp_plan_status(p, p->streams[0]) : ADERSTP_OK;
}

int aderstp_convert_layout(int order, int quantities, int64_t n_elem, int src_layout,
                           int src_stride, const double* src, int dst_layout, int dst_stride,
                           double* dst, void* stream) {
  if (order < 1 || order > 64 || quantities < 1 || src_stride < quantities || dst_stride < quantities)
    return fail(ADERSTP_ERR_INVALID_ARG, "convert_layout: bad shape");
  if ((src_layout != ADERSTP_LAYOUT_AOS && src_layout != ADERSTP_LAYOUT_AOSOA) ||
      (dst_layout != ADERSTP_LAYOUT_AOS && dst_layout != ADERSTP_LAYOUT_AOSOA))
    return fail(ADERSTP_ERR_INVALID_ARG, "convert_layout: unknown layout");
  if (n_elem < 0 || (n_elem > 0 && (!src || !dst)))
    return fail(ADERSTP_ERR_INVALID_ARG, "convert_layout: bad buffers");
  if (src == dst && n_elem > 0) return fail(ADERSTP_ERR_INVALID_ARG, "convert_layout: in-place not supported");
  cudaError_t e = aderstp::launch_convert(order, quantities, n_elem, src_layout, src_stride, src,
                                          dst_layout, dst_stride, dst, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "convert_layout");
  return ADERSTP_OK;
}

int aderstp_generate(int dist, uint64_t seed, int order, int64_t e0, int64_t n_elem, int grid,
                     int layout, int q_stride, double* q, double* par, void* stream) {
  if (dist < 0 || dist > 2) return fail(ADERSTP_ERR_INVALID_ARG, "generate: unknown distribution");
  if (order < 1 || order > aderstp::kMaxOrder || q_stride < 9 || e0 < 0 || n_elem < 0)
    return fail(ADERSTP_ERR_INVALID_ARG, "generate: bad shape");
  if (dist == 2 && grid < 1) return fail(ADERSTP_ERR_INVALID_ARG, "generate: grid must be >= 1");
  HostBasis b;
  aderstp::make_host_basis(order, &b);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (q && q_stride > 9 && n_elem > 0) {
    cudaError_t e = cudaMemsetAsync(q, 0, sizeof(double) * (size_t)n_elem * order * order * order * q_stride, st);
    if (e != cudaSuccess) return cuda_fail(e, "generate");
  }
  cudaError_t e = aderstp::launch_generate(dist, seed, order, e0, n_elem, grid, layout, q_stride,
                                           b, q, par, st);
  if (e != cudaSuccess) return cuda_fail(e, "generate");
  return ADERSTP_OK;
}

}  // extern "C"

// ---- GPU corrector and time loop ------------------------------------

namespace {

int validate_mesh(const aderstp_plan* p, const aderstp_mesh* mesh, const double* u, const double* par,
                  const char* who) {
  if (!p || !mesh || !u) return fail(ADERSTP_ERR_INVALID_ARG, std::string(who) + ": null argument");
  if (mesh->elements_per_dim < 1)
    return fail(ADERSTP_ERR_INVALID_ARG, "Mesh: need at least one element per dimension");
  if (!(mesh->domain_len > 0.0)) return fail(ADERSTP_ERR_INVALID_ARG, "Mesh: domain length must be positive");
  if ((double)mesh->elements_per_dim * mesh->elements_per_dim * mesh->elements_per_dim > 2147483647.0)
    return fail(ADERSTP_ERR_INVALID_ARG, std::string(who) + ": mesh too large");
  if (p->lp.kind == ADERSTP_PDE_ELASTIC && !par)
    return fail(ADERSTP_ERR_INVALID_ARG, std::string(who) + ": elastic kinds need per-element parameters");
  return ADERSTP_OK;
}

// One corrector step on the elements of `a` (a slab, or the whole mesh when a.nz == 0), with
// lp's status word: the volume term u += V(qavg) (the general kernel for general systems, the
// tensor-core nDof 8 kernel in its volume mode for the elastic system, else inside the corrector
// kernel), the point source u[comp] += proj * sint (solver.cpp:206-216), the surface terms.
cudaError_t corrector_launch(const aderstp_plan* p, const aderstp::LaunchPlan& lp, aderstp::CorrArgs a,
                             double dt, double t, cudaStream_t st) {
  const long long E = (long long)a.e * a.e * (a.nz > 0 ? a.nz : a.e);
  if (lp.src_comp >= 0) {  // ScaledPde(1/h, 1/h^3): the source scale of an element of size h
    aderstp::LaunchPlan sl = lp;
    sl.src_scale = a.inv_h * a.inv_h * a.inv_h;
    a.src_comp = lp.src_comp;
    a.src_sint = source_integral(sl, dt, t);
    a.src_proj = p->src_proj;
  }
  if (E == 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  if (a.qavg && aderstp::general_selected(lp)) {
    aderstp::BatchArgs vb{a.u, nullptr, nullptr, nullptr, nullptr, nullptr, E, 1.0, 0.0};
    vb.u_next = a.u;
    vb.vol_r = a.qavg;
    aderstp::LaunchPlan gl = lp;
    gl.gen.scale = a.inv_h;  // ScaledPde: flux and ncp x 1/h
    e = aderstp::launch_general(gl, vb, st);
    a.qavg = nullptr;  // the volume term is applied
  } else if (a.qavg && aderstp::dmma8_applicable(lp) && !lp.force_generic && !lp.no_dmma8 && al16(a.u) &&
             al16(a.qavg)) {
    // elastic nDof 8: the volume term on the tensor cores -- stp_dmma8's last Horner step with the
    // iterate started from qavg on the 1/h-scaled material, u <- u + V(qavg) in place
    aderstp::BatchArgs vb{a.u, nullptr, nullptr, nullptr, nullptr, nullptr, E, 1.0, 0.0};
    vb.u_next = a.u;
    vb.vol_r = a.qavg;
    double* par_s = nullptr;
    e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&par_s), sizeof(double) * 3 * E, p->pool, st);
    if (e == cudaSuccess) e = aderstp::launch_scale_par(a.par, lp.par_kind, a.inv_h, E, par_s, st);
    aderstp::LaunchPlan sp = lp;
    sp.par_kind = ADERSTP_PAR_LAMBDA_MU_RHO;
    vb.par = par_s;
    if (e == cudaSuccess) e = aderstp::launch_dmma8(sp, vb, st);
    if (par_s) cudaFreeAsync(par_s, st);
    a.qavg = nullptr;
  }
  if (e == cudaSuccess) e = aderstp::launch_correct(lp, a, st);
  return e;
}

}  // namespace

int aderstp_correct_batch(const aderstp_plan* p, const aderstp_mesh* mesh, double* u, const double* par,
                          const double* qavg, const double* face_q, const double* face_f,
                          double max_wavespeed, double dt, double t, void* stream) {
  int rc = validate_mesh(p, mesh, u, par, "corrector_step");
  if (rc != ADERSTP_OK) return rc;
  if (!qavg || !face_q || !face_f)
    return fail(ADERSTP_ERR_INVALID_ARG, "corrector_step: one predictor output per element required");
  if (p->lp.kind != ADERSTP_PDE_ELASTIC && !(max_wavespeed >= 0.0))
    return fail(ADERSTP_ERR_INVALID_ARG, "corrector_step: max_wavespeed required for table PDEs");
  const double inv_h = mesh->elements_per_dim / mesh->domain_len;
  aderstp::CorrArgs a{u, par, qavg, face_q, face_f, mesh->elements_per_dim, inv_h,
                      max_wavespeed >= 0.0 ? max_wavespeed * inv_h : -1.0};
  cudaError_t e = corrector_launch(p, p->lp, a, dt, t, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "correct_batch launch");
  return ADERSTP_OK;
}

namespace {

// The time loop of run_simulation (src/solver.cpp:313-359) on the slab [z0, z0 + nz): predictor on
// ScaledPde(1/h), a rank sync, the corrector (z-neighbours outside the slab from lo / hi), a rank
// sync with the stability flag.  face_q / face_f: caller buffers (n_local x 6 x n^2 m).
int run_loop(const aderstp_plan* p, const aderstp_mesh* mesh, int z0, int nz, double* u, const double* par,
             double* face_q, double* face_f, const aderstp::HaloRef& lo, const aderstp::HaloRef& hi, double cfl,
             double t_end, double smax, bool per_face_smax, aderstp_rank_sync_fn sync, void* ctx,
             int64_t* steps, double* t_final, cudaStream_t st) {
  const bool elastic = p->lp.kind == ADERSTP_PDE_ELASTIC;
  const int e = mesh->elements_per_dim;
  const long long E = (long long)e * e * nz;
  const int n = p->lp.n;
  const double h = mesh->domain_len / e, s = 1.0 / h;
  aderstp::LaunchPlan sp = p->lp;  // the predictor on ScaledPde(1/h, 1/h^3)
  sp.gen.scale = s;
  sp.src_scale = s * s * s;
  if (!elastic)
    for (int q = 0; q < aderstp::kMaxM; ++q)
      for (int d = 0; d < 3; ++d)
        for (int k = 0; k < aderstp::kMaxTerms; ++k) {
          sp.tc[q][d][k] *= s;
          sp.fc[q][d][k] *= s;
        }
  double *par_s = nullptr, *qavg = nullptr;
  unsigned int* status = nullptr;  // this call's own check word (slabs sharing a plan never mix)
  auto cleanup = [&]() {
    if (par_s) cudaFreeAsync(par_s, st);
    if (qavg) cudaFreeAsync(qavg, st);
    if (status) cudaFreeAsync(status, st);
  };
  cudaError_t err = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&status), sizeof(unsigned int), p->pool, st);
  if (err == cudaSuccess) err = cudaMemsetAsync(status, 0, sizeof(unsigned int), st);
  sp.d_status = status;
  aderstp::LaunchPlan cp = p->lp;  // the corrector reports into the same word
  cp.d_status = status;
  if (err == cudaSuccess && elastic) {
    err = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&par_s), sizeof(double) * 3 * (E > 0 ? E : 1), p->pool, st);
    if (err == cudaSuccess) err = aderstp::launch_scale_par(par, p->lp.par_kind, s, E, par_s, st);
    sp.par_kind = ADERSTP_PAR_LAMBDA_MU_RHO;
  }
  aderstp::BatchArgs probe{u, elastic ? par_s : par, nullptr, nullptr, face_q, face_f, E, 1.0, 0.0};
  probe.u_next = u;
  const bool fused = aderstp::fused_supported(sp, probe);
  if (err == cudaSuccess && !fused)
    err = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&qavg), sizeof(double) * (size_t)n * n * n * p->lp.out_stride * (E > 0 ? E : 1),
                                  p->pool, st);
  if (err != cudaSuccess) {
    cleanup();
    return cuda_fail(err, "run_simulation setup");
  }
  const double dt0 = smax > 0.0 ? cfl * h / (3.0 * smax * (2.0 * n - 1.0)) : std::numeric_limits<double>::infinity();
  double t = 0.0;
  int64_t done = 0;
  int rc = ADERSTP_OK;
  // rank-sync flag bits: 1 non-finite, 2 material, 4 a CUDA error on some rank.  Every rank makes
  // the same two sync calls per step whatever happened locally, so a failing rank never leaves
  // the others waiting in a collective: all of them leave the loop at the same step.
  constexpr int kRankError = 4;
  while (t < t_end - 1e-14 * std::max(1.0, t_end)) {
    const double dt = std::min(dt0, t_end - t);
    aderstp::BatchArgs ba{u, elastic ? par_s : par, fused ? nullptr : qavg, nullptr, face_q, face_f, E, dt, t};
    if (fused) ba.u_next = u;
    err = E > 0 ? aderstp::launch_stp(sp, ba, st) : cudaSuccess;
    // other slabs read this slab's faces: the rank sync needs them complete (one GPU: the
    // corrector below is stream-ordered after the predictor, no host round trip)
    if (err == cudaSuccess && sync) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) rc = cuda_fail(err, "run_simulation predictor");
    const int pre = sync ? sync(ctx, err != cudaSuccess ? kRankError : 0) : 0;  // every slab's faces are complete
    if (err != cudaSuccess) break;
    if (pre & kRankError) {
      rc = fail(ADERSTP_ERR_CUDA, "run_simulation: another rank failed");
      break;
    }
    aderstp::CorrArgs ca{u, par, fused ? nullptr : qavg, face_q, face_f, e, s, per_face_smax ? -1.0 : smax * s};
    ca.z0 = z0;
    ca.nz = nz;
    ca.lo = lo;
    ca.hi = hi;
    err = corrector_launch(p, cp, ca, dt, t, st);
    unsigned int flags = 0;
    if (err == cudaSuccess) err = cudaMemcpyAsync(&flags, status, sizeof flags, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err == cudaSuccess && flags) err = cudaMemsetAsync(status, 0, sizeof flags, st);
    if (err != cudaSuccess) rc = cuda_fail(err, "run_simulation corrector");
    const int local = err != cudaSuccess ? kRankError : (int)flags;
    const int any = sync ? sync(ctx, local) : local;  // nobody reads the faces any more
    if (err != cudaSuccess) break;
    if (any & kRankError) {
      rc = fail(ADERSTP_ERR_CUDA, "run_simulation: another rank failed");
      break;
    }
    if (any) {
      rc = fail((any & 2) ? ADERSTP_ERR_MATERIAL : ADERSTP_ERR_NONFINITE,
                (any & 2) ? "elastic_pde: need rho > 0, mu >= 0, lambda + 2mu > 0"
                          : "corrector_step: non-finite update (unstable)");
      break;
    }
    t += dt;
    ++done;
  }
  if (steps) *steps = done;
  if (t_final) *t_final = t;
  cleanup();
  return rc;
}

aderstp::HaloRef halo_of(const aderstp_halo* h) {
  aderstp::HaloRef r;
  if (h) {
    r.face_q = h->face_q;
    r.face_f = h->face_f;
    r.par = h->par;
    r.z_base = h->z_base;
  }
  return r;
}

int validate_slab(const aderstp_mesh* mesh, const aderstp_slab* slab, const aderstp_halo* lo,
                  const aderstp_halo* hi, bool elastic, const char* who) {
  if (!slab) return fail(ADERSTP_ERR_INVALID_ARG, std::string(who) + ": null slab");
  const int e = mesh->elements_per_dim;
  if (slab->z0 < 0 || slab->nz < 1 || slab->z0 + slab->nz > e)
    return fail(ADERSTP_ERR_INVALID_ARG, std::string(who) + ": slab outside the mesh");
  if (slab->nz < e) {
    if (!lo || !hi || !lo->face_q || !lo->face_f || !hi->face_q || !hi->face_f)
      return fail(ADERSTP_ERR_INVALID_ARG, std::string(who) + ": a partial slab needs both halos");
    if (elastic && (!lo->par || !hi->par))
      return fail(ADERSTP_ERR_INVALID_ARG, std::string(who) + ": elastic halos need the neighbours' material");
  }
  return ADERSTP_OK;
}

}  // namespace

int aderstp_correct_slab(const aderstp_plan* p, const aderstp_mesh* mesh, const aderstp_slab* slab, double* u,
                         const double* par, const double* qavg, const double* face_q, const double* face_f,
                         const aderstp_halo* lo, const aderstp_halo* hi, double max_wavespeed, double dt,
                         double t, void* stream) {
  int rc = validate_mesh(p, mesh, u, par, "corrector_step");
  if (rc == ADERSTP_OK) rc = validate_slab(mesh, slab, lo, hi, p->lp.kind == ADERSTP_PDE_ELASTIC, "corrector_step");
  if (rc != ADERSTP_OK) return rc;
  if (!qavg || !face_q || !face_f)
    return fail(ADERSTP_ERR_INVALID_ARG, "corrector_step: one predictor output per element required");
  if (p->lp.kind != ADERSTP_PDE_ELASTIC && !(max_wavespeed >= 0.0))
    return fail(ADERSTP_ERR_INVALID_ARG, "corrector_step: max_wavespeed required for table PDEs");
  const double inv_h = mesh->elements_per_dim / mesh->domain_len;
  aderstp::CorrArgs a{u, par, qavg, face_q, face_f, mesh->elements_per_dim, inv_h,
                      max_wavespeed >= 0.0 ? max_wavespeed * inv_h : -1.0};
  a.z0 = slab->z0;
  a.nz = slab->nz;
  a.lo = halo_of(lo);
  a.hi = halo_of(hi);
  cudaError_t e = corrector_launch(p, p->lp, a, dt, t, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "correct_slab launch");
  return ADERSTP_OK;
}

int aderstp_run_simulation_slab(const aderstp_plan* p, const aderstp_mesh* mesh, const aderstp_slab* slab,
                                double* u, const double* par, double* face_q, double* face_f,
                                const aderstp_halo* lo, const aderstp_halo* hi, double cfl, double t_end,
                                double max_wavespeed, aderstp_rank_sync_fn sync, void* ctx, int64_t* steps,
                                double* t_final, void* stream) {
  if (steps) *steps = 0;
  if (t_final) *t_final = 0.0;
  int rc = validate_mesh(p, mesh, u, par, "run_simulation");
  const bool elastic = p && p->lp.kind == ADERSTP_PDE_ELASTIC;
  if (rc == ADERSTP_OK) rc = validate_slab(mesh, slab, lo, hi, elastic, "run_simulation");
  if (rc != ADERSTP_OK) return rc;
  if (!face_q || !face_f) return fail(ADERSTP_ERR_INVALID_ARG, "run_simulation: null face buffers");
  if (!(cfl > 0.0) || !(t_end >= 0.0)) return fail(ADERSTP_ERR_INVALID_ARG, "run_simulation: bad cfl or t_end");
  if (!(max_wavespeed > 0.0))
    return fail(ADERSTP_ERR_INVALID_ARG, "run_simulation: the global max_wavespeed must be positive");
  return run_loop(p, mesh, slab->z0, slab->nz, u, par, face_q, face_f, halo_of(lo), halo_of(hi), cfl, t_end,
                  max_wavespeed, elastic, sync, ctx, steps, t_final, static_cast<cudaStream_t>(stream));
}

int aderstp_device_alloc(size_t bytes, void** ptr) {
  if (!ptr) return fail(ADERSTP_ERR_INVALID_ARG, "device_alloc: null pointer");
  cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 1);
  return e == cudaSuccess ? ADERSTP_OK : cuda_fail(e, "device_alloc");
}
int aderstp_device_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? ADERSTP_OK : cuda_fail(e, "device_free");
}
int aderstp_ipc_handle(const void* ptr, void* handle64) {
  if (!ptr || !handle64) return fail(ADERSTP_ERR_INVALID_ARG, "ipc_handle: null argument");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(ptr));
  if (e != cudaSuccess) return cuda_fail(e, "ipc_handle");
  static_assert(sizeof h == 64, "CUDA IPC handles are 64 bytes");
  std::memcpy(handle64, &h, sizeof h);
  return ADERSTP_OK;
}
int aderstp_ipc_open(const void* handle64, void** ptr) {
  if (!handle64 || !ptr) return fail(ADERSTP_ERR_INVALID_ARG, "ipc_open: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? ADERSTP_OK : cuda_fail(e, "ipc_open");
}
int aderstp_ipc_close(void* ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? ADERSTP_OK : cuda_fail(e, "ipc_close");
}

int aderstp_run_simulation(const aderstp_plan* p, const aderstp_mesh* mesh, double* u, const double* par,
                           double cfl, double t_end, double max_wavespeed, int64_t* steps, double* t_final,
                           void* stream) {
  if (steps) *steps = 0;
  if (t_final) *t_final = 0.0;
  int rc = validate_mesh(p, mesh, u, par, "run_simulation");
  if (rc != ADERSTP_OK) return rc;
  if (!(cfl > 0.0) || !(t_end >= 0.0)) return fail(ADERSTP_ERR_INVALID_ARG, "run_simulation: bad cfl or t_end");
  const bool elastic = p->lp.kind == ADERSTP_PDE_ELASTIC;
  if (!elastic && !(max_wavespeed >= 0.0))
    return fail(ADERSTP_ERR_INVALID_ARG, "run_simulation: max_wavespeed required for table PDEs");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int e = mesh->elements_per_dim;
  const long long E = (long long)e * e * e;
  const size_t face = 6 * (size_t)p->lp.n * p->lp.n * p->lp.m;
  double* faces = nullptr;
  unsigned long long* d_cp = nullptr;
  double smax = max_wavespeed;
  // scratch from the plan's pool (kept between calls: no re-mapping of the face buffers per call)
  cudaError_t err = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&faces), sizeof(double) * 2 * face * (E > 0 ? E : 1),
                                            p->pool, st);
  if (err == cudaSuccess && elastic && !(smax >= 0.0)) {  // the global max cp (stable_dt)
    unsigned long long bits = 0;
    err = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&d_cp), sizeof bits, p->pool, st);
    if (err == cudaSuccess) err = aderstp::launch_max_cp(par, p->lp.par_kind, E, d_cp, st);
    if (err == cudaSuccess) err = cudaMemcpyAsync(&bits, d_cp, sizeof bits, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    std::memcpy(&smax, &bits, sizeof smax);
  }
  if (err == cudaSuccess) {
    const aderstp::HaloRef none;
    rc = run_loop(p, mesh, 0, e, u, par, faces, faces + face * E, none, none, cfl, t_end, smax,
                  elastic && max_wavespeed < 0.0, nullptr, nullptr, steps, t_final, st);
  } else {
    rc = cuda_fail(err, "run_simulation setup");
  }
  if (faces) cudaFreeAsync(faces, st);
  if (d_cp) cudaFreeAsync(d_cp, st);
  cudaStreamSynchronize(st);  // the call is synchronous, like the reference's
  return rc;
}
