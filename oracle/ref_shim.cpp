// TEST INFRASTRUCTURE — C shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  Only tests/, smoke() and
// bench.py's reference/cpu_baseline legs load it; the product never links it.
//
// It drives the reference's own public API exactly the way its production caller does:
// one ScratchArena per OpenMP worker (proj/src/solver.cpp:324-345), predict(variant, ...)
// (proj/include/ader/predictor.hpp:118-120) followed by extrapolate_faces (:125), and one
// LinearPde object per element built by the reference's factories (proj/include/ader/pde.hpp:62-84).
//
// Batch layout on both sides of this shim is the canonical unpadded one:
//   q, qavg : [e][k3][k2][k1][s]          (s fastest, m quantities, no padding)
//   favg    : [e][d][k3][k2][k1][s]       (d = 0,1,2)
//   face_q/f: [e][f][a][b][s]             (f = -x,+x,-y,+y,-z,+z; (a,b) as in predictor.hpp:16-21)
#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "ader/basis.hpp"
#include "ader/layout.hpp"
#include "ader/pde.hpp"
#include "ader/predictor.hpp"
#include "ader/solver.hpp"
#include "ader/util.hpp"

namespace {

thread_local std::string g_err;

// pde_kind values (mirrored in oracle/stp_oracle.h and the product's aderstp.h)
enum : int {
  kElastic = 0,        // par[e] = (lambda, mu, rho)
  kAdvection = 1,      // args = (vx, vy, vz)
  kNcpAdvection = 2,   // args = (vx, vy, vz)
  kDemo = 3,           // paper demo, m = 6
  kElasticSource = 4,  // par[e] = (lambda, mu, rho); args = point source spec (7 doubles)
  kSourceOnly = 5,     // args = point source spec
  kMatrix = 6,         // a user LinearPde given by matrices (ref_set_matrix_pde), see MatrixPde
};

ader::PointSourceSpec source_from(const double* a) {
  ader::PointSourceSpec s;
  s.position = {a[0], a[1], a[2]};
  s.component = static_cast<int>(a[3]);
  s.amplitude = a[4];
  s.center = a[5];
  s.width = a[6];
  return s;
}

// A user LinearPde defined by its coefficient matrices (see ref_set_matrix_pde): flux and ncp
// are the matrix products, max_wavespeed the given value, and an optional Gaussian point source
// whose time derivatives and position come from the reference's own source_only_pde
// (proj/src/pde.cpp:286-308), so the source path is the unmodified reference's.
class MatrixPde final : public ader::LinearPde {
public:
  MatrixPde(int m, const double* A, const double* B, const double* src = nullptr, double smax = 1.0)
      : ader::LinearPde(m, src ? 1 : 0), a_(A, A + 3 * m * m), b_(B ? std::vector<double>(B, B + 3 * m * m)
                                                                    : std::vector<double>(3 * m * m, 0.0)),
        smax_(smax) {
    if (src) src_ = ader::source_only_pde(m, source_from(src));
  }
  void flux(const double* q, int dim, double* f) const override { apply(a_, q, dim, f); }
  void ncp(const double* grad, int dim, double* out) const override { apply(b_, grad, dim, out); }
  void source_derivative(int order, double t, int src, double* out) const override {
    if (src_) src_->source_derivative(order, t, src, out);
    else ader::LinearPde::source_derivative(order, t, src, out);
  }
  std::array<double, 3> source_position(int src) const override {
    return src_ ? src_->source_position(src) : ader::LinearPde::source_position(src);
  }
  double max_wavespeed() const override { return smax_; }

private:
  void apply(const std::vector<double>& mat, const double* x, int dim, double* y) const {
    const double* a = mat.data() + static_cast<std::size_t>(dim) * m_ * m_;
    for (int r = 0; r < m_; ++r) {
      double s = 0.0;
      for (int j = 0; j < m_; ++j) s += a[r * m_ + j] * x[j];
      y[r] = s;
    }
  }
  std::vector<double> a_, b_;
  double smax_;
  std::unique_ptr<ader::LinearPde> src_;
};

// the matrix PDE that pde kind kMatrix builds (set by ref_set_matrix_pde)
struct MatrixSpec {
  int m = 0;
  std::vector<double> a, b, src;
  double smax = 1.0;
} g_matrix;

std::unique_ptr<ader::LinearPde> make_pde(int kind, int m, const double* par, const double* args) {
  switch (kind) {
    case kElastic: return ader::elastic_pde(par[0], par[1], par[2]);
    case kAdvection: return ader::advection_pde({args[0], args[1], args[2]}, m);
    case kNcpAdvection: return ader::ncp_advection_pde({args[0], args[1], args[2]}, m);
    case kDemo: return ader::paper_demo_pde();
    case kElasticSource: return ader::elastic_pde(par[0], par[1], par[2], source_from(args));
    case kSourceOnly: return ader::source_only_pde(m, source_from(args));
    case kMatrix:
      if (g_matrix.m != m) throw std::invalid_argument("ref_shim: matrix pde not set for this m");
      return std::make_unique<MatrixPde>(m, g_matrix.a.data(), g_matrix.b.data(),
                                         g_matrix.src.empty() ? nullptr : g_matrix.src.data(), g_matrix.smax);
  }
  throw std::invalid_argument("ref_shim: unknown pde kind");
}

bool per_element_par(int kind) { return kind == kElastic || kind == kElasticSource; }


int stp_batch(int variant, int n, int m, long n_elem, const double* q, const double* par,
              const double* args, int pde_kind, std::shared_ptr<ader::LinearPde> given, double dt,
              double t_start, double* qavg, double* favg, double* face_q, double* face_f,
              int n_threads, double* seconds) {
  try {
    const ader::Variant v = static_cast<ader::Variant>(variant);
    ader::SolverConfig cfg;
    cfg.order = n;
    cfg.quantities = m;
    cfg.vec_width = 8;
    const ader::BasisOperators ops = ader::make_basis(n);
    const ader::LayoutSpec sp = ader::LayoutSpec::aos(n, m, cfg.vec_width);
    const long nn = static_cast<long>(n) * n * n;
    const long vol = nn * m, face = static_cast<long>(n) * n * m;
    if (n_threads <= 0) n_threads = omp_get_max_threads();

    std::shared_ptr<ader::LinearPde> shared = given;
    if (!shared && !per_element_par(pde_kind)) shared = make_pde(pde_kind, m, nullptr, args);
    if (shared && shared->quantities() != m) throw std::invalid_argument("ref_shim: m mismatch");

    std::vector<std::string> errors(n_threads);
    const auto tic = std::chrono::steady_clock::now();
#pragma omp parallel num_threads(n_threads)
    {
      const int tid = omp_get_thread_num();
      try {
        ader::ScratchArena arena(v, cfg);
        ader::ElementTensor qe(sp);
        ader::PredictorOutput out(sp);
#pragma omp for schedule(static)
        for (long e = 0; e < n_elem; ++e) {
          std::unique_ptr<ader::LinearPde> own;
          const ader::LinearPde* pde = shared.get();
          if (!pde) {
            own = make_pde(pde_kind, m, par + 3 * e, args);
            pde = own.get();
          }
          const double* qs = q + e * vol;
          for (long k = 0; k < nn; ++k)
            std::memcpy(qe.data() + k * sp.m_pad, qs + k * m, sizeof(double) * m);
          ader::predict(v, qe, *pde, dt, ops, arena, out, t_start);
          ader::extrapolate_faces(out, ops);
          double* qa = qavg + e * vol;
          for (long k = 0; k < nn; ++k)
            std::memcpy(qa + k * m, out.qavg.data() + k * sp.m_pad, sizeof(double) * m);
          if (favg) {
            for (int d = 0; d < 3; ++d) {
              double* fa = favg + (e * 3 + d) * vol;
              for (long k = 0; k < nn; ++k)
                std::memcpy(fa + k * m, out.favg[d].data() + k * sp.m_pad, sizeof(double) * m);
            }
          }
          for (int f = 0; f < 6; ++f) {
            if (face_q) std::memcpy(face_q + (e * 6 + f) * face, out.face_q[f].data(), sizeof(double) * face);
            if (face_f) std::memcpy(face_f + (e * 6 + f) * face, out.face_f[f].data(), sizeof(double) * face);
          }
        }
      } catch (const std::exception& ex) {
        errors[tid] = ex.what();
      }
    }
    const auto toc = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(toc - tic).count();
    for (const std::string& s : errors)
      if (!s.empty()) {
        g_err = s;
        return -1;
      }
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Batched reference predictor. variant: 0 generic, 1 log, 2 splitck, 3 splitck_aosoa
// (proj/include/ader/config.hpp:11).  Returns 0 on success, -1 if the reference threw
// (message in ref_last_error).  *seconds receives the wall time of the predict loop alone.
int ref_stp_batch(int variant, int n, int m, long n_elem, const double* q, const double* par,
                  const double* args, int pde_kind, double dt, double t_start, double* qavg,
                  double* favg, double* face_q, double* face_f, int n_threads, double* seconds) {
  return stp_batch(variant, n, m, n_elem, q, par, args, pde_kind, nullptr, dt, t_start, qavg, favg,
                   face_q, face_f, n_threads, seconds);
}

// The matrix PDE of pde kind 6 (kMatrix) for every entry point of this shim: A[d] (m x m,
// row-major, F_d(q) = A_d q), B[d] (ncp, B_d grad; may be null), an optional point source
// (7 doubles as in pde_args; null = none) and the max_wavespeed() the solver sees.  A user
// LinearPde subclass (proj/include/ader/pde.hpp:21-46) of the kind the reference's own tests
// probe (proj/tests/test_pde.cpp:14-24).
int ref_set_matrix_pde(int m, const double* A, const double* B, const double* src, double max_wavespeed) {
  try {
    g_matrix.m = m;
    g_matrix.a.assign(A, A + 3 * m * m);
    if (B) g_matrix.b.assign(B, B + 3 * m * m);
    else g_matrix.b.assign(3 * m * m, 0.0);
    if (src) g_matrix.src.assign(src, src + 7);
    else g_matrix.src.clear();
    g_matrix.smax = max_wavespeed;
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

int ref_stp_batch_matrix(int variant, int n, int m, long n_elem, const double* q, const double* A,
                         const double* B, double dt, double* qavg, double* favg, double* face_q,
                         double* face_f, int n_threads, double* seconds) {
  if (ref_set_matrix_pde(m, A, B, nullptr, 1.0) != 0) return -1;
  return stp_batch(variant, n, m, n_elem, q, nullptr, nullptr, kMatrix, nullptr, dt, 0.0, qavg, favg,
                   face_q, face_f, n_threads, seconds);
}

// Basis operators of the reference (proj/src/basis.cpp:110-122).
int ref_make_basis(int n, double* nodes, double* weights, double* d, double* face_left,
                   double* face_right) {
  try {
    const ader::BasisOperators ops = ader::make_basis(n);
    std::memcpy(nodes, ops.nodes.data(), sizeof(double) * n);
    std::memcpy(weights, ops.weights.data(), sizeof(double) * n);
    std::memcpy(d, ops.d.data(), sizeof(double) * n * n);
    std::memcpy(face_left, ops.face_left.data(), sizeof(double) * n);
    std::memcpy(face_right, ops.face_right.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// First `count` outputs of the reference SplitMix64 (proj/include/ader/util.hpp:72-90).
void ref_splitmix64(std::uint64_t seed, long count, std::uint64_t* out) {
  ader::SplitMix64 rng(seed);
  for (long i = 0; i < count; ++i) out[i] = rng.next();
}

// Reference flop_count / scratch_bytes (proj/src/predictor_common.cpp:70-91).
std::uint64_t ref_flop_count(int variant, int n, int m) {
  ader::SolverConfig cfg;
  cfg.order = n;
  cfg.quantities = m;
  return ader::flop_count(static_cast<ader::Variant>(variant), cfg);
}

// Dense volume operator of the reference (proj/src/predictor_common.cpp:343-360) for a
// shared (non per-element) PDE or the elastic PDE with par = (lambda, mu, rho).
int ref_volume_operator(int n, int m, int pde_kind, const double* par, const double* args,
                        double* out) {
  try {
    ader::SolverConfig cfg;
    cfg.order = n;
    cfg.quantities = m;
    auto pde = make_pde(pde_kind, m, par, args);
    const ader::BasisOperators ops = ader::make_basis(n);
    const std::vector<double> v = ader::materialize_volume_operator(*pde, ops, cfg);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// ---- corrector and time loop (proj/src/solver.cpp), mesh state canonical [c][k3][k2][k1][s] ----

namespace {

void load_mesh(ader::Mesh& mesh, const double* u) {
  const ader::LayoutSpec& sp = mesh.spec;
  const long nn = static_cast<long>(sp.n) * sp.n * sp.n;
  for (std::size_t c = 0; c < mesh.cells.size(); ++c)
    for (long k = 0; k < nn; ++k)
      std::memcpy(mesh.cells[c].data() + k * sp.m_pad, u + (c * nn + k) * sp.m, sizeof(double) * sp.m);
}

void store_mesh(const ader::Mesh& mesh, double* u) {
  const ader::LayoutSpec& sp = mesh.spec;
  const long nn = static_cast<long>(sp.n) * sp.n * sp.n;
  for (std::size_t c = 0; c < mesh.cells.size(); ++c)
    for (long k = 0; k < nn; ++k)
      std::memcpy(u + (c * nn + k) * sp.m, mesh.cells[c].data() + k * sp.m_pad, sizeof(double) * sp.m);
}

}  // namespace

// ader::corrector_step on an e^3 periodic mesh (one shared PDE: par = (lambda, mu, rho) for the
// elastic kind, args otherwise) from given predictor outputs (qavg canonical, faces
// [c][f][a][b][s]).  u is updated in place.  Returns 0, -1 on a reference exception, -2 when
// the reference reports a non-finite update.
int ref_corrector_step(int n, int m, int e, double domain_len, int pde_kind, const double* par,
                       const double* args, double dt, double t, double* u, const double* qavg,
                       const double* face_q, const double* face_f, int workers) {
  try {
    ader::SolverConfig cfg;
    cfg.order = n;
    cfg.quantities = m;
    cfg.vec_width = 8;
    ader::Mesh mesh(e, cfg, domain_len);
    const ader::BasisOperators ops = ader::make_basis(n);
    auto pde = make_pde(pde_kind, m, par, args);
    load_mesh(mesh, u);
    const ader::LayoutSpec& sp = mesh.spec;
    const long nn = static_cast<long>(n) * n * n, face = static_cast<long>(n) * n * m;
    std::vector<ader::PredictorOutput> outs;
    outs.reserve(mesh.cells.size());
    for (std::size_t c = 0; c < mesh.cells.size(); ++c) {
      outs.emplace_back(sp);
      for (long k = 0; k < nn; ++k)
        std::memcpy(outs[c].qavg.data() + k * sp.m_pad, qavg + (c * nn + k) * m, sizeof(double) * m);
      for (int f = 0; f < 6; ++f) {
        std::memcpy(outs[c].face_q[f].data(), face_q + (c * 6 + f) * face, sizeof(double) * face);
        std::memcpy(outs[c].face_f[f].data(), face_f + (c * 6 + f) * face, sizeof(double) * face);
      }
    }
    try {
      ader::corrector_step(mesh, outs, *pde, ops, dt, t, workers > 0 ? workers : 1);
    } catch (const std::runtime_error& ex) {
      g_err = ex.what();
      store_mesh(mesh, u);
      return -2;
    }
    store_mesh(mesh, u);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// ader::run_simulation (splitck unless variant says otherwise) on an e^3 periodic mesh with
// one shared PDE; u (canonical) in/out.  stable / steps / t_final mirror RunResult.
int ref_run_simulation(int n, int m, int e, double domain_len, int pde_kind, const double* par,
                       const double* args, double cfl, double t_end, int variant, double* u,
                       int workers, int* stable, int* steps, double* t_final) {
  try {
    ader::SolverConfig cfg;
    cfg.order = n;
    cfg.quantities = m;
    cfg.vec_width = 8;
    cfg.cfl = cfl;
    ader::Mesh mesh(e, cfg, domain_len);
    auto pde = make_pde(pde_kind, m, par, args);
    load_mesh(mesh, u);
    const ader::RunResult r = ader::run_simulation(*pde, cfg, mesh, t_end, static_cast<ader::Variant>(variant),
                                                   nullptr, workers > 0 ? workers : 1);
    store_mesh(mesh, u);
    if (stable) *stable = r.stable ? 1 : 0;
    if (steps) *steps = r.steps;
    if (t_final) *t_final = r.t_final;
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// PDE max_wavespeed of the reference factories (include/ader/pde.hpp:38)
double ref_max_wavespeed(int pde_kind, int m, const double* par, const double* args) {
  try {
    return make_pde(pde_kind, m, par, args)->max_wavespeed();
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1.0;
  }
}

}  // extern "C"
