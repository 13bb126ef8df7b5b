// aderstp.hpp -- header-only C++ adapter over the C ABI (include/aderstp.h).
//
// Mirrors the reference's predictor entry point for a caller that holds elements in the
// reference's own containers (ElementTensor AoS, m_pad = 16; PredictorOutput), so the drop-in
// is a one-line change at the call site:
//
//   reference (per element, CPU)                     this adapter (per batch, B200)
//   ader::predict(v, q, pde, dt, ops, arena, out, t0) aderstp::Predictor::predict(...)
//   ader::extrapolate_faces(out, ops)                 (fused into the same call)
//   (proj/include/ader/predictor.hpp:118-125)
//
// Any constant-coefficient LinearPde (proj/include/ader/pde.hpp:21-46) is accepted through
// aderstp::probe_linear_pde: F_d and B_d are linear, so evaluating the user's flux/ncp on the
// unit vectors yields the matrices A_d, B_d exactly (the reference's own probing idiom,
// proj/tests/test_pde.cpp:14-24).  The elastic system with per-element material uses the
// dedicated elastic kernels instead (aderstp::elastic_config).
#ifndef ADERSTP_HPP
#define ADERSTP_HPP

#include <algorithm>
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "aderstp.h"

namespace aderstp {

class Error : public std::invalid_argument {
 public:
  Error(int code, const std::string& msg) : std::invalid_argument(msg), code(code) {}
  int code;
};

inline void check(int rc) {
  if (rc != ADERSTP_OK) throw Error(rc, std::string("aderstp: ") + aderstp_last_error());
}

// Probed matrices of a linear PDE: a[d][s*m + r] = F_d(e_r)_s, b[d][s*m + r] = (B_d e_r)_s.
struct LinearMatrices {
  int m = 0;
  std::array<std::vector<double>, 3> a, b;
  // one Gaussian point source (PointSourceSpec, proj/include/ader/pde.hpp:47-56): position[3],
  // component, amplitude, center, width -- a user LinearPde with source_count() == 1 whose
  // source_derivative() is the reference's Gaussian; set with add_point_source()
  bool has_source = false;
  std::array<double, 7> source{};
  double max_wavespeed = 0.0;  // the user's max_wavespeed(), for stable_dt / the corrector
};

inline void add_point_source(LinearMatrices& lm, const std::array<double, 3>& position, int component,
                             double amplitude, double center, double width) {
  lm.has_source = true;
  lm.source = {position[0], position[1], position[2], static_cast<double>(component), amplitude, center, width};
}

// Works with any type exposing the reference's LinearPde hooks: quantities(),
// flux(const double*, int, double*) and ncp(const double*, int, double*).
template <class Pde>
LinearMatrices probe_linear_pde(const Pde& pde) {
  LinearMatrices lm;
  lm.m = pde.quantities();
  const int m = lm.m;
  std::vector<double> e(m, 0.0), f(m, 0.0);
  for (int d = 0; d < 3; ++d) {
    lm.a[d].assign(static_cast<size_t>(m) * m, 0.0);
    lm.b[d].assign(static_cast<size_t>(m) * m, 0.0);
    for (int r = 0; r < m; ++r) {
      e[r] = 1.0;
      pde.flux(e.data(), d, f.data());
      for (int s = 0; s < m; ++s) lm.a[d][static_cast<size_t>(s) * m + r] = f[s];
      pde.ncp(e.data(), d, f.data());
      for (int s = 0; s < m; ++s) lm.b[d][static_cast<size_t>(s) * m + r] = f[s];
      e[r] = 0.0;
    }
  }
  lm.max_wavespeed = pde.max_wavespeed();
  return lm;
}

inline aderstp_config base_config(int order, int quantities, int layout, int q_stride, int out_stride) {
  aderstp_config c{};
  c.order = order;
  c.quantities = quantities;
  c.layout = layout;
  c.q_stride = q_stride;
  c.out_stride = out_stride;
  c.check_inputs = 1;
  return c;
}

// Elastic system with per-element (lambda, mu, rho) or (rho, cp, cs).
inline aderstp_config elastic_config(int order, int layout = ADERSTP_LAYOUT_AOS, int q_stride = 16,
                                     int out_stride = 16, int par_kind = ADERSTP_PAR_LAMBDA_MU_RHO) {
  aderstp_config c = base_config(order, 9, layout, q_stride, out_stride);
  c.pde_kind = ADERSTP_PDE_ELASTIC;
  c.par_kind = par_kind;
  return c;
}

// RAII plan.  For ADERSTP_PDE_LINEAR the probed matrices must outlive only the constructor.
class Predictor {
 public:
  explicit Predictor(const aderstp_config& cfg) { check(aderstp_plan_create(&cfg, &plan_)); }
  Predictor(int order, const LinearMatrices& lm, int layout = ADERSTP_LAYOUT_AOS, int q_stride = 0,
            int out_stride = 0) {
    aderstp_config c = base_config(order, lm.m, layout, q_stride ? q_stride : lm.m,
                                   out_stride ? out_stride : lm.m);
    c.pde_kind = ADERSTP_PDE_LINEAR;
    for (int d = 0; d < 3; ++d) {
      c.linear[d] = lm.a[d].data();
      c.linear[3 + d] = lm.b[d].data();
    }
    if (lm.has_source) {
      for (int i = 0; i < 7; ++i) c.pde_args[i] = lm.source[i];
      c.pde_args[7] = 1.0;
    }
    check(aderstp_plan_create(&c, &plan_));
  }
  Predictor(const Predictor&) = delete;
  Predictor& operator=(const Predictor&) = delete;
  ~Predictor() { aderstp_plan_destroy(plan_); }

  // Device buffers, asynchronous on `stream` (see aderstp.h for the layouts).
  void predict_device(int64_t n_elem, const double* q, const double* par, double dt, double t_start,
                      double* qavg, double* favg, double* face_q, double* face_f, void* stream = nullptr) const {
    check(aderstp_predict_batch(plan_, n_elem, q, par, dt, t_start, qavg, favg, face_q, face_f, stream));
  }
  // Host buffers, synchronous; throws like the reference's validate_stp on bad input.
  void predict(int64_t n_elem, const double* q, const double* par, double dt, double t_start, double* qavg,
               double* favg, double* face_q, double* face_f) {
    check(aderstp_predict_batch_host(plan_, n_elem, q, par, dt, t_start, qavg, favg, face_q, face_f));
  }
  void status(void* stream = nullptr) { check(aderstp_plan_status(plan_, stream)); }

  // ader::corrector_step(mesh, outs, pde, ops, dt, t) (proj/src/solver.cpp:257-311) on a periodic
  // e^3 mesh, device buffers.
  void correct_device(const aderstp_mesh& mesh, double* u, const double* par, const double* qavg,
                      const double* face_q, const double* face_f, double max_wavespeed, double dt, double t,
                      void* stream = nullptr) const {
    check(aderstp_correct_batch(plan_, &mesh, u, par, qavg, face_q, face_f, max_wavespeed, dt, t, stream));
  }
  // ader::run_simulation (proj/src/solver.cpp:313-359); returns the reference's RunResult fields.
  struct RunResult {
    int64_t steps = 0;
    double t_final = 0.0;
    bool stable = true;
  };
  RunResult run_simulation_device(const aderstp_mesh& mesh, double* u, const double* par, double cfl,
                                  double t_end, double max_wavespeed, void* stream = nullptr) const {
    RunResult r;
    const int rc = aderstp_run_simulation(plan_, &mesh, u, par, cfl, t_end, max_wavespeed, &r.steps,
                                          &r.t_final, stream);
    if (rc == ADERSTP_ERR_NONFINITE) r.stable = false;
    else check(rc);
    return r;
  }
  aderstp_plan* handle() const { return plan_; }

 private:
  aderstp_plan* plan_ = nullptr;
};

// Drop-in batch call over the reference's own containers: `cells` is a sequence of ElementTensor-
// like objects (data() / size(), the AoS m_pad layout of the plan) and `outs` of PredictorOutput-
// like objects (qavg, favg[3] tensors and face_q[6], face_f[6] vectors,
// proj/include/ader/predictor.hpp:22-29).  One call replaces the per-element
// predict(...) + extrapolate_faces(...) loop of run_simulation (proj/src/solver.cpp:334-345);
// par: per-element material (elastic) or nullptr.
template <class Cells, class Outs>
void predict_elements(Predictor& gpu, const Cells& cells, const double* par, double dt, double t_start, Outs& outs) {
  const size_t E = cells.size();
  if (E == 0) return;
  if (outs.size() != E) throw Error(ADERSTP_ERR_INVALID_ARG, "aderstp: one PredictorOutput per element required");
  const size_t vol = cells[0].size(), face = outs[0].face_q[0].size();
  std::vector<double> q(E * vol), qavg(E * vol), favg(3 * E * vol), fq(6 * E * face), ff(6 * E * face);
  for (size_t e = 0; e < E; ++e) std::copy(cells[e].data(), cells[e].data() + vol, q.data() + e * vol);
  gpu.predict(static_cast<int64_t>(E), q.data(), par, dt, t_start, qavg.data(), favg.data(), fq.data(), ff.data());
  for (size_t e = 0; e < E; ++e) {
    std::copy(qavg.data() + e * vol, qavg.data() + (e + 1) * vol, outs[e].qavg.data());
    for (int d = 0; d < 3; ++d)
      std::copy(favg.data() + (3 * e + d) * vol, favg.data() + (3 * e + d + 1) * vol, outs[e].favg[d].data());
    for (int f = 0; f < 6; ++f) {
      std::copy(fq.data() + (6 * e + f) * face, fq.data() + (6 * e + f + 1) * face, outs[e].face_q[f].data());
      std::copy(ff.data() + (6 * e + f) * face, ff.data() + (6 * e + f + 1) * face, outs[e].face_f[f].data());
    }
  }
}

}  // namespace aderstp

#endif  // ADERSTP_HPP
