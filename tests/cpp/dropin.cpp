// TEST INFRASTRUCTURE: drop-in check of the C++ adapter (include/aderstp.hpp) against the
// UNMODIFIED reference, driven exactly like a reference caller would drive it.  Built by
// oracle/Makefile (target `ref`, needs /root/reference) into oracle/_ref/dropin.
//
// For each case it fills reference ElementTensors (AoS, m_pad = 16, proj/include/ader/layout.hpp),
// runs ader::predict(splitck) + ader::extrapolate_faces element by element on the CPU, runs the
// same batch through aderstp::Predictor on the GPU (host buffers in the reference's own AoS
// layout, PredictorOutput face arrays) and compares with the reference's rel_diff metric.
// Exit code 0 iff every case is within 1e-12.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

#include "../../include/aderstp.hpp"
#include "ader/basis.hpp"
#include "ader/layout.hpp"
#include "ader/pde.hpp"
#include "ader/predictor.hpp"
#include "ader/util.hpp"

namespace {

double rel_diff(const double* a, const double* b, size_t len) {
  double d = 0.0, s = 0.0;
  for (size_t i = 0; i < len; ++i) {
    d = std::max(d, std::abs(a[i] - b[i]));
    s = std::max(s, std::abs(a[i]));
  }
  return d / std::max(s, 1e-300);
}

// Runs E elements through the reference and through the GPU adapter; returns the worst deviation.
template <class MakePde>
double run_case(const char* name, int n, int m, int E, aderstp::Predictor& gpu, MakePde make_pde,
                const std::vector<double>& par, double dt, double t0) {
  const ader::LayoutSpec sp = ader::LayoutSpec::aos(n, m, 8);
  const ader::BasisOperators ops = ader::make_basis(n);
  ader::SolverConfig cfg;
  cfg.order = n;
  cfg.quantities = m;
  ader::ScratchArena arena(ader::Variant::splitck, cfg);
  const size_t vol = sp.size(), face = static_cast<size_t>(n) * n * m;
  std::vector<double> q(E * vol), qavg(E * vol), favg(3 * E * vol), fq(6 * E * face), ff(6 * E * face);
  ader::SplitMix64 rng(1234 + n + m);
  std::vector<ader::PredictorOutput> ref;
  for (int e = 0; e < E; ++e) {
    ader::ElementTensor t(sp);
    for (int k3 = 0; k3 < n; ++k3)
      for (int k2 = 0; k2 < n; ++k2)
        for (int k1 = 0; k1 < n; ++k1)
          for (int s = 0; s < m; ++s) t.at(k3, k2, k1, s) = rng.next_symmetric();
    std::memcpy(q.data() + e * vol, t.data(), vol * sizeof(double));
    auto pde = make_pde(e);
    ref.emplace_back(sp);
    ader::predict(ader::Variant::splitck, t, *pde, dt, ops, arena, ref.back(), t0);
    ader::extrapolate_faces(ref.back(), ops);
  }
  gpu.predict(E, q.data(), par.empty() ? nullptr : par.data(), dt, t0, qavg.data(), favg.data(), fq.data(), ff.data());
  double worst = 0.0;
  for (int e = 0; e < E; ++e) {
    worst = std::max(worst, rel_diff(ref[e].qavg.data(), qavg.data() + e * vol, vol));
    for (int d = 0; d < 3; ++d)
      worst = std::max(worst, rel_diff(ref[e].favg[d].data(), favg.data() + (3 * e + d) * vol, vol));
    for (int f = 0; f < 6; ++f) {
      worst = std::max(worst, rel_diff(ref[e].face_q[f].data(), fq.data() + (6 * e + f) * face, face));
      worst = std::max(worst, rel_diff(ref[e].face_f[f].data(), ff.data() + (6 * e + f) * face, face));
    }
    // padding lanes of the AoS outputs stay exactly zero (proj/tests/test_predictor.cpp:157-170)
    for (size_t node = 0; node < vol / sp.m_pad; ++node)
      for (int s = m; s < sp.m_pad; ++s)
        if (qavg[e * vol + node * sp.m_pad + s] != 0.0) worst = 1.0;
  }
  std::printf("%-28s n=%d m=%d E=%d worst rel_diff %.3e\n", name, n, m, E, worst);
  return worst;
}

}  // namespace

int main() {
  double worst = 0.0;
  try {
    // elastic, per-element material, reference AoS layout (m_pad = 16) in and out
    for (int n : {3, 4, 6, 8, 10}) {
      const int E = 37;
      std::vector<double> par(3 * E);
      for (int e = 0; e < E; ++e) {
        par[3 * e] = 2.0 + 0.01 * e;      // lambda
        par[3 * e + 1] = 1.0 + 0.005 * e;  // mu
        par[3 * e + 2] = 1.5 - 0.01 * e;   // rho
      }
      aderstp::Predictor gpu(aderstp::elastic_config(n));
      const double dt = 0.4 / (3.0 * 3.0 * (2.0 * n - 1.0));
      worst = std::max(worst, run_case("elastic (per element)", n, 9, E, gpu,
                                       [&](int e) { return ader::elastic_pde(par[3 * e], par[3 * e + 1], par[3 * e + 2]); },
                                       par, dt, 0.0));
    }
    // arbitrary reference LinearPde objects through the probed-matrix path
    {
      auto pde = ader::advection_pde({1.0, 0.5, 0.25}, 3);
      aderstp::Predictor gpu(5, aderstp::probe_linear_pde(*pde), ADERSTP_LAYOUT_AOS, 8, 8);
      worst = std::max(worst, run_case("advection (probed)", 5, 3, 9, gpu,
                                       [&](int) { return ader::advection_pde({1.0, 0.5, 0.25}, 3); }, {}, 0.02, 0.0));
    }
    {
      auto pde = ader::ncp_advection_pde({1.0, 0.5, 0.25}, 2);
      aderstp::Predictor gpu(4, aderstp::probe_linear_pde(*pde), ADERSTP_LAYOUT_AOS, 8, 8);
      worst = std::max(worst, run_case("ncp-advection (probed)", 4, 2, 9, gpu,
                                       [&](int) { return ader::ncp_advection_pde({1.0, 0.5, 0.25}, 2); }, {}, 0.02, 0.0));
    }
    {
      auto pde = ader::paper_demo_pde();
      aderstp::Predictor gpu(6, aderstp::probe_linear_pde(*pde), ADERSTP_LAYOUT_AOS, 8, 8);
      worst = std::max(worst, run_case("paper demo (probed)", 6, 6, 9, gpu,
                                       [&](int) { return ader::paper_demo_pde(); }, {}, 0.01, 0.0));
    }
    // aderstp::predict_elements straight on the reference's containers (ElementTensor in,
    // PredictorOutput out), as run_simulation would call it
    {
      const int n = 8, E = 11;
      const ader::LayoutSpec sp = ader::LayoutSpec::aos(n, 9, 8);
      const ader::BasisOperators ops = ader::make_basis(n);
      ader::SolverConfig cfg;
      cfg.order = n;
      ader::ScratchArena arena(ader::Variant::splitck, cfg);
      std::vector<ader::ElementTensor> cells;
      std::vector<ader::PredictorOutput> outs, ref;
      std::vector<double> par;
      ader::SplitMix64 rng(99);
      for (int e = 0; e < E; ++e) {
        cells.emplace_back(sp);
        for (int k3 = 0; k3 < n; ++k3)
          for (int k2 = 0; k2 < n; ++k2)
            for (int k1 = 0; k1 < n; ++k1)
              for (int s = 0; s < 9; ++s) cells.back().at(k3, k2, k1, s) = rng.next_symmetric();
        par.insert(par.end(), {2.0 + 0.02 * e, 1.0, 1.2});
        outs.emplace_back(sp);
        ref.emplace_back(sp);
        auto pde = ader::elastic_pde(par[3 * e], par[3 * e + 1], par[3 * e + 2]);
        ader::predict(ader::Variant::splitck, cells.back(), *pde, 1e-3, ops, arena, ref.back(), 0.0);
        ader::extrapolate_faces(ref.back(), ops);
      }
      aderstp::Predictor gpu(aderstp::elastic_config(n));
      aderstp::predict_elements(gpu, cells, par.data(), 1e-3, 0.0, outs);
      double w = 0.0;
      for (int e = 0; e < E; ++e) {
        w = std::max(w, rel_diff(ref[e].qavg.data(), outs[e].qavg.data(), sp.size()));
        for (int d = 0; d < 3; ++d) w = std::max(w, rel_diff(ref[e].favg[d].data(), outs[e].favg[d].data(), sp.size()));
        for (int f = 0; f < 6; ++f) {
          w = std::max(w, rel_diff(ref[e].face_q[f].data(), outs[e].face_q[f].data(), outs[e].face_q[f].size()));
          w = std::max(w, rel_diff(ref[e].face_f[f].data(), outs[e].face_f[f].data(), outs[e].face_f[f].size()));
        }
      }
      std::printf("%-28s n=%d E=%d worst rel_diff %.3e\n", "predict_elements (containers)", n, E, w);
      worst = std::max(worst, w);
    }
    // the reference's validate_stp rejects non-finite input: so does the adapter
    {
      aderstp::Predictor gpu(aderstp::elastic_config(4));
      std::vector<double> q(64 * 16, 0.0), par{2.0, 1.0, 1.0}, out(64 * 16 * 4), fq(6 * 16 * 9), ff(6 * 16 * 9);
      q[3] = std::nan("");
      bool threw = false;
      try {
        gpu.predict(1, q.data(), par.data(), 0.01, 0.0, out.data(), out.data() + 64 * 16, fq.data(), ff.data());
      } catch (const aderstp::Error& e) {
        threw = e.code == ADERSTP_ERR_NONFINITE;
      }
      std::printf("%-28s %s\n", "non-finite input rejected", threw ? "yes" : "NO");
      if (!threw) worst = 1.0;
    }
  } catch (const std::exception& ex) {
    std::printf("error: %s\n", ex.what());
    return 2;
  }
  std::printf("DROPIN %s (worst %.3e, tolerance 1e-12)\n", worst <= 1e-12 ? "PASS" : "FAIL", worst);
  return worst <= 1e-12 ? 0 : 1;
}
