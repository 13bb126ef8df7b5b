// Host-side nodal basis on [0,1], derived from scratch for the plan's kernel constants.
// Same mathematical objects as the reference's make_basis (proj/src/basis.cpp:110-122):
// Gauss-Legendre nodes/weights, Lagrange derivative matrix with the negative-sum diagonal
// (basis.cpp:73-88) and the face values phi_k(0), phi_k(1) (basis.cpp:106-108).
#include <cmath>

#include "aderstp_internal.h"

namespace aderstp {

namespace {

// P_n(t) and P_n'(t) on [-1,1] (Bonnet recurrence; derivative from the standard identity).
void legendre_pair(int n, double t, double& p, double& dp) {
  double a = 1.0, b = t;  // P_0, P_1
  if (n == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  for (int k = 1; k < n; ++k) {
    const double c = ((2.0 * k + 1.0) * t * b - k * a) / (k + 1.0);
    a = b;
    b = c;
  }
  p = b;
  dp = n * (t * b - a) / (t * t - 1.0);
}

void barycentric(int n, const double* x, double* lam) {
  for (int j = 0; j < n; ++j) {
    double prod = 1.0;
    for (int i = 0; i < n; ++i)
      if (i != j) prod *= (x[j] - x[i]);
    lam[j] = 1.0 / prod;
  }
}

}  // namespace

void lagrange_values(int n, const double* nodes, double x, double* vals) {
  double lam[kMaxOrder];
  barycentric(n, nodes, lam);
  for (int j = 0; j < n; ++j) vals[j] = 0.0;
  for (int j = 0; j < n; ++j)
    if (x == nodes[j]) {
      vals[j] = 1.0;
      return;
    }
  double den = 0.0;
  for (int j = 0; j < n; ++j) den += lam[j] / (x - nodes[j]);
  for (int j = 0; j < n; ++j) vals[j] = lam[j] / (x - nodes[j]) / den;
}

int make_host_basis(int n, HostBasis* out) {
  if (n < 1 || n > kMaxOrder) return -1;
  out->n = n;
  const double pi = 3.14159265358979323846;
  // roots of P_n, largest first from the Tricomi-type initial guess, refined by Newton
  for (int i = 0; i < n; ++i) {
    double t = std::cos(pi * (4.0 * i + 3.0) / (4.0 * n + 2.0));
    double p = 0.0, dp = 1.0;
    for (int it = 0; it < 64; ++it) {
      legendre_pair(n, t, p, dp);
      const double step = p / dp;
      t -= step;
      if (std::fabs(step) < 1e-15) break;
    }
    legendre_pair(n, t, p, dp);
    // ascending order on [0,1]
    out->nodes[n - 1 - i] = 0.5 * (1.0 + t);
    out->weights[n - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp);  // = 0.5 * 2/((1-t^2)P'^2)
  }
  if (n == 1) {
    out->nodes[0] = 0.5;
    out->weights[0] = 1.0;
  }
  double lam[kMaxOrder];
  barycentric(n, out->nodes, lam);
  for (int k = 0; k < n; ++k) {
    double row = 0.0;
    for (int l = 0; l < n; ++l) {
      if (l == k) continue;
      const double v = lam[l] / (lam[k] * (out->nodes[k] - out->nodes[l]));
      out->d[k * n + l] = v;
      row += v;
    }
    out->d[k * n + k] = -row;  // rows annihilate constants exactly
  }
  lagrange_values(n, out->nodes, 0.0, out->face_left);
  lagrange_values(n, out->nodes, 1.0, out->face_right);
  return 0;
}

}  // namespace aderstp
