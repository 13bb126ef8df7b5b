/* TEST INFRASTRUCTURE ONLY — see stp_oracle.h.  Plain-C restatement of the reference's
 * SplitCK space-time predictor; each function cites the reference file:line it follows. */
#include "stp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAX_Q 64
#define ORC_MAX_SRC 8
#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------ basis ---- */

/* Legendre P_n(x), P_n'(x) by the three-term recurrence (proj/src/basis.cpp:12-22). */
static void legendre_eval(int n, double x, double* p, double* dp) {
  double pm1 = 1.0, pc = x;
  if (n == 0) {
    *p = 1.0;
    *dp = 0.0;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    const double pn = ((2 * k - 1) * x * pc - (k - 1) * pm1) / k;
    pm1 = pc;
    pc = pn;
  }
  *p = pc;
  *dp = n * (x * pc - pm1) / (x * x - 1.0);
}

/* Gauss-Legendre on [0,1]: Newton from a cosine guess, |dx| < 1e-15 (basis.cpp:26-53). */
static void gauss_legendre01(int n, double* nodes, double* weights) {
  for (int i = 0; i < n; ++i) {
    double x = cos(ORC_PI * (i + 0.75) / (n + 0.5));
    double p, dp;
    for (int it = 0; it < 100; ++it) {
      legendre_eval(n, x, &p, &dp);
      const double dx = p / dp;
      x -= dx;
      if (fabs(dx) < 1e-15) break;
    }
    legendre_eval(n, x, &p, &dp);
    nodes[n - 1 - i] = 0.5 * (x + 1.0);
    weights[n - 1 - i] = 0.5 * (2.0 / ((1.0 - x * x) * dp * dp));
  }
  if (n == 1) {
    nodes[0] = 0.5;
    weights[0] = 1.0;
  }
}

static void bary_weights(int n, const double* x, double* lam) {
  for (int j = 0; j < n; ++j) {
    lam[j] = 1.0;
    for (int i = 0; i < n; ++i)
      if (i != j) lam[j] /= x[j] - x[i];
  }
}

/* phi_k(x) of the nodal Lagrange basis, barycentric, exact at nodes (basis.cpp:90-104). */
void orc_lagrange_values_at(int n, const double* nodes, double x, double* vals) {
  double lam[ORC_MAX_ORDER];
  bary_weights(n, nodes, lam);
  for (int j = 0; j < n; ++j) vals[j] = 0.0;
  for (int j = 0; j < n; ++j)
    if (x == nodes[j]) {
      vals[j] = 1.0;
      return;
    }
  double den = 0.0;
  for (int j = 0; j < n; ++j) den += lam[j] / (x - nodes[j]);
  for (int j = 0; j < n; ++j) vals[j] = (lam[j] / (x - nodes[j])) / den;
}

/* d[k*n+l] = phi_l'(x_k), negative-sum diagonal (basis.cpp:73-88); faces = phi(0), phi(1). */
int orc_make_basis(int n, double* nodes, double* weights, double* d, double* face_left,
                   double* face_right) {
  if (n < 1 || n > ORC_MAX_ORDER) return -1;
  double lam[ORC_MAX_ORDER];
  gauss_legendre01(n, nodes, weights);
  bary_weights(n, nodes, lam);
  for (int k = 0; k < n; ++k) {
    double diag = 0.0;
    for (int l = 0; l < n; ++l) {
      if (l == k) continue;
      d[k * n + l] = (lam[l] / lam[k]) / (nodes[k] - nodes[l]);
      diag -= d[k * n + l];
    }
    d[k * n + k] = diag;
  }
  orc_lagrange_values_at(n, nodes, 0.0, face_left);
  orc_lagrange_values_at(n, nodes, 1.0, face_right);
  return 0;
}

/* ------------------------------------------------------------ SplitMix64 ---- */

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* state advances by the golden gamma before mixing (util.hpp:77-82), so output k is
 * mix(seed + (k+1) * gamma): random access for per-element streams. */
uint64_t orc_splitmix64_at(uint64_t seed, uint64_t k) {
  return mix64(seed + (k + 1) * 0x9e3779b97f4a7c15ull);
}

double orc_u01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
double orc_symmetric(uint64_t x) { return 2.0 * orc_u01(x) - 1.0; } /* util.hpp:84-86 */

static double uab(uint64_t x, double a, double b) { return a + (b - a) * orc_u01(x); }

/* --------------------------------------------------------- input generator -- */

void orc_generate(int dist, uint64_t seed, int n, long e0, long count, int grid, double* q,
                  double* par_rcc) {
  const long nn = (long)n * n * n, vol = nn * 9;
  double nodes[ORC_MAX_ORDER], w[ORC_MAX_ORDER], d[ORC_MAX_ORDER * ORC_MAX_ORDER];
  double fl[ORC_MAX_ORDER], fr[ORC_MAX_ORDER];
  orc_make_basis(n, nodes, w, d, fl, fr);
  /* wave table for dist 2: 9 quantities x 3 waves x (a, kx, ky, kz, phase) */
  double wa[9][3], wk[9][3][3], wp[9][3];
  if (dist == 2) {
    uint64_t g = 0;
    for (int s = 0; s < 9; ++s)
      for (int j = 0; j < 3; ++j) {
        wa[s][j] = uab(orc_splitmix64_at(seed, g++), 0.5, 1.0);
        for (int c = 0; c < 3; ++c) wk[s][j][c] = (double)((int)(orc_splitmix64_at(seed, g++) % 7) - 3);
        wp[s][j] = 2.0 * ORC_PI * orc_u01(orc_splitmix64_at(seed, g++));
      }
  }
  for (long le = 0; le < count; ++le) {
    const long e = e0 + le;
    double* qe = q ? q + le * vol : NULL;
    uint64_t mat_base;
    if (dist == 0) {
      const uint64_t base = (uint64_t)e * (uint64_t)(vol + 3);
      if (qe)
        for (long i = 0; i < vol; ++i) qe[i] = orc_symmetric(orc_splitmix64_at(seed, base + i));
      mat_base = base + vol;
    } else if (dist == 1) {
      const uint64_t base = (uint64_t)e * (uint64_t)(2 * vol + 3);
      if (qe)
        for (long i = 0; i < vol; ++i) {
          const double u1 = ((double)(orc_splitmix64_at(seed, base + 2 * i) >> 11) + 1.0) * 0x1.0p-53;
          const double u2 = orc_u01(orc_splitmix64_at(seed, base + 2 * i + 1));
          qe[i] = sqrt(-2.0 * log(u1)) * cos(2.0 * ORC_PI * u2);
        }
      mat_base = base + 2 * vol;
    } else {
      const long ex = e % grid, ey = (e / grid) % grid, ez = e / ((long)grid * grid);
      if (qe)
        for (int k3 = 0; k3 < n; ++k3)
          for (int k2 = 0; k2 < n; ++k2)
            for (int k1 = 0; k1 < n; ++k1) {
              const double x = ex + nodes[k1], y = ey + nodes[k2], z = ez + nodes[k3];
              for (int s = 0; s < 9; ++s) {
                double v = 0.0;
                for (int j = 0; j < 3; ++j)
                  v += wa[s][j] * sin(2.0 * ORC_PI * (wk[s][j][0] * x + wk[s][j][1] * y + wk[s][j][2] * z) / grid + wp[s][j]);
                qe[(((long)k3 * n + k2) * n + k1) * 9 + s] = v;
              }
            }
      mat_base = 135 + 3 * (uint64_t)e;
    }
    if (par_rcc) {
      par_rcc[3 * le + 0] = uab(orc_splitmix64_at(seed, mat_base + 0), 2.0, 3.0);
      par_rcc[3 * le + 1] = uab(orc_splitmix64_at(seed, mat_base + 1), 4.0, 6.0);
      par_rcc[3 * le + 2] = uab(orc_splitmix64_at(seed, mat_base + 2), 2.0, 3.5);
    }
  }
}

void orc_material_lmr(long count, const double* rcc, double* lmr) {
  for (long e = 0; e < count; ++e) {
    const double rho = rcc[3 * e], cp = rcc[3 * e + 1], cs = rcc[3 * e + 2];
    const double mu = rho * cs * cs;
    lmr[3 * e + 0] = rho * cp * cp - 2.0 * mu;
    lmr[3 * e + 1] = mu;
    lmr[3 * e + 2] = rho;
  }
}

/* -------------------------------------------------------------- PDE hooks ---- */

typedef struct {
  int kind, m;
  double lam, mu, inv_rho; /* elastic (pde.cpp:171-178) */
  double v[3];             /* advection */
  int n_src;               /* point source (pde.hpp:47-56) */
  double src_pos[3], src_amp, src_center, src_width;
  int src_comp;
} orc_pde;

/* F_dim(q) (pde.cpp:61-75 advection, :88-93 ncp-advection, :128-134 demo, :180-218 elastic). */
static void pde_flux(const orc_pde* p, const double* q, int dim, double* f) {
  const int m = p->m;
  switch (p->kind) {
    case ORC_PDE_ELASTIC:
    case ORC_PDE_ELASTIC_SOURCE: {
      const double l = p->lam, mu = p->mu, ir = p->inv_rho, lp2m = l + 2.0 * mu;
      const double u = q[6], v = q[7], w = q[8];
      if (dim == 0) {
        f[0] = lp2m * u; f[1] = l * u; f[2] = l * u; f[3] = mu * v; f[4] = mu * w; f[5] = 0.0;
        f[6] = ir * q[0]; f[7] = ir * q[3]; f[8] = ir * q[4];
      } else if (dim == 1) {
        f[0] = l * v; f[1] = lp2m * v; f[2] = l * v; f[3] = mu * u; f[4] = 0.0; f[5] = mu * w;
        f[6] = ir * q[3]; f[7] = ir * q[1]; f[8] = ir * q[5];
      } else {
        f[0] = l * w; f[1] = l * w; f[2] = lp2m * w; f[3] = 0.0; f[4] = mu * u; f[5] = mu * v;
        f[6] = ir * q[4]; f[7] = ir * q[5]; f[8] = ir * q[2];
      }
      return;
    }
    case ORC_PDE_ADVECTION:
      for (int s = 0; s < m; ++s) f[s] = -p->v[dim] * q[s];
      return;
    case ORC_PDE_DEMO: {
      /* output row r of dim 0 is -(q[r] + two partners); dims 1,2 rotate (0 1 2)(3 4 5) */
      static const int rows[3][3][4] = {
          {{0, 0, 3, 4}, {1, 1, 3, 5}, {2, 2, 4, 5}},
          {{1, 1, 4, 5}, {2, 2, 4, 3}, {0, 0, 5, 3}},
          {{2, 2, 5, 3}, {0, 0, 5, 4}, {1, 1, 3, 4}}};
      for (int s = 0; s < 6; ++s) f[s] = 0.0;
      for (int r = 0; r < 3; ++r) {
        const int* t = rows[dim][r];
        f[t[0]] = -(q[t[1]] + q[t[2]] + q[t[3]]);
      }
      return;
    }
    default: /* ncp-advection, source-only: zero flux */
      for (int s = 0; s < m; ++s) f[s] = 0.0;
      return;
  }
}

/* B_dim * grad (pde.cpp:13-17 default zero, :96-100 ncp-advection). */
static void pde_ncp(const orc_pde* p, const double* g, int dim, double* out) {
  for (int s = 0; s < p->m; ++s) out[s] = p->kind == ORC_PDE_NCP_ADVECTION ? -p->v[dim] * g[s] : 0.0;
}

/* Gaussian amplitude derivative via the probabilists' Hermite recurrence (pde.cpp:48-59). */
static double gauss_deriv(const orc_pde* p, int order, double t) {
  const double u = (t - p->src_center) / p->src_width;
  double hm = 0.0, h = 1.0, scale = 1.0;
  for (int k = 0; k < order; ++k) {
    const double hn = u * h - k * hm;
    hm = h;
    h = hn;
  }
  for (int k = 0; k < order; ++k) scale *= -1.0 / p->src_width;
  return p->src_amp * scale * h * exp(-0.5 * u * u);
}

/* --------------------------------------------------------------- the STP ---- */

/* dst (+)= D along dim, unpadded s-fastest (predictor_common.cpp:148-168). */
static void derive(int dim, int n, int m, const double* dmat, const double* src, double* dst,
                   int accumulate) {
  const long sx = m, sy = (long)n * m, sz = (long)n * n * m;
  const long line = dim == 0 ? sx : dim == 1 ? sy : sz;
  for (int z = 0; z < n; ++z)
    for (int y = 0; y < n; ++y)
      for (int x = 0; x < n; ++x) {
        const int k = dim == 0 ? x : dim == 1 ? y : z;
        const long base = z * sz + y * sy + x * sx;
        const long start = base - k * line;
        for (int s = 0; s < m; ++s) {
          double acc = 0.0;
          for (int l = 0; l < n; ++l) acc += dmat[k * n + l] * src[start + l * line + s];
          dst[base + s] = accumulate ? dst[base + s] + acc : acc;
        }
      }
}

typedef struct {
  int n;
  double nodes[ORC_MAX_ORDER], w[ORC_MAX_ORDER], d[ORC_MAX_ORDER * ORC_MAX_ORDER];
  double fl[ORC_MAX_ORDER], fr[ORC_MAX_ORDER];
  double src_phi[3][ORC_MAX_ORDER];
} orc_basis;

/* One element: stp_splitck (stp_splitck.cpp:13-81) then extrapolate_faces
 * (predictor_common.cpp:311-341).  work holds 4 * n^3 * m doubles. */
static void stp_element(const orc_basis* b, const orc_pde* p, const double* q, double dt,
                        double t0, double* qavg, double* favg, double* fq, double* ff,
                        double* work) {
  const int n = b->n, m = p->m;
  const long nn = (long)n * n * n, vol = nn * m;
  double* pp = work;
  double* pt = work + vol;
  double* fl = work + 2 * vol;
  double* gr = work + 3 * vol;
  double tmp[ORC_MAX_Q], amp[ORC_MAX_Q];
  memcpy(pp, q, sizeof(double) * vol);
  for (long i = 0; i < vol; ++i) qavg[i] = dt * q[i];
  double c = dt;
  for (int o = 1; o < n; ++o) {
    memset(pt, 0, sizeof(double) * vol);
    if (p->n_src) { /* weak Dirac scatter P[k] * S^(o-1)(t0) (predictor_common.cpp:271-283) */
      for (int s = 0; s < m; ++s) amp[s] = 0.0;
      amp[p->src_comp] = gauss_deriv(p, o - 1, t0);
      for (int z = 0; z < n; ++z)
        for (int y = 0; y < n; ++y)
          for (int x = 0; x < n; ++x) {
            const double pz = b->src_phi[2][z] * b->src_phi[1][y] * (1.0 / b->w[z]) * (1.0 / b->w[y]);
            const double pk = pz * b->src_phi[0][x] * (1.0 / b->w[x]);
            double* node = pt + (((long)z * n + y) * n + x) * m;
            for (int s = 0; s < m; ++s) node[s] += pk * amp[s];
          }
    }
    for (int d = 0; d < 3; ++d) {
      for (long k = 0; k < nn; ++k) pde_flux(p, pp + k * m, d, fl + k * m);
      derive(d, n, m, b->d, fl, pt, 1);
      derive(d, n, m, b->d, pp, gr, 0);
      for (long k = 0; k < nn; ++k) {
        pde_ncp(p, gr + k * m, d, tmp);
        for (int s = 0; s < m; ++s) pt[k * m + s] += tmp[s];
      }
    }
    c *= dt / (o + 1); /* dt^(o+1)/(o+1)! (stp_splitck.cpp:64) */
    for (long i = 0; i < vol; ++i) qavg[i] += c * pt[i];
    double* sw = pp;
    pp = pt;
    pt = sw;
  }
  if (favg)
    for (int d = 0; d < 3; ++d)
      for (long k = 0; k < nn; ++k) pde_flux(p, qavg + k * m, d, favg + d * vol + k * m);
  /* faces: contract along the normal dim with phi(0) / phi(1); (a,b) = remaining dims
   * in (z,y,x) order, quantity fastest (predictor.hpp:16-21) */
  const long face = (long)n * n * m;
  for (int d = 0; d < 3; ++d)
    for (int side = 0; side < 2; ++side) {
      const double* coef = side ? b->fr : b->fl;
      double* oq = fq ? fq + (2 * d + side) * face : NULL;
      double* of = ff ? ff + (2 * d + side) * face : NULL;
      for (int a = 0; a < n; ++a)
        for (int bb = 0; bb < n; ++bb)
          for (int s = 0; s < m; ++s) {
            double aq = 0.0, af = 0.0;
            for (int j = 0; j < n; ++j) {
              const int k3 = d == 2 ? j : a;
              const int k2 = d == 0 ? bb : d == 1 ? j : a;
              const int k1 = d == 0 ? j : bb;
              const long idx = (((long)k3 * n + k2) * n + k1) * m + s;
              aq += coef[j] * qavg[idx];
              if (favg) af += coef[j] * favg[d * vol + idx];
            }
            if (oq) oq[((long)a * n + bb) * m + s] = aq;
            if (of) of[((long)a * n + bb) * m + s] = af;
          }
    }
}

int orc_stp_batch(int n, int m, long n_elem, const double* q, const double* par,
                  const double* args, int pde_kind, double dt, double t_start, double* qavg,
                  double* favg, double* face_q, double* face_f, int n_threads) {
  if (n < 1 || n > ORC_MAX_ORDER || m < 1 || m > ORC_MAX_Q || !(dt > 0.0) || n_elem < 0) return -1;
  if (pde_kind < 0 || pde_kind > ORC_PDE_SOURCE_ONLY) return -1;
  if ((pde_kind == ORC_PDE_ELASTIC || pde_kind == ORC_PDE_ELASTIC_SOURCE) && (m != 9 || !par)) return -1;
  if (pde_kind == ORC_PDE_DEMO && m != 6) return -1;
  if (face_f && !favg) return -1;
  const long nn = (long)n * n * n, vol = nn * m, face = (long)n * n * m;
  for (long i = 0; i < n_elem * vol; ++i)
    if (!isfinite(q[i])) return -1; /* validate_stp's finiteness sweep (:143-145) */
  orc_basis b;
  b.n = n;
  orc_make_basis(n, b.nodes, b.w, b.d, b.fl, b.fr);
  orc_pde base;
  memset(&base, 0, sizeof base);
  base.kind = pde_kind;
  base.m = m;
  if (pde_kind == ORC_PDE_ADVECTION || pde_kind == ORC_PDE_NCP_ADVECTION)
    for (int i = 0; i < 3; ++i) base.v[i] = args[i];
  if (pde_kind == ORC_PDE_ELASTIC_SOURCE || pde_kind == ORC_PDE_SOURCE_ONLY) {
    base.n_src = 1;
    for (int i = 0; i < 3; ++i) base.src_pos[i] = args[i];
    base.src_comp = (int)args[3];
    base.src_amp = args[4];
    base.src_center = args[5];
    base.src_width = args[6];
    if (base.src_comp < 0 || base.src_comp >= m) return -1;
    for (int dd = 0; dd < 3; ++dd) orc_lagrange_values_at(n, b.nodes, base.src_pos[dd], b.src_phi[dd]);
  }
  int bad = 0;
  if (n_threads < 1) n_threads = 1;
#pragma omp parallel num_threads(n_threads)
  {
    double* work = (double*)malloc(sizeof(double) * 4 * vol);
#pragma omp for schedule(static)
    for (long e = 0; e < n_elem; ++e) {
      orc_pde p = base;
      if (pde_kind == ORC_PDE_ELASTIC || pde_kind == ORC_PDE_ELASTIC_SOURCE) {
        const double lam = par[3 * e], mu = par[3 * e + 1], rho = par[3 * e + 2];
        if (!(rho > 0.0) || mu < 0.0 || !(lam + 2.0 * mu > 0.0)) { /* pde.cpp:175-176 */
#pragma omp atomic write
          bad = 1;
          continue;
        }
        p.lam = lam;
        p.mu = mu;
        p.inv_rho = 1.0 / rho;
      }
      stp_element(&b, &p, q + e * vol, dt, t_start, qavg + e * vol, favg ? favg + e * 3 * vol : NULL,
                  face_q ? face_q + e * 6 * face : NULL, face_f ? face_f + e * 6 * face : NULL, work);
    }
    free(work);
  }
  return bad ? -1 : 0;
}

/* ------------------------------------------------------------ corrector ----- */

int orc_corrector_step(int n, int m, int e, double domain_len, int pde_kind, const double* par3,
                       const double* args, double max_wavespeed, double* u, const double* qavg,
                       const double* face_q, const double* face_f) {
  if (n < 1 || n > ORC_MAX_ORDER || m < 1 || m > ORC_MAX_Q || e < 1 || !(domain_len > 0.0)) return -1;
  if (pde_kind == ORC_PDE_ELASTIC_SOURCE || pde_kind == ORC_PDE_SOURCE_ONLY) return -1;
  if (pde_kind == ORC_PDE_ELASTIC && (m != 9 || !par3)) return -1;
  orc_basis b;
  b.n = n;
  orc_make_basis(n, b.nodes, b.w, b.d, b.fl, b.fr);
  orc_pde p;
  memset(&p, 0, sizeof p);
  p.kind = pde_kind;
  p.m = m;
  if (pde_kind == ORC_PDE_ELASTIC) {
    p.lam = par3[0];
    p.mu = par3[1];
    p.inv_rho = 1.0 / par3[2];
  }
  if (pde_kind == ORC_PDE_ADVECTION || pde_kind == ORC_PDE_NCP_ADVECTION)
    for (int i = 0; i < 3; ++i) p.v[i] = args[i];
  const double h = domain_len / e, gs = 1.0 / h, smax = gs * max_wavespeed; /* ScaledPde (solver.cpp:111-156) */
  const long nn = (long)n * n * n, vol = nn * m, face = (long)n * n * m;
  const long cells = (long)e * e * e;
  double* fw = (double*)malloc(sizeof(double) * vol);
  double* gw = (double*)malloc(sizeof(double) * vol);
  double* vv = (double*)malloc(sizeof(double) * vol);
  double* fh = (double*)malloc(sizeof(double) * face);
  double tmp[ORC_MAX_Q];
  int bad = 0;
  for (long c = 0; c < cells; ++c) {
    const int ix = (int)(c % e), iy = (int)((c / e) % e), iz = (int)(c / ((long)e * e));
    const double* qa = qavg + c * vol;
    double* uc = u + c * vol;
    /* volume: sum_d D_d F_d(qavg) + B_d (D_d qavg), flux and ncp scaled by 1/h */
    memset(vv, 0, sizeof(double) * vol);
    for (int d = 0; d < 3; ++d) {
      for (long k = 0; k < nn; ++k) {
        pde_flux(&p, qa + k * m, d, fw + k * m);
        for (int s = 0; s < m; ++s) fw[k * m + s] *= gs;
      }
      derive(d, n, m, b.d, fw, vv, 1);
      derive(d, n, m, b.d, qa, gw, 0);
      for (long k = 0; k < nn; ++k) {
        pde_ncp(&p, gw + k * m, d, tmp);
        for (int s = 0; s < m; ++s) vv[k * m + s] += gs * tmp[s];
      }
    }
    for (long i = 0; i < vol; ++i) uc[i] += vv[i];
    /* surface (solver.cpp:211-250): plus side = the neighbour in +d */
    for (int d = 0; d < 3; ++d)
      for (int side = 0; side < 2; ++side) {
        const int step = side == 0 ? -1 : 1;
        const int nx = ((ix + (d == 0 ? step : 0)) % e + e) % e;
        const int ny = ((iy + (d == 1 ? step : 0)) % e + e) % e;
        const int nz = ((iz + (d == 2 ? step : 0)) % e + e) % e;
        const long nb = ((long)nz * e + ny) * e + nx;
        const double* mq = face_q + c * 6 * face;
        const double* mf = face_f + c * 6 * face;
        const double* tq = face_q + nb * 6 * face;
        const double* tf = face_f + nb * 6 * face;
        const double* q_plus = side == 1 ? tq + (2 * d) * face : mq + (2 * d) * face;
        const double* q_minus = side == 1 ? mq + (2 * d + 1) * face : tq + (2 * d + 1) * face;
        const double* f_plus = side == 1 ? tf + (2 * d) * face : mf + (2 * d) * face;
        const double* f_minus = side == 1 ? mf + (2 * d + 1) * face : tf + (2 * d + 1) * face;
        for (long i = 0; i < face; ++i)
          fh[i] = 0.5 * (f_plus[i] + f_minus[i]) - 0.5 * smax * (q_minus[i] - q_plus[i]);
        const double* fs = mf + (2 * d + side) * face;
        const double* coeff = side == 0 ? b.fl : b.fr;
        const double sign = side == 0 ? -1.0 : 1.0;
        for (int a = 0; a < n; ++a)
          for (int bb = 0; bb < n; ++bb)
            for (int j = 0; j < n; ++j) {
              const double scale = sign * coeff[j] * (1.0 / b.w[j]);
              const long node = d == 0 ? ((long)a * n + bb) * n + j : d == 1 ? ((long)a * n + j) * n + bb
                                                                            : ((long)j * n + a) * n + bb;
              for (int s = 0; s < m; ++s)
                uc[node * m + s] += scale * (fh[((long)a * n + bb) * m + s] - fs[((long)a * n + bb) * m + s]);
            }
      }
    for (long i = 0; i < vol; ++i)
      if (!isfinite(uc[i])) bad = 1;
  }
  free(fw);
  free(gw);
  free(vv);
  free(fh);
  return bad ? -2 : 0;
}

/* -------------------------------------------------------------- layouts ----- */

void orc_canonical_to_aosoa(int n, int m, int qs, long n_elem, const double* src, double* dst) {
  const long nn = (long)n * n * n;
  for (long e = 0; e < n_elem; ++e)
    for (int k3 = 0; k3 < n; ++k3)
      for (int k2 = 0; k2 < n; ++k2)
        for (int s = 0; s < qs; ++s)
          for (int k1 = 0; k1 < n; ++k1)
            dst[e * (long)n * n * qs * n + (((long)k3 * n + k2) * qs + s) * n + k1] =
                s < m ? src[e * nn * m + (((long)k3 * n + k2) * n + k1) * m + s] : 0.0;
}

void orc_aosoa_to_canonical(int n, int m, int qs, long n_elem, const double* src, double* dst) {
  const long nn = (long)n * n * n;
  for (long e = 0; e < n_elem; ++e)
    for (int k3 = 0; k3 < n; ++k3)
      for (int k2 = 0; k2 < n; ++k2)
        for (int k1 = 0; k1 < n; ++k1)
          for (int s = 0; s < m; ++s)
            dst[e * nn * m + (((long)k3 * n + k2) * n + k1) * m + s] =
                src[e * (long)n * n * qs * n + (((long)k3 * n + k2) * qs + s) * n + k1];
}
