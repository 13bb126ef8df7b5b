/* TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C11) of the reference's linear Space-Time Predictor hot path, used
 * exclusively as the parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  The product (paper_2003_12787_b200/libaderstp.so) never links or calls it.
 *
 * Parity pinning: every function below is checked against the unmodified reference compiled
 * into oracle/_ref/ (tests/test_oracle.py) and against the committed golden vectors under
 * tests/golden/ that were generated from oracle/_ref by tests/golden/make_golden.py.
 *
 * Canonical batch layout used by this oracle (same as oracle/ref_shim.cpp):
 *   q, qavg : [e][k3][k2][k1][s]        favg : [e][d][k3][k2][k1][s]
 *   face_q, face_f : [e][f][a][b][s]    f = -x,+x,-y,+y,-z,+z
 */
#ifndef STP_ORACLE_H
#define STP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_PDE_ELASTIC = 0,        /* par[e] = (lambda, mu, rho)                        */
  ORC_PDE_ADVECTION = 1,      /* args = (vx, vy, vz)                               */
  ORC_PDE_NCP_ADVECTION = 2,  /* args = (vx, vy, vz)                               */
  ORC_PDE_DEMO = 3,           /* paper demo system, m = 6                          */
  ORC_PDE_ELASTIC_SOURCE = 4, /* par[e] = (lambda, mu, rho); args = source (7)     */
  ORC_PDE_SOURCE_ONLY = 5     /* args = source (px,py,pz,component,amp,center,width) */
};

#define ORC_MAX_ORDER 31

/* proj/src/basis.cpp:26-53, :73-88, :90-104, :110-122 */
int orc_make_basis(int n, double* nodes, double* weights, double* d, double* face_left,
                   double* face_right);
void orc_lagrange_values_at(int n, const double* nodes, double x, double* vals);

/* proj/include/ader/util.hpp:72-90: output number k (0-based) of SplitMix64(seed). */
uint64_t orc_splitmix64_at(uint64_t seed, uint64_t k);
double orc_u01(uint64_t x);
double orc_symmetric(uint64_t x);

/* Seeded synthetic inputs (the BASELINE.json configs), canonical layout, elements
 * [e0, e0+count).  par_rcc receives (rho, cp, cs) per element.  dist: 0 = U[-1,1],
 * 1 = N(0,1) (Box-Muller), 2 = sum of three random-phase sinusoids per quantity on a
 * periodic grid of `grid` elements per side. */
void orc_generate(int dist, uint64_t seed, int n, long e0, long count, int grid, double* q,
                  double* par_rcc);
/* (rho, cp, cs) -> (lambda, mu, rho):  mu = rho cs^2, lambda = rho cp^2 - 2 mu */
void orc_material_lmr(long count, const double* par_rcc, double* par_lmr);

/* SplitCK predictor + face extrapolation for a batch (proj/src/stp_splitck.cpp:13-81,
 * proj/src/predictor_common.cpp:311-341), OpenMP over elements when n_threads > 1.
 * favg / face_q / face_f may be NULL.  Returns 0, or -1 on invalid arguments (the
 * conditions of validate_stp, proj/src/predictor_common.cpp:129-146). */
int orc_stp_batch(int n, int m, long n_elem, const double* q, const double* par,
                  const double* args, int pde_kind, double dt, double t_start, double* qavg,
                  double* favg, double* face_q, double* face_f, int n_threads);

/* One corrector step (proj/src/solver.cpp:257-311, correct_cell :184-253) on a periodic e^3
 * mesh of element size h = domain_len / e with ONE material / PDE for all elements (like the
 * reference): u += V(qavg) on the 1/h-scaled PDE (apply_volume_once,
 * predictor_common.cpp:243-259) + the Rusanov surface fluctuations lifted through the inverse
 * mass; smax = max_wavespeed / h.  u, qavg canonical; faces [c][f][a][b][s].  Point sources are
 * not supported (as in the GPU corrector).  Returns 0, -1 on bad arguments, -2 when the update
 * is not finite ("corrector_step: non-finite update"). */
int orc_corrector_step(int n, int m, int e, double domain_len, int pde_kind, const double* par3,
                       const double* args, double max_wavespeed, double* u, const double* qavg,
                       const double* face_q, const double* face_f);

/* Canonical <-> native AoSoA ([k3][k2][s<q_stride][k1]) per element. */
void orc_canonical_to_aosoa(int n, int m, int q_stride, long n_elem, const double* src,
                            double* dst);
void orc_aosoa_to_canonical(int n, int m, int q_stride, long n_elem, const double* src,
                            double* dst);

#ifdef __cplusplus
}
#endif

#endif
