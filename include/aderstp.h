/*
 * aderstp — B200-native (sm_100a) linear ADER-DG Space-Time Predictor, C ABI.
 *
 * This is the drop-in boundary for the reference's hot path.  Each entry point names the
 * reference interface it replaces (paths relative to /root/reference/proj):
 *
 *   aderstp_predict_batch       <- ader::predict(Variant, const ElementTensor& q, const LinearPde&,
 *                                  double dt, const BasisOperators&, ScratchArena&,
 *                                  PredictorOutput&, double t_start)
 *                                  include/ader/predictor.hpp:118-120 (+ stp_* :94-116)
 *                                  followed by ader::extrapolate_faces(PredictorOutput&, ...)
 *                                  include/ader/predictor.hpp:125
 *                                  One call = one batch of independent elements on the GPU.
 *   aderstp_predict_batch_host  <- same, with host buffers (the call a CPU caller such as
 *                                  run_simulation, src/solver.cpp:334-345, makes); copies in and
 *                                  out are pipelined against the kernel.
 *   aderstp_plan_create         <- SolverConfig (include/ader/config.hpp:21-28) + make_basis
 *                                  (include/ader/basis.hpp:37, src/basis.cpp:110-122) + the
 *                                  LinearPde factories (include/ader/pde.hpp:62-84).  Kernels never
 *                                  allocate (include/ader/predictor.hpp:31-34): all state lives
 *                                  in the plan.
 *   aderstp_basis               <- ader::make_basis (src/basis.cpp:110-122), host side.
 *   aderstp_flop_count          <- ader::flop_count (include/ader/predictor.hpp:86), reporting the
 *                                  algorithmic count of this implementation.
 *   aderstp_correct_batch       <- ader::corrector_step(Mesh&, std::vector<PredictorOutput>&,
 *                                  const LinearPde&, const BasisOperators&, double dt, double t,
 *                                  int workers)  include/ader/solver.hpp:87-93, src/solver.cpp:257-311
 *   aderstp_run_simulation      <- ader::run_simulation(const LinearPde&, const SolverConfig&, Mesh&,
 *                                  double t_end, Variant, const AnalyticFn*, int workers)
 *                                  include/ader/solver.hpp:102-104, src/solver.cpp:313-359
 *   aderstp_last_error          <- the std::invalid_argument messages of validate_stp
 *                                  (src/predictor_common.cpp:129-146); nothing is thrown across
 *                                  the ABI.
 *
 * All device pointers are plain CUDA device addresses; `stream` is a cudaStream_t (NULL = the
 * legacy default stream).  Calls are asynchronous on `stream` unless stated otherwise.
 * Thread-safe for distinct (plan, stream) pairs.
 *
 * Batch layouts (e = element index, n = order = nodes per dim, m = quantities):
 *   q            ADERSTP_LAYOUT_AOSOA : [e][k3][k2][s < q_stride][k1]     (native, x fastest)
 *                ADERSTP_LAYOUT_AOS   : [e][k3][k2][k1][s < q_stride]     (reference ElementTensor,
 *                                                                           q_stride = m_pad = 16)
 *   qavg         same layout kind as q, quantity slots = out_stride (padding written as 0.0)
 *   favg         [e][d = 0..2][ one qavg-shaped tensor ]
 *   face_q/f     [e][f][a][b][s < m], f = -x,+x,-y,+y,-z,+z; (a,b) = the two in-face dims in
 *                (z,y,x) order; exactly the reference's PredictorOutput::face_q/face_f arrays
 *                (include/ader/predictor.hpp:16-29).
 *   par          [e][3]: (lambda, mu, rho) or (rho, cp, cs) per element (elastic kinds only).
 */
#ifndef ADERSTP_H
#define ADERSTP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADERSTP_ABI_VERSION 2

/* status codes */
#define ADERSTP_OK 0
#define ADERSTP_ERR_INVALID_ARG 1   /* shape / pointer / dt checks of validate_stp            */
#define ADERSTP_ERR_UNSUPPORTED 2   /* order or quantity count without a compiled kernel        */
#define ADERSTP_ERR_NONFINITE 3     /* "stp: non-finite input DOFs" (predictor_common.cpp:143)   */
#define ADERSTP_ERR_MATERIAL 4      /* "elastic_pde: need rho > 0, mu >= 0, lambda + 2mu > 0"   */
#define ADERSTP_ERR_CUDA 5          /* CUDA runtime error (message in aderstp_last_error)        */

/* PDE kinds: the reference's factories (include/ader/pde.hpp:62-84) */
#define ADERSTP_PDE_ELASTIC 0        /* elastic_pde(lambda, mu, rho) per element, m = 9           */
#define ADERSTP_PDE_ADVECTION 1      /* advection_pde(v, m): pde_args[0..2] = v                   */
#define ADERSTP_PDE_NCP_ADVECTION 2  /* ncp_advection_pde(v, m): pde_args[0..2] = v               */
#define ADERSTP_PDE_DEMO 3           /* paper_demo_pde(), m = 6                                   */
#define ADERSTP_PDE_ELASTIC_SOURCE 4 /* elastic_pde(lambda, mu, rho, PointSourceSpec) per element */
#define ADERSTP_PDE_SOURCE_ONLY 5    /* source_only_pde(m, PointSourceSpec)                       */
#define ADERSTP_PDE_LINEAR 6         /* any constant-coefficient LinearPde, given by its probed
                                        flux Jacobians A_d and ncp matrices B_d (aderstp_config) */

/* point source spec in pde_args (include/ader/pde.hpp:47-56):
 *   [0..2] position, [3] component, [4] amplitude, [5] center, [6] width
 * ELASTIC_SOURCE and SOURCE_ONLY always carry one; ADERSTP_PDE_LINEAR carries one when
 * pde_args[7] != 0 (a user LinearPde with source_count() == 1, pde.hpp:37-39). */

#define ADERSTP_PAR_LAMBDA_MU_RHO 0
#define ADERSTP_PAR_RHO_CP_CS 1

#define ADERSTP_LAYOUT_AOSOA 0
#define ADERSTP_LAYOUT_AOS 1

/* quantities per node: any m <= 64 (systems beyond the term-table kernels -- m > 16 or more than
 * four nonzeros in a row of A_d + B_d -- run on the general kernel, stp_general.cu) */
#define ADERSTP_MAX_QUANTITIES 64

typedef struct aderstp_config {
  int order;       /* n = nodes per dimension (reference cfg.order); 2..10 compiled      */
  int quantities;  /* m; 9 for the elastic kinds                                          */
  int pde_kind;    /* ADERSTP_PDE_*                                                       */
  int layout;      /* ADERSTP_LAYOUT_* for q, qavg, favg                                  */
  int q_stride;    /* quantity slots per node in q (>= m); 0 = m                          */
  int out_stride;  /* quantity slots per node in qavg/favg (>= m); 0 = m                  */
  int par_kind;    /* ADERSTP_PAR_* (elastic kinds)                                       */
  int check_inputs;/* 1 = flag non-finite q / invalid material (validate_stp semantics)  */
  double pde_args[8];
  /* ADERSTP_PDE_LINEAR only: row-major m x m, linear[d] = A_d (flux Jacobian, F_d(q) = A_d q)
   * and linear[3 + d] = B_d (ncp: out = B_d * grad_d q); NULL entries mean zero. */
  const double* linear[6];
} aderstp_config;

typedef struct aderstp_plan aderstp_plan;

/* ---- plan ---------------------------------------------------------------------------- */
int aderstp_plan_create(const aderstp_config* cfg, aderstp_plan** plan);
void aderstp_plan_destroy(aderstp_plan* plan);
/* Elements per second of this plan are independent; the plan is immutable after creation. */

/* ---- the hot path ---------------------------------------------------------------------- */
/* Device buffers.  favg, face_q and face_f may be NULL (not computed / not written).
 * Asynchronous; with check_inputs the input checks are reported by aderstp_plan_status. */
int aderstp_predict_batch(const aderstp_plan* plan, int64_t n_elem, const double* q,
                          const double* par, double dt, double t_start, double* qavg,
                          double* favg, double* face_q, double* face_f, void* stream);

/* Host buffers (pinned or pageable).  Synchronous: splits the batch into chunks and overlaps
 * host->device copies, the kernel and device->host copies on three streams (chunk i on
 * stream i mod 3), using device scratch owned by the plan (allocated on first use, or up front
 * by aderstp_plan_reserve_host_path -- the only allocation this call can make).  Returns the
 * input-check status directly. */
int aderstp_predict_batch_host(aderstp_plan* plan, int64_t n_elem, const double* q,
                               const double* par, double dt, double t_start, double* qavg,
                               double* favg, double* face_q, double* face_f);
int aderstp_plan_reserve_host_path(aderstp_plan* plan, int64_t chunk_elems);

/* The plan keeps the device scratch its calls allocated (AoS staging <= 512 MiB per call, the
 * time loop's face buffers) in a stream-ordered pool until it is destroyed; this returns that
 * memory to the device now (synchronises the device). */
int aderstp_plan_trim(aderstp_plan* plan);

/* Synchronises `stream` and returns (and clears) the input-check status of the plan's
 * previous launches: ADERSTP_OK, ADERSTP_ERR_NONFINITE or ADERSTP_ERR_MATERIAL. */
int aderstp_plan_status(aderstp_plan* plan, void* stream);

/* ---- layouts (reference AoS <-> native AoSoA, include/ader/layout.hpp:44-50,
 *      src/layout.cpp:168-194), device buffers, asynchronous ------------------------------ */
int aderstp_convert_layout(int order, int quantities, int64_t n_elem, int src_layout,
                           int src_stride, const double* src, int dst_layout, int dst_stride,
                           double* dst, void* stream);

/* ---- seeded synthetic inputs on the device (BASELINE.json configs) --------------------
 * dist 0: Q ~ U[-1,1]; 1: Q ~ N(0,1) (Box-Muller); 2: three random-phase sinusoids per
 * quantity on a periodic grid of `grid` elements per side.  Elements [e0, e0+n_elem) of the
 * stream defined in DESIGN.md (SplitMix64, element-major draw order); par receives
 * (rho, cp, cs) per element.  q uses the plan-independent layout given here, m = 9. */
int aderstp_generate(int dist, uint64_t seed, int order, int64_t e0, int64_t n_elem, int grid,
                     int layout, int q_stride, double* q, double* par, void* stream);

/* ---- the GPU time loop around the predictor --------------------
 * Uniform periodic Cartesian mesh on [0, domain_len]^3 with e elements per dimension (ader::Mesh,
 * include/ader/solver.hpp:16-32): element (ix, iy, iz) is (iz*e + iy)*e + ix and its state is one
 * q-layout tensor of the plan (layout, q_stride). */
typedef struct aderstp_mesh {
  int elements_per_dim;
  double domain_len;
} aderstp_mesh;

/* corrector_step(mesh, outs, pde, ops, dt, t) (src/solver.cpp:257-311; correct_cell :184-253):
 * u += V(qavg) + the point source's projection x its time integral over [t, t + dt] (:206-216,
 * integrals :266-278) + the Rusanov surface fluctuations lifted through the inverse mass, from
 * this step's predictor outputs of every element (qavg in the plan's output layout, face_q /
 * face_f).  The predictor outputs must come from the PDE scaled by 1/h (ScaledPde,
 * src/solver.cpp:111-156), as aderstp_run_simulation does.  max_wavespeed: the PDE's unscaled
 * max_wavespeed(); for ADERSTP_PDE_ELASTIC a negative value means "per face, the larger cp of its
 * two elements" (per-element material has no reference counterpart; with one material it equals
 * the reference).  dt and t only enter through the point source.  Device buffers, asynchronous; a
 * non-finite update is reported by aderstp_plan_status as ADERSTP_ERR_NONFINITE (the reference
 * throws "corrector_step: non-finite update"). */
int aderstp_correct_batch(const aderstp_plan* plan, const aderstp_mesh* mesh, double* u,
                          const double* par, const double* qavg, const double* face_q,
                          const double* face_f, double max_wavespeed, double dt, double t,
                          void* stream);

/* run_simulation (src/solver.cpp:313-359): steps of dt = min(stable_dt, t_end - t) until t_end,
 * each = aderstp_predict_batch on the 1/h-scaled PDE + aderstp_correct_batch, with
 * stable_dt = cfl h / (3 smax (2n - 1)) (:170-174).  u: device state (in/out); par: per-element
 * material (elastic) or NULL.  max_wavespeed as above (elastic, negative: the max over elements
 * of cp).  Synchronous.  Returns ADERSTP_ERR_NONFINITE when a step produced a non-finite state
 * (RunResult.stable = false); *steps and *t_final report the completed steps. */
int aderstp_run_simulation(const aderstp_plan* plan, const aderstp_mesh* mesh, double* u,
                           const double* par, double cfl, double t_end, double max_wavespeed,
                           int64_t* steps, double* t_final, void* stream);

/* ---- the time loop over several GPUs: z-slabs of the mesh, one per rank -------------------
 * Rank r owns the layers [z0, z0 + nz) (elements (iz - z0) e^2 + iy e + ix of its arrays).  The
 * corrector reads the predictor faces of the two neighbouring slabs straight from their memory
 * (peer pointers over NVLink: aderstp_ipc_handle / aderstp_ipc_open), inside the same kernel
 * that applies them -- there is no separate halo copy.  With one slab (nz = e) the halos are
 * unused and everything equals aderstp_correct_batch / aderstp_run_simulation. */
typedef struct aderstp_slab {
  int z0;
  int nz;
} aderstp_slab;

typedef struct aderstp_halo {
  const double* face_q; /* the neighbouring slab's face_q / face_f (its predictor outputs)        */
  const double* face_f;
  const double* par;    /* its per-element material (elastic kinds: per-face smax), else NULL     */
  int z_base;           /* its first layer                                                        */
} aderstp_halo;

int aderstp_correct_slab(const aderstp_plan* plan, const aderstp_mesh* mesh, const aderstp_slab* slab,
                         double* u, const double* par, const double* qavg, const double* face_q,
                         const double* face_f, const aderstp_halo* lo, const aderstp_halo* hi,
                         double max_wavespeed, double dt, double t, void* stream);

/* Host synchronisation between the ranks, called twice per step: after the predictor (the faces
 * of every slab are complete) and after the corrector (nobody reads them any more).  It receives
 * this rank's flag (non-zero = non-finite state) and returns the maximum over all ranks. */
typedef int (*aderstp_rank_sync_fn)(void* ctx, int local_flag);

/* run_simulation on this rank's slab: face_q / face_f are this rank's predictor output buffers
 * (n_local x 6 x n^2 m doubles each, shared with the neighbours), lo / hi the neighbours' (peer
 * pointers).  max_wavespeed > 0 is the GLOBAL maximum wave speed (same dt on every rank); the
 * elastic corrector uses the per-face max(cp) from par and the halos' par. */
int aderstp_run_simulation_slab(const aderstp_plan* plan, const aderstp_mesh* mesh, const aderstp_slab* slab,
                                double* u, const double* par, double* face_q, double* face_f,
                                const aderstp_halo* lo, const aderstp_halo* hi, double cfl, double t_end,
                                double max_wavespeed, aderstp_rank_sync_fn sync, void* ctx, int64_t* steps,
                                double* t_final, void* stream);

/* device buffers shareable with other processes (cudaMalloc'd, so their IPC handle addresses
 * the buffer itself) and CUDA IPC handles (64 bytes) */
int aderstp_device_alloc(size_t bytes, void** ptr);
int aderstp_device_free(void* ptr);
int aderstp_ipc_handle(const void* ptr, void* handle64);
int aderstp_ipc_open(const void* handle64, void** ptr);
int aderstp_ipc_close(void* ptr);

/* ---- host helpers -------------------------------------------------------------------- */
int aderstp_basis(int order, double* nodes, double* weights, double* d, double* face_left,
                  double* face_right);
/* algorithmic fp64 FLOPs and HBM bytes per element of the elastic STP */
double aderstp_flop_count(int order, int quantities);
double aderstp_byte_count(int order, int quantities, int with_favg);
int aderstp_supported_order(int order);
const char* aderstp_last_error(void);
int aderstp_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* ADERSTP_H */
