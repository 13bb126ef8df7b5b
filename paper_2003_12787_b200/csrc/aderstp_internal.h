// Internal interface between the host C ABI (capi.cpp) and the sm_100a kernels (stp_kernels.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace aderstp {

constexpr int kMinOrder = 2;
constexpr int kMaxOrder = 10;
constexpr int kMaxM = 16;      // quantities of the term-table kernels (stp_kernel, corrector tables)
constexpr int kMaxTerms = 4;   // nonzeros per (row s, dim d) of a table PDE
constexpr long long kGenScratchBytes = 512ll << 20;  // general kernel's global scratch per launch
// stp_wpe beats stp_dmmap at nDof 4 from ~3,000 elements on, at nDof 5 from ~16,000
constexpr long long kWpeMinElems4 = 8192, kWpeMinElems5 = 32768;

// Host-side basis, derived from scratch (basis.cpp).  d[k*n + l] = phi_l'(x_k).
struct HostBasis {
  int n = 0;
  double nodes[kMaxOrder], weights[kMaxOrder], d[kMaxOrder * kMaxOrder];
  double face_left[kMaxOrder], face_right[kMaxOrder];
};
int make_host_basis(int n, HostBasis* out);
void lagrange_values(int n, const double* nodes, double x, double* vals);

// Everything a kernel launch needs besides the batch pointers; lives in the plan.
struct LaunchPlan {
  int n = 0, m = 0, kind = 0;        // order, quantities, ADERSTP_PDE_*
  int layout = 0, q_stride = 0, out_stride = 0, par_kind = 0, check = 0;
  HostBasis basis;
  // table PDE terms (non-elastic kinds), t_s += sum_k tc * D_d (p_{tr}) and favg via fr/fc
  int n_terms = 1;
  signed char tr[kMaxM][3][kMaxTerms];
  double tc[kMaxM][3][kMaxTerms];
  signed char fr[kMaxM][3][kMaxTerms];
  double fc[kMaxM][3][kMaxTerms];
  // point source: component < 0 means none; proj factors phi_d(x_src)/w per dim;
  int src_comp = -1;
  double src_pos[3] = {0, 0, 0};
  double src_amp = 0, src_center = 0, src_width = 1;
  double src_proj[3][kMaxOrder];
  double src_scale = 1.0;            // ScaledPde source scale 1/h^3 in the time loop (solver.cpp:147-150)
  // general kernel (stp_general.cu): device CSR rows of C_d = A_d + B_d and of A_d, per (s, d)
  struct GeneralTables {
    const int* t_ptr = nullptr;
    const int* t_col = nullptr;
    int t_nnz = 0;
    const double* t_dense = nullptr;  // C_d dense [d][j][s < m rounded up to 8] (general kernel)
    const double* f_dense = nullptr;  // A_d dense, same layout (stp_gdense favg / face_f)
    const double* t_val = nullptr;
    const int* f_ptr = nullptr;
    const int* f_col = nullptr;
    const double* f_val = nullptr;
    double scale = 1.0;              // ScaledPde gradient scale 1/h in the time loop
    cudaMemPool_t pool = nullptr;    // the plan's pool (global scratch for large m N^3)
  } gen;
  unsigned int* d_status = nullptr;  // device word: bit0 non-finite q, bit1 bad material
  int force_generic = 0;             // env ADERSTP_FORCE_GENERIC=1: skip specialised kernels
  int no_dmma8 = 0;                  // env ADERSTP_NO_DMMA8=1: nDof 8 on the line-pass kernel
  int dmma8_prefetch = 0;            // L2 prefetch distance (elements) of q; env ADERSTP_PREFETCH, 0 = off
  int aos_chunk = 0;                 // env ADERSTP_AOS_CHUNK: elements per chunk of the AoS staged path (tests)
  int pass_slots = 0;                // env ADERSTP_PASS_SLOTS: 6 = line-pass kernel, 12 = bipartite, 0 auto
  int aos_staged = 0;                // env ADERSTP_AOS_STAGED=1: reference layout through the transposes
  int no_dmmap = 0;                  // env ADERSTP_NO_DMMAP=1: nDof 4..7 on the line-pass kernel
  int no_gdense = 0;                 // env ADERSTP_NO_GDENSE=1: dense systems at nDof 8 on stp_general
  int wpe = 2;                       // warp-per-element kernel: 0 off, 1 forced at nDof 4 / 6, 2 automatic
                                     // (nDof 4 / 5 from kWpeMinElems4 / 5 elements on); env ADERSTP_WPE=0|1
};

struct BatchArgs {
  const double* q;
  const double* par;
  double* qavg;
  double* favg;
  double* face_q;
  double* face_f;
  long long n_elem;
  double dt;
  double t_start;
  // fused time-step mode (GPU time loop): also write u_next = q + L(qavg) in q's layout, i.e. the
  // corrector's volume term (solver.cpp:199-207) applied by one more Horner step; qavg may then be
  // null.  Only kernels with fused_supported() honour it.
  double* u_next = nullptr;
  // volume mode (with u_next, stp_dmma8 only): the corrector's volume term alone, u_next = q +
  // L(vol_r) with vol_r = qavg (compact AoSoA); no faces, no Horner recursion
  const double* vol_r = nullptr;
};

// corrector.cu: GPU corrector step (proj/src/solver.cpp:184-311) and time-loop helpers
// Predictor outputs of a z-slab of the mesh held elsewhere (a neighbouring rank's buffers, read
// through peer memory over NVLink), element (iz - z_base mod e) * e^2 + iy * e + ix.
struct HaloRef {
  const double* face_q = nullptr;
  const double* face_f = nullptr;
  const double* par = nullptr;
  int z_base = 0;
};
struct CorrArgs {
  double* u;             // mesh state of the slab, the plan's q layout, local element (iz-z0)*e^2 + iy*e + ix
  const double* par;     // per-element material (elastic)
  const double* qavg;    // null: surface terms only (the fused predictor applied the volume term)
  const double* face_q;
  const double* face_f;
  int e;                 // elements per dimension (periodic)
  double inv_h;          // 1 / h
  double smax;           // scaled max wave speed, < 0: elastic per-face max(cp) / h
  int z0 = 0, nz = 0;    // this slab: layers [z0, z0 + nz); nz = 0 means the whole mesh
  HaloRef lo, hi;        // the slabs below / above (used for z-neighbours outside [z0, z0 + nz))
  // point source (correct_cell, solver.cpp:206-216): u[comp] += proj[node] * sint
  int src_comp = -1;
  double src_sint = 0.0;
  const double* src_proj = nullptr;  // n^3 doubles, point_source_projection (basis.cpp:124-142)
};
cudaError_t launch_correct(const LaunchPlan& p, const CorrArgs& a, cudaStream_t stream);
cudaError_t launch_scale_par(const double* in, int par_kind, double s, long long n, double* out,
                             cudaStream_t stream);
cudaError_t launch_max_cp(const double* par, int par_kind, long long n, unsigned long long* out,
                          cudaStream_t stream);

// stp_general.cu: any m, dense / sparse matrices, point source, every order and layout
bool general_selected(const LaunchPlan& p);
cudaError_t launch_general(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);
void source_amplitudes(const LaunchPlan& p, double t, int n, double* amp);  // S^(o)(t) x src_scale
// stp_gdense.cu: the general systems at nDof 8 (m <= 21, no point source) on the tensor cores
bool gdense_applicable(const LaunchPlan& p, const BatchArgs& a);
cudaError_t launch_gdense(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);

// stp_kernels.cu
cudaError_t launch_stp(const LaunchPlan& plan, const BatchArgs& args, cudaStream_t stream);
bool fused_supported(const LaunchPlan& plan, const BatchArgs& args);  // u_next honoured by the dispatch
cudaError_t launch_convert(int n, int m, long long n_elem, int src_layout, int src_stride,
                           const double* src, int dst_layout, int dst_stride, double* dst,
                           cudaStream_t stream);
cudaError_t launch_generate(int dist, uint64_t seed, int n, long long e0, long long n_elem,
                            int grid, int layout, int q_stride, const HostBasis& basis,
                            double* q, double* par, cudaStream_t stream);
bool kernel_available(int n);
// stp_dmma8.cu: nDof = 8 elastic kernel on the fp64 tensor cores
bool dmma8_applicable(const LaunchPlan& p);
bool dmma8_aos_applicable(const LaunchPlan& p, const BatchArgs& a);
bool dmma8_table_applicable(const LaunchPlan& p, const BatchArgs& a);
// stp_dmma_table.cu: table PDEs at nDof 4..7 on zero-padded DMMA tiles
bool dmmat_applicable(const LaunchPlan& p, const BatchArgs& a);
cudaError_t init_dmmat(const LaunchPlan& p);
cudaError_t launch_dmmat(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);
cudaError_t launch_dmma8_table(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);
bool bip_aos_applicable(const LaunchPlan& p, const BatchArgs& a);
bool dmmap_aos_applicable(const LaunchPlan& p, const BatchArgs& a);
cudaError_t launch_bip(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);
cudaError_t init_dmma8(const LaunchPlan& p);  // once per device, at plan creation
// stp_dmma.cu: nDof 4..7 on zero-padded 8x8 DMMA tiles
bool dmmap_applicable(const LaunchPlan& p);
cudaError_t init_dmmap(const LaunchPlan& p);
cudaError_t launch_dmmap(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);
// stp_wpe.cu: nDof 4, 6 with one warp per element (DFMA tile tasks, no CTA barrier)
bool wpe_applicable(const LaunchPlan& p, const BatchArgs& a);
cudaError_t init_wpe(const LaunchPlan& p);
cudaError_t launch_wpe(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);
// stp_pass.cu: line-pass elastic kernel for every order (even/odd split D, uniform operands)
bool pass_applicable(const LaunchPlan& p);
// table PDEs (term tables) at nDof 9, 10 on line passes (stp_tlp); init_pass uploads its even/odd D
bool tlp_applicable(const LaunchPlan& p, const BatchArgs& a);
cudaError_t launch_tlp(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);
cudaError_t init_pass(const LaunchPlan& p);
cudaError_t launch_pass(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);
bool bip_selected(const LaunchPlan& p, const BatchArgs& a);  // launch_pass takes the bipartite kernel
cudaError_t launch_dmma8(const LaunchPlan& p, const BatchArgs& a, cudaStream_t stream);

// Elastic flux tables for the tuned kernels' epilogues (proj/src/pde.cpp:180-218):
// F_d(q)_s = c[coef(s,d)] q[in(s,d)] with c = (lambda + 2 mu, lambda, mu, 1/rho) and coef 4 = an
// exact zero entry.  constexpr, so with compile-time (s, d) every index folds to a constant.
__host__ __device__ constexpr int e_in(int s, int d) {
  constexpr int t[9][3] = {{6, 7, 8}, {6, 7, 8}, {6, 7, 8}, {7, 6, 0}, {8, 0, 6},
                           {0, 8, 7}, {0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
  return t[s][d];
}
__host__ __device__ constexpr int e_coef(int s, int d) {
  constexpr int t[9][3] = {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {2, 2, 4}, {2, 4, 2},
                           {4, 2, 2}, {3, 3, 3}, {3, 3, 3}, {3, 3, 3}};
  return t[s][d];
}

}  // namespace aderstp
