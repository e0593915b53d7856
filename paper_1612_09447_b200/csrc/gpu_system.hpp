// GpuSystem: the B200-resident counterpart of the reference FemSystem
// (proj/include/eqs/fem_system.hpp:30-73) plus the integrator state
// (proj/include/eqs/integrators.hpp:23-29). Host code controls, the device
// holds every vector and matrix. With nranks > 1 each instance owns one
// partition of the node-ownership decomposition (partition.hpp) and talks to
// its peers through a Comm (comm.hpp); with one rank it is the whole problem.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <deque>
#include <functional>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "comm.hpp"
#include "dev.cuh"
#include "eqs_internal.hpp"
#include "partition.hpp"

namespace eqsb {

struct SolveStats {
  long m_solves = 0, pcg_iterations = 0, rho_solves = 0, rho_pcg_iterations = 0;
  long precond_setups = 0, assemblies = 0, applies = 0, spe_fallbacks = 0;
  long svd_count = 0, appends = 0;  // StartVectorEstimator::Stats (start_vector.hpp:45-49)
  long newton_linear_solves = 0, newton_pcg_iterations = 0;  // implicit path (ode_system.hpp:25-26)
  double t_residual = 0, t_solve = 0, t_setup = 0, t_estimator = 0;
};
struct SolveRecord {
  double t = 0;
  int estimator_rank = 0, iterations = 0;
  double initial_rel_residual = 0;
};
struct PcgResult {
  int iterations = 0;
  double rel_residual = 0, initial_rel_residual = 0;
  bool converged = false;
};
struct StepAttempt {
  double t_start = 0, dt = 0;
  bool accepted = false;
  int stages = 0, newton_iterations = 0;
  double error = 0, rho = 0, dt_next = 0;
};
struct RkcOptions {
  double rtol = 1e-2, atol = 1e-8;
  int max_stages = 200, rho_refresh_every = 25;
};
struct SdirkOptions {  // proj/include/eqs/integrators.hpp:106-110
  double rtol = 1e-2, atol = 1e-8;
  double newton_tol = 1e-8;
  int max_newton = 25;
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {  // swap: the old buffer is freed with o
    std::swap(p, o.p);
    std::swap(n, o.n);
    return *this;
  }
  ~DevBuf();
  void alloc(size_t count);
  void upload(const T* host, size_t count, cudaStream_t s);
  void download(T* host, size_t count, cudaStream_t s) const;
};

// halo of one level's index space on this rank (partition.hpp LocalSpace)
struct DevHalo {
  int n_own = 0, n_send = 0;
  DevBuf<int> send_idx;      // concatenated per-peer send lists (local owned indices)
  DevBuf<double> send_buf;
  DevBuf<float> send_buf32;
  std::vector<int> peers, send_off, send_cnt, recv_off, recv_cnt;
};

// device buffers of a SELL copy (sell.hpp), all three value precisions
struct SellBufs {
  DevBuf<long> cp;
  DevBuf<int> bases;
  DevBuf<uint16_t> code;
  DevBuf<double> v64;
  DevBuf<float> v32;
  DevBuf<uint16_t> v16;
  DevBuf<int> pk_cp, pk_bases, pk_perm;  // packed bf16 copy (sell.hpp SELL-P)
  DevBuf<uint32_t> pk_words;
  DevBuf<uint16_t> st_vals;     // stencil-coded bf16 copy (sell.hpp SELL-S)
  DevBuf<unsigned char> st_pid;
  DevBuf<int> st_pat;
  DevBuf<double> st_v64;
  DevBuf<uint16_t> sh_u16;      // symmetric half storage (SELL-SH)
  DevBuf<double> sh_u64;
  DevBuf<unsigned char> sh_spid;
  DevBuf<int> sh_sinfo;
  DevBuf<unsigned char> sh_slow;
  DevBuf<int> sh_slow_base;
};

struct DevLevel {
  int n_own = 0, n_loc = 0, n_global = 0;
  bool replicated = false;           // held whole on every rank (partition.hpp rep_level)
  DevCsr A, P, R;
  DevBuf<int> a_rp, a_ci, p_rp, p_ci, r_rp, r_ci;
  DevBuf<double> a_v, p_v, r_v;
  DevBuf<float> a_vf, p_vf, r_vf;  // fp32 copies for the V-cycle
  SellBufs a_s, p_s, r_s;          // SELL copies (level 0: A shares the PCG operator's)
  DevBuf<double> invd, b, z, z2, t, db, dt;
  DevBuf<float> invd32, b32, z32, z2_32, t32, db32, dt32;  // fp32 V-cycle vectors
  ChebCoef cheb{}, cheb1{};          // degree-2 and degree-1 Chebyshev coefficients
  double lambda_smoother = 0;
  DevHalo halo;
  DevBuf<int> glob;                  // partitioned coarsest level: local -> global ids
  DevBuf<double> full_b, full_z;     // partitioned coarsest level: whole vectors for the dense solve
};

// timing classes (eqs_timing in include/eqs_b200.h)
enum TimeClass { TC_STIFF = 0, TC_PCG = 1, TC_VCYCLE = 2, TC_RKC = 3, TC_SPE = 4, TC_BOUNDARY = 5, TC_PCG_GRAPH = 6, TC_COUNT = 8 };

struct DevLevel;
void cheb_first_kind(double lmax, double ratio, DevLevel& lv);
// set by the C-ABI around the construction of a multi-rank context: called
// once the rank's host setup (problem, M, AMG, partition plan) is done and the
// global hierarchy released, before the collective device build
extern thread_local std::function<void()> setup_gate_release;

class GpuSystem {
 public:
  // comm == nullptr: single rank
  GpuSystem(Problem&& p, int device, std::unique_ptr<Comm> comm = nullptr);
  ~GpuSystem();

  // sizes (global unless noted)
  int n_dofs() const { return n_dofs_; }
  int n_free() const { return n_free_; }
  int n_fixed() const { return n_fixed_; }
  int n_tets() const { return n_tets_; }
  int n_own() const { return n_own_; }  // free dofs owned by this rank
  int rank() const { return comm_->rank(); }
  int nranks() const { return comm_->size(); }
  const PartitionPlan& plan() const { return plan_; }
  const Problem& problem() const { return prob_; }
  const HostCsr& mass_ii() const { return m_ii_; }
  const HostCsr& mass_ib() const { return m_ib_; }
  const AmgHierarchy& amg() const { return amg_; }
  const std::vector<int>& colors();  // lazily computed (bit-exact, matfree.cpp:11-38)
  int n_colors();
  SolveStats& stats() { return stats_; }
  std::vector<SolveRecord>& solve_records() { return records_; }
  cudaStream_t stream() const { return stream_; }
  bool host_only() const { return device_ < 0; }

  // ---- operators on device buffers (local numbering [owned | ghosts | local fixed])
  void kx_apply_full_dev(const double* x_state, const double* v, double* y);  // rows: all local
  void residual_dev(double t, double* x_full, double* r);  // r (owned) = -(K(x)x) - M_IB xdot_B(t)
  void lift_dev(double t, double* x_full);                  // fixed tail <- x_B(t)
  void mass_apply_dev(double* v, double* y);                // v with room for ghosts
  PcgResult pcg_dev(const double* b, const double* x0, double* x, double tol, int max_iter);
  PcgResult eval_rhs_dev(double t, double* x_full, double* f);
  void apply_minv_stiffness_dev(double t, double* x_full, const double* v_own, double* y);
  double estimate_spectral_radius(double t, double* x_full);

  // ---- host-pointer wrappers in reference dof numbering (single rank)
  void kx_apply_host(const double* x_state, const double* v, double* y);
  void kx_residual_host(const double* x_full, const double* b_mass, double* r);
  void eval_residual_host(double t, const double* x, double* r);
  PcgResult eval_rhs_host(double t, const double* x, double* f);
  PcgResult mass_solve_host(const double* b, const double* x0, double tol, int max_iter, double* x);
  double mass_solve_sequence(const double* B, int k, double tol, int max_iter, double* X, int* its);
  void reset_estimator(int mode);  // switch zero/previous/spe/pod_fixed/pod_rolling and drop the history
  int estimator_next_host(const double* b, double* x0);            // returns current_rank()
  // > 0 (threshold >= 0) replaces the value; others keep it
  void set_pod_params(int snapshots, int rank, int capacity, double threshold) {
    if (snapshots > 0) prob_.solver.pod_snapshots = snapshots;
    if (rank > 0) prob_.solver.pod_rank = rank;
    if (capacity > 0) prob_.solver.pod_capacity = capacity;
    if (threshold >= 0.0) prob_.solver.pod_threshold = threshold;
  }
  void estimator_feedback_host(const double* x, int iterations);
  void mass_apply_host(const double* v, double* y);
  void apply_minv_stiffness_host(double t, const double* x_state, const double* v, double* y);
  void lift_full_host(double t, const double* x_free, double* x_full);

  // ---- integrator state (device resident). Host vectors are the owned part
  // (n_own entries, global free order restricted to plan().space[0].owned).
  void set_state(double t, const double* x_own, double dt);
  void get_state(double* x_own);
  double state_t = 0, state_dt = 0;
  long st_accepted = 0, st_rejected = 0, st_stages = 0;
  double rho_value = 0;
  long rho_age = 0;
  bool rho_valid = false;
  double spectral_radius_cached(int refresh_every);
  StepAttempt rkc_step(const RkcOptions& o);
  void rkc_advance_fixed(double dt, int s);
  StepAttempt euler_step(double dt);
  // SDIRK3(2) implicit baseline (integrators.cpp:237-343): Newton per stage with
  // the matrix M + gamma dt K(z) assembled on the device (fem_system.cpp:124-145)
  StepAttempt sdirk_step(const SdirkOptions& o);
  // per-cell kappa of the resident state at state_t, reference tet order (VTK dump)
  void cell_kappa_host(double* kappa);
  // FemSystem::shifted_solve with host vectors (fem_system.cpp:124-145)
  void shifted_solve_host(double t, const double* z, double gdt, const double* rhs, double* delta, bool refresh);
  bool sdirk_advance_fixed(double dt, const SdirkOptions& o);
  long st_newton = 0;
  double* state_dev() { return X_; }
  double* scratch_full() { return full_[0].p != X_ ? full_[0].p : full_[1].p; }

  // ---- options / timing
  int stiffness_mode = 0;  // 0 blocked scatter, 1 coloured, 2 two-pass gather
  int cheb_degree = 2;     // fine level (1 or 2)
  int coarse_degree = 1;   // levels >= 1 (1 or 2)
  int fine_pre_degree = 0; // fine pre-smoother degree override (option 29; 0 = cheb_degree)
  bool stencil_rowsum = true;  // bf16 row-sum correction in the stencil copy's padding (option 30)
  double cheb_ratio = 6.0;
  int cheb_kind = 0;          // 0 first-kind Chebyshev on [lmax/ratio, lmax], 1 fourth-kind
  double cheb_scale = 1.1;    // lmax = cheb_scale x the power estimate of lambda_max(D^-1 A)
  bool use_graphs = true;
  bool pcg_graph_loop = true;  // eqs_set_option 20
  // eqs_set_option 22: the graph-resident PCG loop also on multi-rank NCCL
  // contexts (halo + allreduces captured into the WHILE body). Off by default:
  // NCCL inside a conditional graph body has not run on multi-GPU hardware.
  bool pcg_graph_multi = false;
  bool spe_incremental = true;  // false: the reference's full MGS rebuild on every solve
  void set_cheb(double ratio);
  void set_vcycle_precision(int prec);  // V-cycle matrix values: 0 fp64, 1 fp32, 2 bf16
  void set_sell(bool on);               // SELL-16 copies instead of CSR where available
  void set_stencil(bool on);            // stencil-coded fine-level V-cycle operator where available
  void set_stencil_sym(bool on);        // its symmetric half storage (SELL-SH) where built
  void set_stencil_rowsum(bool on);     // row-sum correction slot of the stencil copy (option 30)
  void truncate_vcycle_prolongators();  // solver.amg_vcycle_truncate
  void restore_reference_hierarchy();
  void set_vcycle_vectors_f32(bool on) {  // V-cycle vectors fp32 (default) or fp64
    invalidate_graphs();
    vcycle_f32_ = on;
  }
  void set_level_tpr(int level, int tpr);  // threads per row of A_l (level 0 also sets M_II)
  void invalidate_graphs();
  int vcycle_precision() const { return vcycle_prec_; }
  bool sell_on() const { return sell_on_; }
  bool timing_on = false;
  bool timing_graph = false;  // timing keeps the graph-resident PCG (one TC_PCG_GRAPH region per solve)
  bool shift_amg = true;      // SDIRK shifted solves: SA-AMG rebuilt per refresh (default) or Jacobi (option 26)
  int wcycle_from = 0;  // > 0: W-cycle (two coarse-grid corrections) on levels >= this (option 28; 0 = V-cycle)
  bool shift_pcg_graph = true;  // shifted AMG solves through pcg_dev (graph loop, fp32 V-cycle; option 27)
  void tic(int cls);
  void toc(int cls, double bytes);
  void timing_resolve(double ms[TC_COUNT], long launches[TC_COUNT], double bytes[TC_COUNT]);
  void timing_reset();
  double kx_bytes() const;  // algorithmic bytes of one K(x)v
  double spmv_bytes(const DevCsr& a) const;
  int amg_levels() const { return (int)levels_.size(); }
  const DevLevel& level(int l) const { return levels_[l]; }

 private:
  void build_device();
  void build_levels();
  void build_halo(const LocalSpace& sp, DevHalo& h);
  template <class T>
  void halo(DevHalo& h, T* vec);  // fill ghosts of vec from the owners
  void allreduce(int slot, int count = 1);
  template <class XT>
  XT* vcycle_t(int l, const XT* b, bool dot_into_rz, const double* r64, double* out64, const XT* pre);
  bool level_takes_pre(int l) const;
  void vcycle_prepare(const double* r);  // fp32 V-cycle: b32, db32 of the fine level from r
  double* vcycle(const double* r);  // fine-level V-cycle: z (fp64), r.z in S_RZ
  // z = M^-1 r (returned buffer), S_RZ <- r.z; prepared: the PCG update already
  // wrote the fp32 V-cycle inputs
  double* precondition(double* r, bool prepared = false);
  void build_kx_gather();
  const std::vector<int>& tet_dofs_host();
  void kx_into(const double* x, const double* v, const double* base, double sign, double* out, int n_out);
  void kx_tets(const double* x, const double* v);
  double read_scalar(int slot);
  void read_scalars(int first, int count, double* out);
  double dot_n(int n, const double* a, const double* b, int slot);  // global dot over n owned entries
  double dot_local(int n, const double* a, const double* b, int slot);  // no reduction over ranks
  double dot_own(const double* a, const double* b, int slot);       // level-0 owned entries
  void check_kernel_flags();
  void sync();
  std::vector<double> set_values(double t, bool rates) const;
  void require_single(const char* what) const;
  // estimator (start_vector.cpp:84-109,152-164)
  bool estimator_next(const double* r, double* x0);
  void estimator_feedback(const double* x, int iterations);
  int estimator_rank_ = 0;
  // incremental SPE basis (Q orthonormal, W = M Q, G = Q'MQ, H = Q R)
  std::vector<std::unique_ptr<DevBuf<double>>> spe_q_[2], spe_w_[2];
  int spe_set_ = 0, spe_k_ = 0;
  bool spe_clean_ = true;
  std::vector<double> spe_G_ = std::vector<double>((size_t)kMaxMulti * kMaxMulti, 0.0);
  std::vector<double> spe_R_ = std::vector<double>((size_t)kMaxWin * kMaxWin, 0.0);
  double* spe_q(int set, int j);
  double* spe_w(int set, int j);
  void spe_alloc(int window);
  void spe_g_column(int k);
  void spe_rebuild();
  void spe_append(double* h);
  void spe_downdate();
  // SDIRK Newton matrix: per M_II entry the element contributions (ascending
  // tet), per-tet packed element matrices, the shifted values and the Jacobi
  // diagonal of the last refresh
  bool sdirk_stages(double dt, const SdirkOptions& o, int& newton_iters, double* est);
  void shifted_solve_dev(double t, double* z_full, double gdt, const double* rhs, double* delta, bool refresh);
  void build_shift_map();
  bool shift_built_ = false, shift_precond_ = false, shift_amg_on_ = false;
  struct ShiftAmg;
  std::unique_ptr<ShiftAmg> sh_amg_;
  void build_shift_amg();
  double* shift_vcycle(const double* r);
  void shift_swap();
  void S_op_view();
  DevBuf<long> sh_ptr_, sh_src_;
  DevBuf<double> sh_S_, sh_vals_, sh_diag_;
  DevBuf<int> sh_err_;
  DevCsr sh_csr_;
  DevBuf<double> sd_buf_[16];
  double* sd(int i);
  // POD estimators (start_vector.cpp:64-71,111-150,165-187): snapshot ring,
  // thin QR of the snapshots (Q, R), Jacobi SVD of R on the host, basis
  // U = Q U_R, W = M U and the reduced inverse (U'MU)^-1
  std::vector<std::unique_ptr<DevBuf<double>>> pod_snap_, pod_q_, pod_u_, pod_w_;
  int pod_nsnap_ = 0, pod_next_slot_ = 0, pod_rank_ = 0;
  bool pod_stale_ = false, pod_built_ = false, pod_ok_ = false;
  std::vector<double> pod_ginv_;
  std::vector<int> iteration_history_;
  DevBuf<double>* pod_buf(std::vector<std::unique_ptr<DevBuf<double>>>& v, int j);
  void multi_dot_chunked(int m, const double* const* V, const double* w, double* out);
  void lincomb_chunked(int m, const double* const* V, const double* c, double* y);
  void pod_build_dev();
  void pod_factor();
  bool pod_start(const double* b, double* x0);
  double pod_rolling_threshold() const;

 public:
  // StartVectorEstimator public API (start_vector.hpp:52-66), device vectors
  bool estimator_next_dev(const double* b, double* x0, int* rank);
  void estimator_feedback_dev(const double* x, int iterations) { estimator_feedback(x, iterations); }

 private:
  int vcycle_prec_ = 2;
  bool vcycle_f32_ = true;
  bool sell_on_ = true;
  cudaGraphExec_t vcycle_graph_ = nullptr;  // captured V-cycle (rebuilt when options change)
  double* vcycle_out_ = nullptr;
  long vcycle_graph_kernels_ = 0;
  double vcycle_graph_bytes_ = 0.0;
  // graph-resident PCG loops (pcg_dev), one per solution pointer x: a WHILE
  // conditional node whose body is one iteration (V-cycle, direction, SpMV+dot,
  // update, device stopping rule)
  std::unordered_map<double*, cudaGraphExec_t> pcg_graphs_;
  std::unordered_map<double*, long> pcg_graph_use_;  // LRU clock per cached graph
  long pcg_graph_clock_ = 0;

 public:
  long pcg_graph_captures = 0;  // whole-PCG graph (re)captures (stats: a cache-thrash signal)

 private:
  long pcg_body_kernels_ = 0;
  double pcg_body_bytes_ = 0.0;
  DevBuf<double> pcg_stat_;
  double* pcg_pinned_ = nullptr;  // host pinned [9]: stat in / out
  cudaGraphExec_t pcg_loop_graph(double* x, bool f32);
  PcgResult pcg_dev_graph(const double* b, bool use_x0, const double* x0, double* x, double tol, int max_iter,
                          double bnorm);

  Problem prob_;
  int device_ = 0;
  std::unique_ptr<Comm> comm_;
  cudaStream_t stream_ = nullptr;
  int n_dofs_ = 0, n_free_ = 0, n_fixed_ = 0, n_tets_ = 0, n_local_ = 4, order_ = 1, n_sets_ = 0;
  int n_own_ = 0, n_ghost_ = 0, n_loc_ = 0, n_fixloc_ = 0, n_full_ = 0, n_tets_loc_ = 0;
  PartitionPlan plan_;
  std::vector<int> loc2ref_;  // local full index -> reference dof id
  std::vector<int> colors_;
  int n_colors_ = -1;
  HostCsr m_ii_, m_ib_;
  AmgHierarchy amg_;
  std::vector<AmgHostLevel> amg_stash_;  // reference P_1/R_1/A_l (l >= 2) while the V-cycle's are built
  std::vector<double> amg_stash_coarse_inv_;
  SolveStats stats_;
  std::vector<SolveRecord> records_;

  // device mesh data
  DevBuf<double> coords_;  // [n_full][4]
  DevBuf<int> tet_dofs_;   // [n_tets_loc][n_local] local full numbering
  DevBuf<unsigned char> tet_mat_;
  DevBuf<long> slot_ptr_;  // two-pass gather mode (stiffness_mode 2), built on first use
  DevBuf<int> slots_;
  DevBuf<double> ytet_;
  bool slots_built_ = false;
  std::vector<int> tet_dofs_h_;
  // blocked scatter (kxblock.hpp, default)
  DevBuf<int> kb_tets_, kb_tet0_, kb_dof0_, kb_sptr_, kb_lout_, kb_bdof_, kb_bptr_, kb_bpart_;
  DevBuf<unsigned char> kb_mat_;
  DevBuf<uint16_t> kb_slots_, kb_tloc_;
  DevBuf<int> kb_ldof_;
  DevBuf<double> kb_partials_, kb_bxyz_;
  KxDev kxd_;
  long kx_partials_ = 0, kx_ldofs_ = 0, kx_slots_ = 0;
  DevBuf<int> err_;  // kernel error flags
  DevBuf<int> set_of_fixed_;
  DevBuf<int> bl_rows_;
  DevBuf<double> bl_coef_;
  int n_bl_rows_ = 0;
  // colour batches (lazy)
  DevBuf<int> color_tets_;
  std::vector<long> color_off_;
  // matrices
  DevCsr mii_;
  DevBuf<int> mii_rp_, mii_ci_;
  DevBuf<double> mii_v_, mii_invd_;
  SellBufs mii_s_;
  DevLevel dummy_level_;
  DevHalo halo0_;  // level-0 (fine dof) halo
  std::vector<DevLevel> levels_;
  DevBuf<double> coarse_inv_;
  DevBuf<float> coarse_inv32_;  // fp32 copy for the fp32 V-cycle's dense coarse solve
  int coarse_n_ = 0;
  int dev_levels_ = 1;          // levels of the device V-cycle (<= the hierarchy's)
  int dev_coarse_n_ = 0;
  std::vector<double> dev_coarse_inv_;  // host staging of the dense coarse inverse
  // reductions
  DevBuf<double> red_partials_, red_scal_;
  DevBuf<unsigned> red_counters_;
  Reducer red_{};
  double* pinned_ = nullptr;  // host pinned scalar mirror [S_COUNT + 8]
  // work vectors (level-0 vectors that are gathered carry room for ghosts)
  DevBuf<double> w_r_, w_z_, w_p_, w_q_, w_full_a_, w_full_b_, w_free_a_, w_free_b_;
  DevBuf<double> full_[4], F0_, F_, Fn_, rho_v_, rho_w_;  // full_: state + 3 stage buffers
  double* X_ = nullptr;
  // estimator history (device ring)
  std::vector<std::unique_ptr<DevBuf<double>>> hist_pool_;
  std::deque<double*> history_;
  // timing
  struct Ev {
    cudaEvent_t a, b;
    int cls;
    double bytes;
  };
  std::vector<Ev> events_;
  std::vector<cudaEvent_t> ev_pool_;
  int open_cls_ = -1, nest_ = 0;
  cudaEvent_t open_ev_ = nullptr;
  double open_bytes_ = 0.0;
  double acc_ms_[TC_COUNT] = {}, acc_bytes_[TC_COUNT] = {};
  long acc_n_[TC_COUNT] = {};
  cudaEvent_t get_event();
};

void cuda_check(cudaError_t e, const char* what);

}  // namespace eqsb
