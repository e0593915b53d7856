/*
 * eqs_b200.h — C-ABI of the B200-native RKC electro-quasistatic hot path
 * (arXiv 1612.09447), the drop-in boundary for the reference `eqsim` solver.
 *
 * Every entry point replaces one reference C++ interface; the citation in
 * front of each declaration names it (paths relative to /root/reference).
 * Plain pointers and sizes only. Return value: EQS_OK or an error code that
 * maps 1:1 onto the reference exception classes (proj/include/eqs/errors.hpp:10-37,
 * std::invalid_argument), so a C++ shim can rethrow the same class and the
 * reference's catch sites (proj/src/integrators.cpp:217,
 * proj/src/scenario.cpp:353-368) keep working. eqs_last_error() returns the
 * message of the last failing call on the calling thread.
 *
 * Pointer conventions: functions without a `_dev` suffix take HOST buffers
 * (copied in and out inside the call); `_dev` variants take device pointers
 * on the context's GPU and run on the context's stream. All calls are
 * synchronous with respect to the host. One context per host thread.
 */
#ifndef EQS_B200_H
#define EQS_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define EQS_OK 0
#define EQS_ERR_CONFIG 1           /* eqs::ConfigError */
#define EQS_ERR_NUMERICAL 2        /* eqs::NumericalError */
#define EQS_ERR_GEOMETRY 3         /* eqs::GeometryError */
#define EQS_ERR_INVALID_ARGUMENT 4 /* std::invalid_argument */
#define EQS_ERR_PARSE 5            /* eqs::ParseError */
#define EQS_ERR_CUDA 6             /* CUDA / NCCL failure (no reference counterpart) */
#define EQS_ERR_OTHER 7            /* any other std::exception */

typedef struct eqs_ctx eqs_ctx;

/* proj/include/eqs/materials.hpp:11-33 (ConstantConductivity / MicrovaristorConductivity) */
typedef struct {
  int region;     /* region id the material applies to */
  int kind;       /* 0 = constant, 1 = microvaristor */
  double eps_r;
  double kappa;   /* constant */
  double kappa_lo, kappa_hi, e_switch, width; /* microvaristor */
} eqs_material;

/* proj/include/eqs/excitation.hpp:13-27 */
typedef struct {
  int kind;       /* 0 = sinusoid, 1 = ramp, 2 = constant */
  double amplitude, frequency, phase; /* sinusoid */
  double rise_time;                   /* ramp (amplitude shared) */
  double value;                       /* constant */
} eqs_waveform;

/* proj/include/eqs/fem_system.hpp:15-21, amg.hpp:12-18, start_vector.hpp:29-38 */
typedef struct {
  int precond;            /* 0 = jacobi, 1 = ssor (GPU substitute: jacobi-preconditioned), 2 = amg */
  double rel_tol;         /* 1e-12 */
  int max_iter;           /* 500 */
  double rho_solve_tol;   /* 1e-4 */
  double amg_strength_threshold; /* 0.08 */
  double amg_prolongation_omega; /* 4/3 */
  int amg_smoother_sweeps;       /* 1 (GPU: Chebyshev degree 2 pre and post) */
  int amg_max_levels;            /* 10 */
  int amg_coarse_limit;          /* 64 */
  int estimator_mode;     /* 0 = zero, 1 = previous, 2 = spe, 3 = pod_fixed, 4 = pod_rolling */
  int spe_window;         /* 8 */
  double mgs_drop_tol;    /* 1e-8 */
  double amg_coarse_filter; /* additive: V-cycle coarse-operator filter eps (0 = off; configs default 0.0025) */
  int amg_dense_coarse;     /* additive: direct (dense) solve of the first coarse level with at most this many
                               rows in the device V-cycle; <= 0 = recurse to the coarsest (configs default 512) */
  /* start_vector.hpp:31-35 (POD modes); <= 0 selects the reference default */
  int pod_snapshots;        /* 40: pod_fixed solves collected before the basis is built */
  int pod_rank;             /* 10 */
  int pod_capacity;         /* 20: pod_rolling ring size */
  double pod_threshold;     /* pod_rolling: append when iterations exceed this; <= 0: 1.25 x running median */
} eqs_solver_params;

/* Problem description consumed by eqs_create: the arrays the reference's
 * FemSystem ctor reads through its const references
 * (proj/src/fem_system.cpp:27-36, proj/include/eqs/fem_system.hpp:59-62).
 * eqs_create COPIES everything; no host pointer is kept after it returns. */
typedef struct {
  int n_nodes;
  int n_tets;
  const double* nodes;       /* [n_nodes][3], metres (TetMesh::nodes, mesh.hpp:14) */
  const int* tets;           /* [n_tets][4], finalized orientation (mesh.hpp:15) */
  const int* region_id;      /* [n_tets] (mesh.hpp:16) */
  int order;                 /* 1 or 2 (DofMap::order, dofmap.hpp:23) */
  int n_dofs;
  const int* element_dofs;   /* [n_tets][n_local], n_local = 4 or 10 (dofmap.hpp:28) */
  int n_free;
  const int* free_dofs;      /* ascending (dofmap.hpp:30) */
  int n_fixed;
  const int* fixed_dofs;     /* ascending (dofmap.hpp:31) */
  const int* fixed_set;      /* [n_dofs] set index or -1 (dofmap.hpp:34) */
  int n_sets;
  const eqs_waveform* set_waveforms; /* [n_sets], by DofMap::set_names index */
  int n_materials;
  const eqs_material* materials;
  eqs_solver_params solver;
  int device;                /* CUDA device ordinal */
} eqs_problem_desc;

typedef struct {
  long n_nodes, n_tets, n_dofs, n_free, n_fixed, n_local, order, n_colors;
  long nnz_mass_free, nnz_mass_ib;
  long amg_levels;
} eqs_sizes;

/* proj/include/eqs/pcg.hpp:51-57 */
typedef struct {
  int iterations;
  double rel_residual;
  double initial_rel_residual;
  int converged;
} eqs_pcg_result;

/* proj/include/eqs/ode_system.hpp:11-31 */
typedef struct {
  long m_solves, pcg_iterations, rho_solves, rho_pcg_iterations;
  long newton_linear_solves, newton_pcg_iterations;
  long precond_setups, assemblies, svd_count;
  double time_residual, time_solve, time_setup, time_estimator;
  long applies;              /* MatFreeStiffness::applies() (matfree.hpp:43) */
  long spe_fallbacks;
  long estimator_appends;    /* StartVectorEstimator::Stats::appends (start_vector.hpp:47) */
} eqs_solve_stats;

/* proj/include/eqs/integrators.hpp:91-95 */
typedef struct {
  double rtol, atol;         /* StepControl (integrators.hpp:44-47) */
  int max_stages;            /* 200 */
  int rho_refresh_every;     /* 25 */
} eqs_rkc_options;

/* proj/include/eqs/integrators.hpp:106-110 (SdirkOptions); newton_tol <= 0 / max_newton <= 0 select
 * the reference defaults 1e-8 / 25 */
typedef struct {
  double rtol, atol;
  double newton_tol;
  int max_newton;
} eqs_sdirk_options;

/* proj/include/eqs/integrators.hpp:32-41 */
typedef struct {
  double t_start, dt;
  int accepted, stages, newton_iterations;
  double error, rho, dt_next;
} eqs_step_attempt;

/* proj/include/eqs/integrators.hpp:9-29 (IntegratorState incl. RhoCache) */
typedef struct {
  double t, dt;
  long accepted, rejected, stages;
  double rho_value;
  long rho_age;
  int rho_valid;
} eqs_state_info;

/* Device time per kernel class (CUDA events on the context stream), ms and
 * launches, accumulated since the last eqs_timing_reset. Classes:
 * 0 stiffness K(x)v, 1 PCG SpMV+vectors, 2 V-cycle, 3 RKC stage/error,
 * 4 SPE estimator, 5 boundary/lift, 6 whole graph-resident PCG loop (V-cycle +
 * SpMV + vectors; only with option 24, which keeps the graph loop while timing).
 * Only collected when enabled. */
typedef struct {
  double ms[8];
  long launches[8];
  double bytes[8];           /* algorithmic bytes moved (SURVEY.md §8d formulas) */
} eqs_timing;

/* ----------------------------------------------------------------- errors */
const char* eqs_last_error(void);

/* ----------------------------------------------------------------- lifetime */
/* FemSystem ctor (proj/src/fem_system.cpp:27-36) + MatFreeStiffness ctor
 * (proj/src/matfree.cpp:40-52: colouring) + the preconditioner build that the
 * reference does lazily on first use (proj/src/fem_system.cpp:48-54). */
int eqs_create(const eqs_problem_desc* desc, eqs_ctx** out);
/* SimConfig::from_json_text (proj/src/scenario.cpp:110-211) + mesh build
 * (generate_box_mesh / load_msh, scenario.cpp:224-229) + build_dof_map
 * (dofmap.cpp:22-91) + eqs_create. `workers` overrides the config (<=0 keeps it). */
int eqs_create_from_config(const char* json_text, int device, eqs_ctx** out);
void eqs_destroy(eqs_ctx* ctx);
int eqs_get_sizes(eqs_ctx* ctx, eqs_sizes* out);

/* ----------------------------------------------------------------- distributed (node ownership) */
/* One process per GPU: rank 0 calls eqs_nccl_unique_id (128 bytes), shares
 * it (e.g. torch.distributed broadcast), then every rank calls
 * eqs_create_distributed. Host vectors of a distributed context are the
 * owned part (eqs_get_owned). */
int eqs_nccl_unique_id(char* id128);
int eqs_create_distributed(const char* json_text, int device, int nranks, int rank, const char* id128,
                           eqs_ctx** out);
/* One process per rank on one node, halos and allreduces host-staged through
 * a POSIX shared-memory segment `shm_name` (same name on every rank, e.g.
 * "/eqs_<uuid>"): the backend for ranks that share a GPU or where NCCL is
 * unavailable. Deterministic (rank-order sums, bit-identical to the
 * virtual-rank group). Not graph-capturable: PCG keeps the host loop. */
int eqs_create_distributed_shm(const char* json_text, int device, int nranks, int rank, const char* shm_name,
                               eqs_ctx** out);
/* The same transport on host buffers, without a GPU (tests of the protocol). */
typedef struct eqs_comm eqs_comm;
int eqs_comm_open_shm(const char* shm_name, int nranks, int rank, eqs_comm** out);
void eqs_comm_close(eqs_comm* c);
int eqs_comm_barrier(eqs_comm* c);
int eqs_comm_allreduce_host(eqs_comm* c, double* buf, int count);
int eqs_comm_exchange_host(eqs_comm* c, int n_msgs, const int* peers, const double* const* send,
                           const int* send_counts, double* const* recv, const int* recv_counts);
/* nranks virtual ranks in one process (threads, device-to-device halos);
 * every later call on these contexts must be made concurrently from one
 * thread per rank. Used to test the partitioned path on a single GPU. */
int eqs_create_virtual_group(const char* json_text, int device, int nranks, eqs_ctx** out);
/* host-only partition plan of `rank` (no device, no collectives) */
int eqs_create_partition_host(const char* json_text, int nranks, int rank, eqs_ctx** out);
/* partition of the context's rank: info = {rank, nranks, levels, n_own(level 0)} */
int eqs_partition_info(eqs_ctx* ctx, long* info4);
/* level sizes {n_global, n_own, n_ghost, n_peers_recv, n_peers_send, n_local_tets, n_local_fixed,
   replicated (1: the level is held whole on every rank)} */
int eqs_partition_level(eqs_ctx* ctx, int level, long* info8);
/* owner rank per global index of a level; owned / ghost global ids of this rank */
int eqs_partition_owner(eqs_ctx* ctx, int level, int* owner);
int eqs_partition_owned(eqs_ctx* ctx, int level, int* ids);
int eqs_partition_ghosts(eqs_ctx* ctx, int level, int* ids);
/* global ids this rank sends to `peer` at a level, in the peer's ghost order (returns count) */
int eqs_partition_send(eqs_ctx* ctx, int level, int peer, int* ids, int* count);

/* ----------------------------------------------------------------- setup artefacts (bit-exact checks) */
/* color_elements (proj/src/matfree.cpp:11-38): colour of every tet. */
int eqs_get_colors(eqs_ctx* ctx, int* color_of_tet);
/* TetMesh / DofMap arrays as built by eqs_create_from_config. */
int eqs_get_mesh(eqs_ctx* ctx, double* nodes, int* tets, int* region_id);
int eqs_get_dofs(eqs_ctx* ctx, int* element_dofs, int* free_dofs, int* fixed_dofs);
/* assemble_mass + split_dirichlet (proj/src/assembly.cpp:172-176,188-193): M_II (which=0) or M_IB (1). */
int eqs_get_mass(eqs_ctx* ctx, int which, int* row_ptr, int* col_idx, double* values);
/* AmgPreconditioner hierarchy (proj/src/amg.cpp:90-143): rows/nnz per level,
 * aggregates of level l (proj/src/amg.cpp:49-88). */
int eqs_amg_levels(eqs_ctx* ctx, int* n_levels, long* rows_nnz);
int eqs_amg_aggregates(eqs_ctx* ctx, int level, int* agg);
/* A (which 0), P (1) or R (2) of an AMG level in CSR (AmgPreconditioner levels,
 * proj/include/eqs/amg.hpp:40-50). Call with null arrays to get dims =
 * {rows, cols, nnz}. Single-rank contexts. */
int eqs_amg_level_csr(eqs_ctx* ctx, int level, int which, int* dims, int* row_ptr, int* col_idx, double* values);

/* ----------------------------------------------------------------- operators */
/* MatFreeStiffness::apply (proj/src/matfree.cpp:90-98): y = K(x_state) v, full dof vectors. */
int eqs_kx_apply(eqs_ctx* ctx, const double* x_state, const double* v, double* y);
int eqs_kx_apply_dev(eqs_ctx* ctx, const double* x_state, const double* v, double* y);
/* MatFreeStiffness::residual (proj/src/matfree.cpp:138-143): r = b_mass - (K(x)x)|free. */
int eqs_kx_residual(eqs_ctx* ctx, const double* x_full, const double* b_mass, double* r);
int eqs_kx_residual_dev(eqs_ctx* ctx, const double* x_full, const double* b_mass, double* r);
/* FemSystem::mass_apply (proj/src/fem_system.cpp:101): y = M_II v. */
int eqs_mass_apply(eqs_ctx* ctx, const double* v, double* y);
/* pcg_solve(CsrOperator(M_II), mass preconditioner, b, x0, tol, max_iter)
 * (proj/src/pcg.cpp:9-72). x0 may be NULL (zero start). Non-convergence is
 * reported in res->converged, not as an error (test_solvers.cpp:108-116). */
int eqs_mass_solve(eqs_ctx* ctx, const double* b, const double* x0, double tol, int max_iter, double* x,
                   eqs_pcg_result* res);
/* Multiple-right-hand-side sequence (no reference
 * counterpart beyond the eval_rhs solve path): the k right-hand sides
 * B[k][n_free] are uploaded, then solved in order on the device with the
 * context's start-vector estimator (x0 = estimator.next(b), PCG, feedback),
 * exactly as eval_rhs does (fem_system.cpp:80-90). X[k][n_free] may be NULL;
 * iterations[k] receives the PCG iterations; *device_ms the device time of
 * the k solves. Non-convergence is a NumericalError. */
int eqs_mass_solve_sequence(eqs_ctx* ctx, const double* B, int k, double tol, int max_iter, double* X,
                            int* iterations, double* device_ms);

/* ----------------------------------------------------------------- OdeSystem (proj/include/eqs/ode_system.hpp:45-73) */
/* FemSystem::eval_residual (fem_system.cpp:62-67). */
/* StartVectorEstimator::next(M_II, b) / feedback(x, iterations) / current_rank()
 * (proj/include/eqs/start_vector.hpp:52-66, proj/src/start_vector.cpp:84-187) on
 * the context's own estimator. Host vectors of n_free; x0 is zero when the
 * estimator has no basis yet. Single-rank contexts. */
int eqs_estimator_next(eqs_ctx* ctx, const double* b, double* x0, int* rank);
int eqs_estimator_feedback(eqs_ctx* ctx, const double* x, int iterations);

int eqs_eval_residual(eqs_ctx* ctx, double t, const double* x, double* r);
/* FemSystem::eval_rhs (fem_system.cpp:69-99): f = M^-1 (b - K(x)x); throws
 * NumericalError (returns EQS_ERR_NUMERICAL) when the mass solve fails. */
int eqs_eval_rhs(eqs_ctx* ctx, double t, const double* x, double* f, eqs_pcg_result* res);
/* FemSystem::apply_minv_stiffness (fem_system.cpp:103-122). */
int eqs_apply_minv_stiffness(eqs_ctx* ctx, double t, const double* x_state, const double* v, double* y);
/* FemSystem::lift_full (fem_system.cpp:56-60). */
int eqs_lift_full(eqs_ctx* ctx, double t, const double* x_free, double* x_full);
int eqs_get_stats(eqs_ctx* ctx, eqs_solve_stats* out);

/* ----------------------------------------------------------------- integrators (device-resident state) */
/* IntegratorState (integrators.hpp:23-29): upload/download of the resident state. */
int eqs_set_state(eqs_ctx* ctx, double t, const double* x, double dt);
int eqs_get_state(eqs_ctx* ctx, double* x, eqs_state_info* info);
/* RhoCache of the resident state (integrators.hpp:17-21): pin/inspect the cached rho. */
int eqs_set_rho(eqs_ctx* ctx, double value, int valid, long age);
/* estimate_spectral_radius (proj/src/integrators.cpp:49-75) at (t, x) of the resident state. */
int eqs_spectral_radius(eqs_ctx* ctx, double* rho);
/* rkc_step (proj/src/integrators.cpp:177-225) on the resident state. */
int eqs_rkc_step(eqs_ctx* ctx, const eqs_rkc_options* opts, eqs_step_attempt* att);
/* rkc_advance_fixed (proj/src/integrators.cpp:227-235), nsteps times. */
int eqs_rkc_advance_fixed(eqs_ctx* ctx, double dt, int s, int nsteps);
/* euler_step (proj/src/integrators.cpp:33-47). */
int eqs_euler_step(eqs_ctx* ctx, double dt, eqs_step_attempt* att);
/* sdirk_step / sdirk_advance_fixed (proj/src/integrators.cpp:297-341): stiffly
 * accurate SDIRK3(2), Newton per stage with M + gamma dt K(z) assembled on the
 * device every iteration (fem_system.cpp:124-145; Jacobi-preconditioned PCG,
 * DESIGN.md §4). Single-rank contexts. advance_fixed returns NumericalError
 * when a stage's Newton iteration fails. */
int eqs_sdirk_step(eqs_ctx* ctx, const eqs_sdirk_options* opts, eqs_step_attempt* att);
/* OdeSystem::shifted_solve (ode_system.hpp:63-68, fem_system.cpp:124-145):
 * (M_II + gdt K_II(lift(t, z))) delta = rhs, host vectors of n_free; the
 * preconditioner is refreshed when refresh_precond != 0 or on first use. */
int eqs_shifted_solve(eqs_ctx* ctx, double t, const double* z, double gdt, const double* rhs, double* delta,
                      int refresh_precond);
int eqs_sdirk_advance_fixed(eqs_ctx* ctx, double dt, int nsteps, const eqs_sdirk_options* opts);

/* ----------------------------------------------------------------- scenario (proj/src/scenario.cpp:217-383) */
typedef struct {
  int exit_code;             /* 0 ok, 1 config error, 2 solver failure */
  long accepted, rejected, stages;
  eqs_solve_stats stats;
  double final_t;
  double wall_time;
  long n_free;
} eqs_run_result;
/* run_scenario: writes metrics/probe/solves CSVs into out_dir per the config's
 * output block. x_final (capacity x_cap) receives the final free vector. */
int eqs_run_scenario(const char* json_text, const char* out_dir, int device, eqs_run_result* res, double* x_final,
                     long x_cap);

/* ----------------------------------------------------------------- instrumentation */
int eqs_timing_enable(eqs_ctx* ctx, int on);
int eqs_timing_get(eqs_ctx* ctx, eqs_timing* out);
int eqs_timing_reset(eqs_ctx* ctx);
/* Tuning knobs (not in the reference): 0 = stiffness mode (0 gather, 1 coloured),
 * 1 = fine-level Chebyshev degree (1 or 2), 2 = Chebyshev eigenvalue ratio,
 * 3 = coarse-level Chebyshev degree (1 or 2), 4 = V-cycle matrix values
 * (0 fp64, 1 fp32, 2 bf16; default 2), 5/6/7 = CSR threads per row of levels
 * 0/1/2, 8 = CUDA graphs (0/1), 9 = incremental SPE (0/1), 10 = SELL-16
 * operators (0/1; default 1), 11 = fp32 V-cycle vectors (0/1; default 1),
 * 12 = start-vector estimator (0 zero, 1 previous, 2 spe, 3 pod_fixed, 4 pod_rolling;
 * resets its history), 15/16/17/18 = POD snapshots / rank / capacity / threshold
 * (estimator config keys "snapshots", "rank", "capacity", "threshold"; take effect
 * at the next reset), 19 = stencil-coded fine-level V-cycle operator (0/1; default 1
 * where the rows share at most 255 column-offset patterns), 20 = graph-resident
 * PCG iteration loop (0/1; default 1: iterations 2.. run inside one CUDA graph
 * with a device-side stopping rule, no host round trip per iteration),
 * 21 = programmatic dependent launch of the row/vector kernels (0/1; default 1;
 * process-wide), 22 = the graph-resident PCG loop on multi-rank NCCL contexts
 * too (0/1; default 0: halo and allreduce calls captured into the loop body),
 * 23 = symmetric half storage of the stencil-coded fine operator (0/1; only when
 * the context was created with EQS_SELL_SH=1 in the environment and the operator
 * is single-rank, bitwise symmetric and 16 slots wide: rows store their upper
 * slots only and read lower values from the mirror rows; bit-identical products,
 * about half the matrix bytes, but slower on B200: DESIGN.md §8),
 * 13 = smoother polynomial (0 first-kind Chebyshev, 1 fourth-kind, 2 fourth-kind
 * with optimised weights), 14 = lambda_max safety factor (default 1.1),
 * 24 = per-class timing keeps the graph-resident PCG loop (0/1; default 0: the
 * whole loop is timed as class 6 instead of classes 1 and 2), 26 = SDIRK shifted
 * solves preconditioned by an SA-AMG of the shifted matrix rebuilt on the device
 * at every preconditioner refresh (1, default, with solver.preconditioner amg) or
 * by Jacobi (0), 27 = SDIRK shifted AMG solves through the graph-resident PCG
 * loop with an fp32 V-cycle (1, default) or the host-driven fp64 loop (0),
 * 28 = W-cycle (two coarse-grid corrections) on levels >= value (0 = V-cycle,
 * the default; slower at C3).
 * 29 = fine-level pre-smoother degree (0 = option 1's degree, the default;
 *      1 = one fused Jacobi-type pass; the cycle is then not symmetric).
 * 30 = row-sum correction of the stencil-coded bf16 fine-level V-cycle
 *      operator (1, the default: the bf16 rounding error of each row sum is
 *      stored in the row's first padded slot on the diagonal; 0 = plain bf16).
 * The PCG operator and vectors are fp64 in every setting. */
int eqs_set_option(eqs_ctx* ctx, int key, double value);
/* The CUDA stream (cudaStream_t) every device call of this context runs on. */
int eqs_get_stream(eqs_ctx* ctx, void** stream);
/* Kernels launched by this library since load (process-wide). */
long eqs_launch_count(void);
/* test_helpers.hpp:15-21 random_vec: mt19937(seed) + uniform[-1,1) (synthetic inputs). */
int eqs_random_vec(int n, unsigned seed, double* out);

#ifdef __cplusplus
}
#endif
#endif /* EQS_B200_H */
