// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Plain C++20 CPU restatement of the reference `eqsim` hot path
// (/root/reference/proj, arXiv 1612.09447), used as the parity checker for the
// B200 product path. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it. The product library
// (paper_1612_09447_b200/libeqs_b200.so) never links or calls anything here.
//
// Every function cites the reference file:line it restates. Eigen is replaced
// by std::vector loops with the same per-element operation order; reductions
// are sequential (Eigen's packet reductions differ from them only in the last
// ulps, which no reference test pins — SURVEY.md §8c).
//
// Parity pin: the oracle is checked against the reference's own known-answer
// tests: reference-tet P1 matrix, P2 moment oracle, kappa
// midpoint, fused == assembled, ones-vector, DC residual, PCG semantics, AMG
// Galerkin/SPD/reuse, RKC amplification/order/stability, spectral-radius
// bracket, capacitive tracking, RC divider. See tests/test_oracle_*.py.
#pragma once

#include <array>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

namespace ora {

// Sum of f(0..n-1) in the order of Eigen 3.4's LinearVectorizedTraversal
// redux with SSE2 packets of 2 doubles (the default x86-64 build of the
// reference, proj/CMakeLists.txt: Release, no -march): two packet
// accumulators over blocks of 4, then the leftover packet, the horizontal
// add and the scalar tail. Used for every Eigen dot/norm/squaredNorm the
// reference calls (pcg.cpp, amg.cpp:28-45, integrators.cpp:56-65,
// start_vector.cpp) so the restatement matches the compiled reference
// (oracle/_ref, built against the same order in oracle/ref_shim/Eigen/Core)
// bit for bit where it matters: the AMG hierarchy depends on omega through
// borderline strength decisions.
template <class F>
inline double eigen_redux_sum(size_t n, F&& c) {
  if (n == 0) return 0.0;
  const size_t a2 = n / 4 * 4, a1 = n / 2 * 2;
  if (a1 == 0) return c(0);
  double p00 = c(0), p01 = c(1);
  if (a1 > 2) {
    double p10 = c(2), p11 = c(3);
    for (size_t i = 4; i < a2; i += 4) {
      p00 = p00 + c(i);
      p01 = p01 + c(i + 1);
      p10 = p10 + c(i + 2);
      p11 = p11 + c(i + 3);
    }
    p00 = p00 + p10;
    p01 = p01 + p11;
    if (a1 > a2) {
      p00 = p00 + c(a2);
      p01 = p01 + c(a2 + 1);
    }
  }
  double r = p00 + p01;
  for (size_t i = a1; i < n; ++i) r = r + c(i);
  return r;
}


using Vec = std::vector<double>;

// proj/include/eqs/types.hpp:12
inline constexpr double vacuum_permittivity = 8.8541878128e-12;

// proj/include/eqs/errors.hpp:10-37
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GeometryError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericalError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- mesh
// proj/include/eqs/mesh.hpp:13-31
struct TetMesh {
  std::vector<std::array<double, 3>> nodes;
  std::vector<std::array<int, 4>> tets;
  std::vector<int> region_id;
  std::map<std::string, std::vector<int>> boundary_sets;
  int n_nodes() const { return (int)nodes.size(); }
  int n_tets() const { return (int)tets.size(); }
  double tet_volume(int t) const;
  std::array<double, 3> tet_centroid(int t) const;
  void finalize();
};
struct LayerSpec {
  std::vector<double> z_planes;
  std::vector<int> regions = {1};
};
TetMesh generate_box_mesh(int nx, int ny, int nz, double lx, double ly, double lz,
                          const LayerSpec& layers = {});
// Additive (not in the reference): deterministic interior-node jitter used for
// the "bushing-like" benchmark meshes. Applied identically by
// the product's host mesh generator.
void jitter_box_mesh(TetMesh& m, int nx, int ny, int nz, double lx, double ly, double lz,
                     double amplitude, unsigned seed);
TetMesh load_msh(const std::string& path);

// ---------------------------------------------------------------- dofmap
inline constexpr int kTetEdgeVertices[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
// proj/include/eqs/dofmap.hpp:22-44
struct DofMap {
  int order = 1;
  int n_dofs = 0;
  int n_local = 4;
  std::vector<std::array<double, 3>> dof_coords;
  std::vector<std::array<int, 10>> element_dofs;
  std::vector<int> free_dofs, fixed_dofs, free_index, fixed_index, fixed_set;
  std::vector<std::string> set_names;
  int n_free() const { return (int)free_dofs.size(); }
  int n_fixed() const { return (int)fixed_dofs.size(); }
  void lift(const Vec& x_free, const Vec& x_fixed, Vec& x_full) const;
  void restrict_free(const Vec& x_full, Vec& x_free) const;
};
DofMap build_dof_map(const TetMesh& mesh, int order, const std::vector<std::string>& dirichlet_sets);

// ---------------------------------------------------------------- materials
struct ConstantConductivity { double kappa; };
struct MicrovaristorConductivity { double kappa_lo, kappa_hi, e_switch, width; };
struct MaterialModel {
  double eps_r = 1.0;
  std::variant<ConstantConductivity, MicrovaristorConductivity> conductivity =
      ConstantConductivity{0.0};
  double permittivity() const { return eps_r * vacuum_permittivity; }
  void validate() const;
};
double kappa_of_e(const MaterialModel& m, double e_mag);
using MaterialTable = std::map<int, MaterialModel>;

// ---------------------------------------------------------------- excitation
struct SinusoidWaveform { double amplitude = 0, frequency = 50, phase = 0; };
struct RampWaveform { double amplitude = 0, rise_time = 1; };
struct ConstantWaveform { double value = 0; };
using Waveform = std::variant<SinusoidWaveform, RampWaveform, ConstantWaveform>;
double waveform_value(const Waveform& w, double t);
double waveform_rate(const Waveform& w, double t);
struct BoundaryExcitation {
  std::map<std::string, Waveform> per_set;
  double value(const std::string& set, double t) const;
  double rate(const std::string& set, double t) const;
  Vec boundary_values(const DofMap& dm, double t) const;
  Vec boundary_rates(const DofMap& dm, double t) const;
};

// ---------------------------------------------------------------- csr
// proj/include/eqs/csr.hpp:13-46
struct CsrMatrix {
  int n_rows = 0, n_cols = 0;
  std::vector<int> row_ptr, col_idx;
  std::vector<double> values;
  int nnz() const { return (int)col_idx.size(); }
  void apply(const Vec& x, Vec& y) const;
  Vec apply(const Vec& x) const { Vec y; apply(x, y); return y; }
  double coeff(int i, int j) const;
  double* find(int i, int j);
  Vec diagonal() const;
  CsrMatrix transposed() const;
  double symmetry_error() const;
  static CsrMatrix from_pattern(std::vector<std::vector<int>> row_cols);
  static CsrMatrix from_triplets(int n_rows, int n_cols, std::vector<std::array<int, 2>> pattern,
                                 const std::vector<double>& vals);
};
CsrMatrix multiply(const CsrMatrix& a, const CsrMatrix& b);
CsrMatrix extract_block(const CsrMatrix& a, const std::vector<int>& rows, const std::vector<int>& cols);
CsrMatrix add(double alpha, const CsrMatrix& a, double beta, const CsrMatrix& b);  // csr.cpp:168-195

// ---------------------------------------------------------------- assembly
struct TetGeometry {
  std::array<std::array<double, 3>, 4> grad_lambda;
  double volume = 0;
};
TetGeometry tet_geometry(const std::array<std::array<double, 3>, 4>& p);
int quadrature_size(int order);
double quadrature_weight(const TetGeometry& geo, int order, int q);
void shape_gradients(const TetGeometry& geo, int order, int q, std::array<std::array<double, 3>, 10>& grads);
double gradient_magnitude(const TetGeometry& geo, int order, int q, const double* x_loc);
void element_laplacian(const TetGeometry& geo, int order, const double* coeff_at_qp, double S[10][10]);
CsrMatrix assemble_mass(const TetMesh& mesh, const DofMap& dm, const MaterialTable& materials);
CsrMatrix assemble_stiffness(const TetMesh& mesh, const DofMap& dm, const MaterialTable& materials,
                             const Vec& x_full);
struct DirichletBlocks { CsrMatrix AII, AIB; };
DirichletBlocks split_dirichlet(const CsrMatrix& a, const DofMap& dm);

// ---------------------------------------------------------------- matfree
std::vector<std::vector<int>> color_elements(const DofMap& dm, int n_tets);
class MatFreeStiffness {
 public:
  MatFreeStiffness(const TetMesh& mesh, const DofMap& dm, const MaterialTable& materials, int workers = 1);
  void apply(const Vec& x_state, const Vec& v, Vec& y) const;
  void residual(const Vec& x_full, const Vec& b_mass, Vec& r) const;
  int n_colors() const { return (int)color_batches_.size(); }
  const std::vector<std::vector<int>>& color_batches() const { return color_batches_; }
  long applies() const { return applies_; }

 private:
  const TetMesh& mesh_;
  const DofMap& dm_;
  int workers_;
  std::vector<const MaterialModel*> material_of_tet_;
  std::vector<std::vector<int>> color_batches_;
  mutable long applies_ = 0;
};

// ---------------------------------------------------------------- solvers
class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  virtual int rows() const = 0;
  virtual void apply(const Vec& x, Vec& y) const = 0;
};
class CsrOperator final : public LinearOperator {
 public:
  explicit CsrOperator(const CsrMatrix& a) : a_(a) {}
  int rows() const override { return a_.n_rows; }
  void apply(const Vec& x, Vec& y) const override { a_.apply(x, y); }
 private:
  const CsrMatrix& a_;
};
class IdentityOperator final : public LinearOperator {
 public:
  explicit IdentityOperator(int n) : n_(n) {}
  int rows() const override { return n_; }
  void apply(const Vec& x, Vec& y) const override { y = x; }
 private:
  int n_;
};
struct PcgResult {
  Vec x;
  int iterations = 0;
  double rel_residual = 0, initial_rel_residual = 0;
  bool converged = false;
};
PcgResult pcg_solve(const LinearOperator& a, const LinearOperator& precond, const Vec& b,
                    const Vec& x0, double rel_tol, int max_iter);

std::vector<int> diagonal_positions(const CsrMatrix& a);
class JacobiPreconditioner final : public LinearOperator {
 public:
  explicit JacobiPreconditioner(const CsrMatrix& a);
  int rows() const override { return (int)inv_diag_.size(); }
  void apply(const Vec& r, Vec& z) const override;
 private:
  Vec inv_diag_;
};
class SsorPreconditioner final : public LinearOperator {
 public:
  explicit SsorPreconditioner(const CsrMatrix& a);
  int rows() const override { return a_.n_rows; }
  void apply(const Vec& r, Vec& z) const override;
 private:
  CsrMatrix a_;
  std::vector<int> diag_pos_;
};
void gauss_seidel_forward(const CsrMatrix& a, const std::vector<int>& diag_pos, const Vec& b, Vec& x);
void gauss_seidel_backward(const CsrMatrix& a, const std::vector<int>& diag_pos, const Vec& b, Vec& x);

// dense symmetric LDLT with diagonal pivoting (restates Eigen::LDLT usage at
// proj/src/amg.cpp:140 and proj/src/start_vector.cpp:42-48)
struct DenseLdlt {
  int n = 0;
  std::vector<double> lmat;       // n*n, unit lower triangle below the diagonal
  std::vector<double> d;          // pivoted diagonal
  std::vector<int> perm;          // transpositions
  bool ok = false;
  void compute(const std::vector<double>& a, int n_);
  void solve(const double* b, double* x) const;
};

struct AmgParams {
  double strength_threshold = 0.08;
  double prolongation_omega = 4.0 / 3.0;
  int smoother_sweeps = 1;
  int max_levels = 10;
  int coarse_limit = 64;
};
struct AmgLevel {
  CsrMatrix A;
  std::vector<int> diag_pos;
  CsrMatrix P, R;
  std::vector<int> aggregates;  // aggregate id per row (empty on the coarsest level)
};
std::vector<int> aggregate(const CsrMatrix& a, double theta);
class AmgPreconditioner final : public LinearOperator {
 public:
  AmgPreconditioner(const CsrMatrix& a, const AmgParams& params = {});
  int rows() const override { return levels_.front().A.n_rows; }
  void apply(const Vec& r, Vec& z) const override { vcycle(0, r, z); }
  int n_levels() const { return (int)levels_.size(); }
  const AmgLevel& level(int l) const { return levels_[l]; }
 private:
  void vcycle(size_t l, const Vec& r, Vec& z) const;
  AmgParams params_;
  std::vector<AmgLevel> levels_;
  DenseLdlt coarse_;
};

// ---------------------------------------------------------------- start vectors
// proj/include/eqs/start_vector.hpp:25-38
enum class EstimatorMode { Zero, Previous, Spe, PodFixed, PodRolling };
const char* estimator_mode_name(EstimatorMode m);
struct EstimatorParams {
  EstimatorMode mode = EstimatorMode::Zero;
  int spe_window = 8;
  int pod_snapshots = 40;    // PodFixed: solves collected before the basis is built
  int pod_rank = 10;
  int pod_capacity = 20;     // PodRolling: ring size
  double pod_threshold = 0;  // PodRolling: append when iterations exceed this; <= 0: 1.25x running median
  double mgs_drop_tol = 1e-8;
};
std::vector<Vec> mgs_orthonormalize(const std::vector<Vec>& vectors, double drop_tol);
Vec spe_start(const std::vector<Vec>& v, const CsrMatrix& m, const Vec& b, bool* ok);
// proj/src/start_vector.cpp:64-71: dominant left singular vectors of the
// snapshot matrix (columns), at most `rank`, truncated at sigma <= 1e-12 sigma_0.
// The reference uses Eigen::JacobiSVD; this is a one-sided (Hestenes) Jacobi
// SVD, which yields the same singular values and (up to sign) vectors.
std::vector<Vec> pod_build(const std::vector<Vec>& snapshots, int rank, std::vector<double>* sigma = nullptr);
class StartVectorEstimator {
 public:
  struct Stats {  // start_vector.hpp:45-49
    long svd_count = 0;
    long appends = 0;
    long spe_fallbacks = 0;
  };
  explicit StartVectorEstimator(const EstimatorParams& p) : params_(p) {}
  Vec next(const CsrMatrix& m, const Vec& b);
  void feedback(const Vec& x, int iterations);
  EstimatorMode mode() const { return params_.mode; }
  int current_rank() const { return basis_rank_; }
  const Stats& stats() const { return stats_; }
  long spe_fallbacks = 0;
 private:
  Vec pod_start(const CsrMatrix& m, const Vec& b);
  void factor_reduced(const CsrMatrix& m);
  double rolling_threshold() const;
  EstimatorParams params_;
  Stats stats_;
  std::deque<Vec> history_;
  int basis_rank_ = 0;
  std::vector<Vec> snapshots_;
  int rolling_next_slot_ = 0;
  bool basis_stale_ = false;
  bool fixed_basis_built_ = false;
  std::vector<Vec> basis_;              // POD basis V
  std::vector<double> reduced_inverse_;  // (V'MV)^-1, row-major
  bool reduced_ok_ = false;
  std::vector<int> iteration_history_;
};

// ---------------------------------------------------------------- system
enum class PrecondKind { Jacobi, Ssor, Amg };
struct LinearSolverParams {
  PrecondKind precond = PrecondKind::Amg;
  double rel_tol = 1e-12;
  int max_iter = 500;
  double rho_solve_tol = 1e-4;
  AmgParams amg;
};
struct PhaseTimers { double residual = 0, solve = 0, setup = 0, estimator = 0; };
struct SolveStats {
  long m_solves = 0, pcg_iterations = 0, rho_solves = 0, rho_pcg_iterations = 0;
  long newton_linear_solves = 0, newton_pcg_iterations = 0;
  long precond_setups = 0, assemblies = 0, svd_count = 0;
  PhaseTimers timers;
};
struct SolveRecord {
  double t = 0;
  std::string estimator_mode;
  int estimator_rank = 0, iterations = 0;
  double initial_rel_residual = 0;
};
class OdeSystem {
 public:
  virtual ~OdeSystem() = default;
  virtual int size() const = 0;
  virtual void eval_rhs(double t, const Vec& x, Vec& f) = 0;
  virtual void eval_residual(double t, const Vec& x, Vec& r) = 0;
  virtual void mass_apply(const Vec& v, Vec& y) const = 0;
  virtual void apply_minv_stiffness(double t, const Vec& x_state, const Vec& v, Vec& y) = 0;
  // (M + gdt K(z)) delta = rhs (ode_system.hpp:63-68, the SDIRK Newton matrix)
  virtual void shifted_solve(double t, const Vec& z, double gdt, const Vec& rhs, Vec& delta, bool refresh_precond) = 0;
  SolveStats& stats() { return stats_; }
 protected:
  SolveStats stats_;
};
class FemSystem : public OdeSystem {
 public:
  FemSystem(const TetMesh& mesh, const DofMap& dm, const MaterialTable& materials,
            const BoundaryExcitation& excitation, const LinearSolverParams& solver,
            const EstimatorParams& estimator, int workers = 1);
  int size() const override { return dm_.n_free(); }
  void eval_rhs(double t, const Vec& x, Vec& f) override;
  void eval_residual(double t, const Vec& x, Vec& r) override;
  void mass_apply(const Vec& v, Vec& y) const override { mass_.AII.apply(v, y); }
  void apply_minv_stiffness(double t, const Vec& x_state, const Vec& v, Vec& y) override;
  void shifted_solve(double t, const Vec& z, double gdt, const Vec& rhs, Vec& delta, bool refresh_precond) override;
  Vec lift_full(double t, const Vec& x_free) const;
  const CsrMatrix& mass_free() const { return mass_.AII; }
  const CsrMatrix& mass_ib() const { return mass_.AIB; }
  const MatFreeStiffness& stiffness_operator() const { return matfree_; }
  StartVectorEstimator& estimator() { return estimator_; }
  std::vector<SolveRecord>& solve_records() { return solve_records_; }
  const LinearOperator& mass_preconditioner();
  const AmgPreconditioner* amg() const { return dynamic_cast<const AmgPreconditioner*>(mass_precond_.get()); }

 private:
  const TetMesh& mesh_;
  const DofMap& dm_;
  const MaterialTable& materials_;
  const BoundaryExcitation& excitation_;
  LinearSolverParams solver_;
  StartVectorEstimator estimator_;
  CsrMatrix mass_full_;
  DirichletBlocks mass_;
  MatFreeStiffness matfree_;
  std::unique_ptr<LinearOperator> mass_precond_;
  std::unique_ptr<LinearOperator> shifted_precond_;
  std::unique_ptr<LinearOperator> make_preconditioner(const CsrMatrix& a);
  std::vector<SolveRecord> solve_records_;
};

// ---------------------------------------------------------------- integrators
struct IntegratorStats { long accepted = 0, rejected = 0, stages = 0, newton_iterations = 0; };
struct RhoCache { double value = 0; long age = 0; bool valid = false; };
struct IntegratorState { double t = 0; Vec x; double dt = 0; IntegratorStats stats; RhoCache rho; };
struct StepAttempt {
  double t_start = 0, dt = 0;
  bool accepted = false;
  int stages = 0, newton_iterations = 0;
  double error = 0, rho = 0, dt_next = 0;
};
struct StepControl { double rtol = 1e-2, atol = 1e-8; };
struct ControllerDecision { bool accept = false; double dt_next = 0; };
ControllerDecision step_controller(double err, double dt, int order);
double weighted_rms(const Vec& est, const Vec& x_old, const Vec& x_new, double atol, double rtol);
StepAttempt euler_step(IntegratorState& state, OdeSystem& system, double dt);
double estimate_spectral_radius(OdeSystem& system, double t, const Vec& x);
double spectral_radius_cached(IntegratorState& state, OdeSystem& system, int refresh_every = 25);
struct RkcCoefficients {
  int s = 0;
  double w0 = 0, w1 = 0;
  std::vector<double> t_w0, tp_w0, tpp_w0, b, a, c;
  double mu1_tilde = 0;
  std::vector<double> mu, nu, mu_tilde, gamma_tilde;
  static RkcCoefficients compute(int s);
  double amplification(double z) const;
  static double stability_boundary(int s) { return 0.653 * (s * s - 1.0); }
};
struct RkcOptions { StepControl control; int max_stages = 200; int rho_refresh_every = 25; };
StepAttempt rkc_step(IntegratorState& state, OdeSystem& system, const RkcOptions& options);
void rkc_advance_fixed(IntegratorState& state, OdeSystem& system, double dt, int s);
// proj/include/eqs/integrators.hpp:106-120
struct SdirkOptions { StepControl control; double newton_tol = 1e-8; int max_newton = 25; };
StepAttempt sdirk_step(IntegratorState& state, OdeSystem& system, const SdirkOptions& options);
bool sdirk_advance_fixed(IntegratorState& state, OdeSystem& system, double dt, const SdirkOptions& options);

// ---------------------------------------------------------------- helpers
Vec random_vec(int n, unsigned seed);  // proj/tests/support/test_helpers.hpp:15-21

// ---------------------------------------------------------------- scenario
enum class IntegratorKind { Euler, Rkc, Sdirk32 };
struct BoxSpec {
  int nx = 1, ny = 1, nz = 1;
  double lx = 1, ly = 1, lz = 1;
  LayerSpec layers;
  double jitter = 0.0;     // additive key; 0 = reference generator
  unsigned jitter_seed = 1612;
};
struct SimConfig {
  std::string name = "scenario";
  std::optional<std::string> mesh_file;
  std::optional<BoxSpec> box;
  int order = 1;
  MaterialTable materials;
  std::map<std::string, Waveform> excitations;
  IntegratorKind integrator = IntegratorKind::Rkc;
  double tolerance = 1e-2, atol = -1, t_end = 0.02, dt0 = 1e-5;
  int max_stages = 200;
  LinearSolverParams solver;
  EstimatorParams estimator;
  std::vector<std::array<double, 3>> probes;
  int workers = 1;
  long max_steps = -1;                     // additive: stop after this many attempts (-1 = none)
  std::string metrics_csv = "metrics.csv";
  static SimConfig from_json_text(const std::string& text);
  double effective_atol() const;
};
TetMesh build_mesh(const SimConfig& c);

// proj/include/eqs/probes.hpp:13-21
struct PointLocation {
  int tet = -1;
  std::array<double, 4> lambda = {0, 0, 0, 0};
};
std::optional<PointLocation> locate_point(const TetMesh& mesh, const std::array<double, 3>& p);
double interpolate(const DofMap& dm, const Vec& x_full, const PointLocation& loc);

// proj/include/eqs/metrics.hpp:13-28, scenario.hpp:67-81
struct StepMetrics {
  long step = 0;
  double t = 0, dt = 0;
  std::string method;
  bool accepted = false;
  int stages = 0, newton_iters = 0;
  long m_solves = 0, pcg_iters = 0;
  double rho = 0;
  std::string estimator_mode;
  int estimator_rank = 0;
  double err_est = 0;
  PhaseTimers timers;
};
struct RunResult {
  int exit_code = 0;
  std::string error, name;
  long accepted = 0, rejected = 0, stages = 0;
  SolveStats stats;
  double wall_time = 0;
  std::vector<StepMetrics> steps;
  std::vector<SolveRecord> solves;
  std::vector<std::pair<double, std::vector<double>>> probe_rows;
  Vec final_x_free;
  double final_t = 0;
};
RunResult run_scenario(const SimConfig& config, const std::string& out_dir);
void write_metrics_csv(const std::string& path, const std::vector<StepMetrics>& rows);

}  // namespace ora
