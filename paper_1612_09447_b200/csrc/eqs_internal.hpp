// Host-side types of the B200 EQS hot path. The host owns setup and control
// (mesh, dofs, colouring, mass assembly, AMG hierarchy, RKC control), the
// device owns every n-length vector and matrix.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace eqsb {

// proj/include/eqs/types.hpp:12
inline constexpr double kVacuumPermittivity = 8.8541878128e-12;

// proj/include/eqs/errors.hpp:10-37 — same taxonomy, mapped to C-ABI codes.
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GeometryError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericalError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

// proj/include/eqs/mesh.hpp:13-31 in SoA-friendly flat arrays.
struct Mesh {
  int n_nodes = 0, n_tets = 0;
  std::vector<double> nodes;   // [n_nodes][3]
  std::vector<int> tets;       // [n_tets][4]
  std::vector<int> region;     // [n_tets]
  std::map<std::string, std::vector<int>> boundary_sets;
  void finalize();             // proj/src/mesh.cpp:57-91
};
struct LayerSpec {
  std::vector<double> z_planes;
  std::vector<int> regions = {1};
};
Mesh generate_box_mesh(int nx, int ny, int nz, double lx, double ly, double lz, const LayerSpec& layers);
void jitter_box_mesh(Mesh& m, int nx, int ny, int nz, double lx, double ly, double lz, double amplitude,
                     unsigned seed);
Mesh load_msh(const std::string& path);

inline constexpr int kTetEdgeVertices[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

// proj/include/eqs/dofmap.hpp:22-44
struct Dofs {
  int order = 1, n_dofs = 0, n_local = 4;
  std::vector<int> element_dofs;  // [n_tets][n_local]
  std::vector<int> free_dofs, fixed_dofs, fixed_set;
  std::vector<std::string> set_names;
  int n_free() const { return (int)free_dofs.size(); }
  int n_fixed() const { return (int)fixed_dofs.size(); }
};
Dofs build_dof_map(const Mesh& mesh, int order, const std::vector<std::string>& dirichlet_sets);

// proj/include/eqs/materials.hpp:11-33
struct Material {
  int kind = 0;  // 0 constant, 1 microvaristor
  double eps_r = 1.0, kappa = 0.0, kappa_lo = 0, kappa_hi = 0, e_switch = 0, width = 0;
  double permittivity() const { return eps_r * kVacuumPermittivity; }
  void validate() const;  // proj/src/materials.cpp:10-23
};

// proj/include/eqs/excitation.hpp:13-27
struct Waveform {
  int kind = 2;  // 0 sinusoid, 1 ramp, 2 constant
  double amplitude = 0, frequency = 50, phase = 0, rise_time = 1, value = 0;
  double value_at(double t) const;  // proj/src/excitation.cpp:10-16
  double rate_at(double t) const;   // proj/src/excitation.cpp:18-26
};

struct SolverParams {
  int precond = 2;  // 0 jacobi, 1 ssor, 2 amg
  double rel_tol = 1e-12;
  int max_iter = 500;
  double rho_solve_tol = 1e-4;
  double amg_theta = 0.08, amg_omega = 4.0 / 3.0;
  int amg_sweeps = 1, amg_max_levels = 10, amg_coarse_limit = 64;
  double amg_coarse_filter = 0.0025;  // additive: V-cycle coarse-operator filter (0 = off)
  std::vector<double> amg_vcycle_truncate = {0.1, 0.15, 0.03};  // additive: per-level V-cycle prolongator
                                                                // truncation thresholds ({} / 0 = off)
  int amg_replicate_rows = 32768;     // additive: coarse levels up to this size are replicated on every rank
  int amg_dense_coarse = 512;         // additive: the device V-cycle solves the first coarse level with at most
                                      // this many rows directly (dense inverse); <= 0: recurse to the
                                      // hierarchy's coarsest (configs default 512)
  int estimator_mode = 0;  // 0 zero, 1 previous, 2 spe, 3 pod_fixed, 4 pod_rolling
  int spe_window = 8;
  int pod_snapshots = 40;    // start_vector.hpp:31-35
  int pod_rank = 10;
  int pod_capacity = 20;
  double pod_threshold = 0;  // <= 0: 1.25 x the running median of the iteration counts
  double mgs_drop_tol = 1e-8;
};

struct HostCsr {
  int n_rows = 0, n_cols = 0;
  std::vector<int> row_ptr, col_idx;
  std::vector<double> values;
  long nnz() const { return (long)col_idx.size(); }
};

// Everything the reference FemSystem references (fem_system.hpp:59-62), owned.
struct Problem {
  Mesh mesh;
  Dofs dm;
  std::map<int, Material> materials;
  std::vector<Waveform> set_waveforms;  // by Dofs::set_names index
  SolverParams solver;
};

// ----------------------------------------------------------------- setup
// color_elements (proj/src/matfree.cpp:11-38), bit-exact, returns colour per tet.
std::vector<int> color_elements(const Dofs& dm, int n_tets, int* n_colors);
// the same colouring on a GPU (k_setup.cu: topological waves over the earlier-neighbour DAG)
std::vector<int> dev_color_elements(const Dofs& dm, int n_tets, int* n_colors, int device, int* waves = nullptr);
// owner rank of every free dof from its partition-axis coordinate: stable radix
// sort on the GPU, contiguous equal chunks (partition_free_dofs, k_setup.cu)
std::vector<int> dev_partition_owner(const std::vector<double>& key, int nranks, int device);
// assemble_mass (proj/src/assembly.cpp:130-176) + split_dirichlet (:188-193).
void assemble_mass_blocks(const Problem& p, HostCsr& m_ii, HostCsr& m_ib);

struct AmgHostLevel {
  HostCsr A, P, R;
  std::vector<int> aggregates;
  double lambda_max_scaled = 0;  // lambda_max(D^-1 A) estimate (power iteration)
};
struct AmgHierarchy {
  std::vector<AmgHostLevel> levels;
  std::vector<double> coarse_inverse;  // dense inverse of the coarsest A (row-major)
  int coarse_n = 0;
};
// AmgPreconditioner ctor (proj/src/amg.cpp:90-143), bit-exact aggregation and
// Galerkin products (deterministic row-parallel SpGEMM). device >= 0: the
// smoothed prolongator and the Galerkin products run on that GPU
// (spgemm_device), bit-identical to the host products.
AmgHierarchy build_amg(const HostCsr& a, const SolverParams& sp, int device = -1);
// C = A B on the GPU with the host product's per-row arithmetic order
// (k_spgemm.cu). With diag, A is replaced by I - omega D^-1 A on the fly.
// A_{k+1} = R_k (A_k P_k) for k = 0.. with A_0 = fine, operands resident on the GPU
std::vector<HostCsr> galerkin_chain_device(const HostCsr& fine, const std::vector<const HostCsr*>& p,
                                           const std::vector<const HostCsr*>& r, int device);
HostCsr spgemm_device(const HostCsr& a, const HostCsr& b, int device, const std::vector<double>* diag = nullptr,
                      double omega = 0.0, long long batch_products = 1ll << 28);
// Device-resident Galerkin chain of build_amg: the fine operator and P stay on
// the GPU; only P (for R = P^T on the host) and the coarse operator come back.
class AmgDeviceBuilder {
 public:
  explicit AmgDeviceBuilder(int device);
  ~AmgDeviceBuilder();
  // P = (I - omega D^-1 A) P_tent (fine is uploaded on the first call only)
  HostCsr prolongator(const HostCsr& fine, const HostCsr& p_tent, const std::vector<double>& d, double omega,
                      long long batch);
  // R (A P) with A and P resident; the result becomes the next fine operator
  HostCsr galerkin(const HostCsr& r, long long batch);
  // One whole level of build_amg on the device (amg.cpp:99-137): strength
  // graph + aggregation, P_tent, lambda_max, smoothed P, R = P^T, R (A P) and
  // the diagonal check, all bit-identical to the host build. The fine
  // operator is uploaded on the first call and the coarse one stays resident.
  // Returns false when coarsening stalls (n_agg >= rows).
  bool next_level(const HostCsr& fine, const SolverParams& sp, long long batch, AmgHostLevel& lv, HostCsr& coarse);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};
// explicit inverse (row-major) of a symmetric matrix through the pivoted LDLT
// below (the coarsest-level solve, amg.cpp:140); threaded for the larger
// dense coarse levels of the device V-cycle (SolverParams::amg_dense_coarse)
std::vector<double> dense_inverse(const HostCsr& a);
// host CSR product / transpose of build_amg (proj/src/csr.cpp:133-166, 52-70)
HostCsr csr_multiply(const HostCsr& a, const HostCsr& b);
HostCsr csr_transposed(const HostCsr& a);
// V-cycle operator of a coarse level: entries with |a_ij| < eps sqrt(|a_ii a_jj|)
// dropped and lumped onto the diagonal (row sums kept). The hierarchy itself
// (P, R, Galerkin A_l) is untouched; only the smoother/residual operator of
// levels >= 1 uses this.
HostCsr filter_lumped(const HostCsr& a, double eps);
double estimate_lambda_max_scaled(const HostCsr& a, int iters, unsigned seed);
// Eigen 3.4 v.norm() in its SSE2 reduction order (host_setup.cpp)
double seq_norm(const std::vector<double>& v);

// symmetric LDLT with diagonal pivoting (Eigen::LDLT semantics)
struct DenseLdlt {
  int n = 0;
  std::vector<double> lmat, d;
  std::vector<int> perm;
  bool ok = false;
  void compute(const std::vector<double>& a, int n_);
  void solve(const double* b, double* x) const;
};

// ----------------------------------------------------------------- RKC
// RkcCoefficients::compute (proj/src/integrators.cpp:86-133)
struct RkcCoefficients {
  int s = 0;
  double w0 = 0, w1 = 0, mu1_tilde = 0;
  std::vector<double> t_w0, tp_w0, tpp_w0, b, a, c, mu, nu, mu_tilde, gamma_tilde;
  static RkcCoefficients compute(int s);
  static double stability_boundary(int s) { return 0.653 * (s * s - 1.0); }
};

// ----------------------------------------------------------------- config
struct SimConfig {
  std::string name = "scenario";
  bool has_file = false;
  std::string mesh_file;
  int nx = 1, ny = 1, nz = 1;
  double lx = 1, ly = 1, lz = 1;
  LayerSpec layers;
  double jitter = 0.0;
  unsigned jitter_seed = 1612;
  int order = 1;
  std::map<int, Material> materials;
  std::map<std::string, Waveform> excitations;
  int integrator = 1;  // 0 euler, 1 rkc, 2 sdirk32 (rejected on GPU)
  double tolerance = 1e-2, atol = -1, t_end = 0.02, dt0 = 1e-5;
  int max_stages = 200;
  long max_steps = -1;  // additive: bounded runs
  SolverParams solver;
  std::vector<std::array<double, 3>> probes;
  std::string metrics_csv = "metrics.csv", probe_csv = "probe.csv", solves_csv, vtk_prefix;
  int vtk_every = 0;
  bool vtk_binary = false;  // additive: legacy binary VTK instead of ASCII
  int workers = 1;
  double effective_atol() const;  // proj/src/scenario.cpp:90-100
};
SimConfig parse_config(const std::string& json_text);  // proj/src/scenario.cpp:110-211
Problem build_problem(const SimConfig& c);

}  // namespace eqsb
