// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/start_vector.cpp (Zero/Previous/SPE), fem_system.cpp and
// integrators.cpp (Euler, RKC, spectral radius).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <map>
#include <random>

#include "oracle.hpp"

namespace ora {

namespace {
double dot(const Vec& a, const Vec& b) {  // Eigen's a.dot(b) summation order
  return eigen_redux_sum(a.size(), [&](size_t i) { return a[i] * b[i]; });
}
double norm(const Vec& a) { return std::sqrt(dot(a, a)); }

class PhaseTimer {  // proj/src/fem_system.cpp:12-23
 public:
  explicit PhaseTimer(double& slot) : slot_(slot), start_(std::chrono::steady_clock::now()) {}
  ~PhaseTimer() { slot_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - start_).count(); }
 private:
  double& slot_;
  std::chrono::steady_clock::time_point start_;
};
}  // namespace

// proj/src/start_vector.cpp:10-28
std::vector<Vec> mgs_orthonormalize(const std::vector<Vec>& vectors, double drop_tol) {
  std::vector<Vec> basis;
  for (const Vec& cand : vectors) {
    const double norm0 = norm(cand);
    if (norm0 == 0.0) continue;
    Vec w = cand;
    for (const Vec& u : basis) {
      const double c = dot(u, w);
      for (size_t i = 0; i < w.size(); ++i) w[i] -= c * u[i];
    }
    if (norm(w) <= drop_tol * norm0) continue;
    for (const Vec& u : basis) {
      const double c = dot(u, w);
      for (size_t i = 0; i < w.size(); ++i) w[i] -= c * u[i];
    }
    const double nrm = norm(w);
    if (nrm <= drop_tol * norm0) continue;
    for (double& e : w) e /= nrm;
    basis.push_back(std::move(w));
  }
  return basis;
}

// proj/src/start_vector.cpp:33-62
Vec spe_start(const std::vector<Vec>& v, const CsrMatrix& m, const Vec& b, bool* ok_out) {
  const int rank = (int)v.size();
  bool ok = rank > 0;
  Vec x0(b.size(), 0.0);
  if (ok) {
    std::vector<Vec> w(rank);
    for (int c = 0; c < rank; ++c) m.apply(v[c], w[c]);
    std::vector<double> g((size_t)rank * rank);
    for (int i = 0; i < rank; ++i)
      for (int j = 0; j < rank; ++j) g[(size_t)i * rank + j] = dot(v[i], w[j]);
    DenseLdlt ldlt;
    ldlt.compute(g, rank);
    double dmax = 0.0, dmin = INFINITY;
    for (double d : ldlt.d) {
      dmax = std::max(dmax, std::abs(d));
      dmin = std::min(dmin, d);
    }
    ok = ldlt.ok && dmax > 0.0 && dmin > 1e-14 * dmax;
    if (ok) {
      // g_inv = ldlt.solve(I); x0 = V (g_inv (V' b))
      std::vector<double> ginv((size_t)rank * rank), e(rank), col(rank);
      for (int c = 0; c < rank; ++c) {
        std::fill(e.begin(), e.end(), 0.0);
        e[c] = 1.0;
        ldlt.solve(e.data(), col.data());
        for (int r = 0; r < rank; ++r) ginv[(size_t)r * rank + c] = col[r];
      }
      std::vector<double> vtb(rank), y(rank, 0.0);
      for (int c = 0; c < rank; ++c) vtb[c] = dot(v[c], b);
      for (int r = 0; r < rank; ++r) {
        double s = 0.0;
        for (int c = 0; c < rank; ++c) s += ginv[(size_t)r * rank + c] * vtb[c];
        y[r] = s;
      }
      for (size_t i = 0; i < b.size(); ++i) {
        double s = 0.0;
        for (int c = 0; c < rank; ++c) s += v[c][i] * y[c];
        x0[i] = s;
      }
    }
  }
  if (ok_out) *ok_out = ok;
  return x0;
}

namespace {
// (V'MV)^-1 (start_vector.cpp:33-50): pivoted LDLT, singular when d_min <= 1e-14 d_max
bool reduced_mass_inverse(const std::vector<Vec>& v, const CsrMatrix& m, std::vector<double>& ginv) {
  const int rank = (int)v.size();
  std::vector<Vec> w(rank);
  for (int c = 0; c < rank; ++c) m.apply(v[c], w[c]);
  std::vector<double> g((size_t)rank * rank);
  for (int i = 0; i < rank; ++i)
    for (int j = 0; j < rank; ++j) g[(size_t)i * rank + j] = dot(v[i], w[j]);
  DenseLdlt ldlt;
  ldlt.compute(g, rank);
  double dmax = 0.0, dmin = INFINITY;
  for (double d : ldlt.d) {
    dmax = std::max(dmax, std::abs(d));
    dmin = std::min(dmin, d);
  }
  if (!(ldlt.ok && dmax > 0.0 && dmin > 1e-14 * dmax)) return false;
  ginv.assign((size_t)rank * rank, 0.0);
  std::vector<double> e(rank), col(rank);
  for (int c = 0; c < rank; ++c) {
    std::fill(e.begin(), e.end(), 0.0);
    e[c] = 1.0;
    ldlt.solve(e.data(), col.data());
    for (int r = 0; r < rank; ++r) ginv[(size_t)r * rank + c] = col[r];
  }
  return true;
}
}  // namespace

// proj/src/start_vector.cpp:64-71 (Eigen::JacobiSVD(snapshots, ComputeThinU)).
// One-sided Jacobi: rotate column pairs until they are mutually orthogonal;
// then sigma_j = |a_j| and u_j = a_j / sigma_j.
std::vector<Vec> pod_build(const std::vector<Vec>& snapshots, int rank, std::vector<double>* sigma_out) {
  std::vector<Vec> a = snapshots;
  const int k = (int)a.size();
  if (k == 0) return {};
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double al = dot(a[p], a[p]), be = dot(a[q], a[q]), ga = dot(a[p], a[q]);
        if (ga == 0.0 || std::abs(ga) <= 1e-15 * std::sqrt(al * be)) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (size_t i = 0; i < a[p].size(); ++i) {
          const double x = a[p][i], y = a[q][i];
          a[p][i] = c * x - s * y;
          a[q][i] = s * x + c * y;
        }
      }
    if (!rotated) break;
  }
  std::vector<std::pair<double, int>> sv(k);
  for (int j = 0; j < k; ++j) sv[j] = {norm(a[j]), j};
  std::stable_sort(sv.begin(), sv.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
  if (sigma_out) {
    sigma_out->clear();
    for (auto& e : sv) sigma_out->push_back(e.first);
  }
  std::vector<Vec> u;
  if (sv[0].first == 0.0) return u;
  for (int j = 0; j < k && j < rank && sv[j].first > 1e-12 * sv[0].first; ++j) {
    Vec c = a[sv[j].second];
    for (double& e : c) e /= sv[j].first;
    u.push_back(std::move(c));
  }
  return u;
}

const char* estimator_mode_name(EstimatorMode m) {
  switch (m) {
    case EstimatorMode::Zero: return "zero";
    case EstimatorMode::Previous: return "previous";
    case EstimatorMode::Spe: return "spe";
    case EstimatorMode::PodFixed: return "pod_fixed";
    case EstimatorMode::PodRolling: return "pod_rolling";
  }
  return "?";
}

// proj/src/start_vector.cpp:111-131
Vec StartVectorEstimator::pod_start(const CsrMatrix& m, const Vec& b) {
  if (params_.mode == EstimatorMode::PodFixed && !fixed_basis_built_ &&
      (int)snapshots_.size() >= params_.pod_snapshots) {
    basis_ = pod_build(snapshots_, params_.pod_rank);
    ++stats_.svd_count;
    fixed_basis_built_ = true;
    factor_reduced(m);
  }
  if (params_.mode == EstimatorMode::PodRolling && basis_stale_ && !snapshots_.empty()) {
    basis_ = pod_build(snapshots_, params_.pod_rank);
    ++stats_.svd_count;
    basis_stale_ = false;
    factor_reduced(m);
  }
  basis_rank_ = (int)basis_.size();
  if (basis_.empty() || !reduced_ok_) return Vec(b.size(), 0.0);
  const int r = (int)basis_.size();
  std::vector<double> vtb(r), y(r, 0.0);
  for (int c = 0; c < r; ++c) vtb[c] = dot(basis_[c], b);
  for (int i = 0; i < r; ++i) {
    double s = 0.0;
    for (int c = 0; c < r; ++c) s += reduced_inverse_[(size_t)i * r + c] * vtb[c];
    y[i] = s;
  }
  Vec x0(b.size(), 0.0);
  for (size_t i = 0; i < b.size(); ++i) {
    double s = 0.0;
    for (int c = 0; c < r; ++c) s += basis_[c][i] * y[c];
    x0[i] = s;
  }
  return x0;
}

// proj/src/start_vector.cpp:133-141
void StartVectorEstimator::factor_reduced(const CsrMatrix& m) {
  reduced_ok_ = !basis_.empty();
  if (!reduced_ok_) return;
  reduced_ok_ = reduced_mass_inverse(basis_, m, reduced_inverse_);
  if (!reduced_ok_) {
    ++stats_.spe_fallbacks;
    ++spe_fallbacks;
    std::fprintf(stderr, "start_vector: singular reduced system, zero start used\n");
  }
}

// proj/src/start_vector.cpp:143-150
double StartVectorEstimator::rolling_threshold() const {
  if (params_.pod_threshold > 0.0) return params_.pod_threshold;
  if (iteration_history_.empty()) return -1.0;
  std::vector<int> h = iteration_history_;
  const size_t mid = h.size() / 2;
  std::nth_element(h.begin(), h.begin() + mid, h.end());
  return 1.25 * (double)h[mid];
}

// proj/src/start_vector.cpp:84-109
Vec StartVectorEstimator::next(const CsrMatrix& m, const Vec& b) {
  switch (params_.mode) {
    case EstimatorMode::Zero: return Vec(b.size(), 0.0);
    case EstimatorMode::Previous: return history_.empty() ? Vec(b.size(), 0.0) : history_.back();
    case EstimatorMode::Spe: {
      if (history_.empty()) return Vec(b.size(), 0.0);
      const std::vector<Vec> v = mgs_orthonormalize({history_.begin(), history_.end()}, params_.mgs_drop_tol);
      basis_rank_ = (int)v.size();
      if (v.empty()) return Vec(b.size(), 0.0);
      bool ok = false;
      Vec x0 = spe_start(v, m, b, &ok);
      if (!ok) {
        ++spe_fallbacks;
        ++stats_.spe_fallbacks;
        std::fprintf(stderr, "start_vector: singular reduced system, zero start used\n");
      }
      return x0;
    }
    case EstimatorMode::PodFixed:
    case EstimatorMode::PodRolling:
      return pod_start(m, b);
  }
  return Vec(b.size(), 0.0);
}
// proj/src/start_vector.cpp:152-187
void StartVectorEstimator::feedback(const Vec& x, int iterations) {
  switch (params_.mode) {
    case EstimatorMode::Zero: break;
    case EstimatorMode::Previous:
      history_.clear();
      history_.push_back(x);
      break;
    case EstimatorMode::Spe:
      history_.push_back(x);
      while ((int)history_.size() > params_.spe_window) history_.pop_front();
      ++stats_.appends;
      break;
    case EstimatorMode::PodFixed:
      if (!fixed_basis_built_ && (int)snapshots_.size() < params_.pod_snapshots) {
        snapshots_.push_back(x);
        ++stats_.appends;
      }
      break;
    case EstimatorMode::PodRolling: {
      const double thr = rolling_threshold();
      if ((double)iterations > thr) {
        if ((int)snapshots_.size() < params_.pod_capacity) {
          snapshots_.push_back(x);
        } else {
          snapshots_[rolling_next_slot_] = x;  // overwrite the oldest
          rolling_next_slot_ = (rolling_next_slot_ + 1) % params_.pod_capacity;
        }
        ++stats_.appends;
        basis_stale_ = true;
      }
      break;
    }
  }
  iteration_history_.push_back(iterations);
}

// proj/src/fem_system.cpp:27-36
FemSystem::FemSystem(const TetMesh& mesh, const DofMap& dm, const MaterialTable& materials,
                     const BoundaryExcitation& excitation, const LinearSolverParams& solver,
                     const EstimatorParams& estimator, int workers)
    : mesh_(mesh), dm_(dm), materials_(materials), excitation_(excitation), solver_(solver),
      estimator_(estimator), matfree_(mesh, dm, materials, workers) {
  PhaseTimer timer(stats_.timers.setup);
  mass_full_ = assemble_mass(mesh_, dm_, materials_);
  ++stats_.assemblies;
  mass_ = split_dirichlet(mass_full_, dm_);
}

// proj/src/fem_system.cpp:38-54
std::unique_ptr<LinearOperator> FemSystem::make_preconditioner(const CsrMatrix& a) {  // fem_system.cpp:38-46
  ++stats_.precond_setups;
  switch (solver_.precond) {
    case PrecondKind::Jacobi: return std::make_unique<JacobiPreconditioner>(a);
    case PrecondKind::Ssor: return std::make_unique<SsorPreconditioner>(a);
    case PrecondKind::Amg: return std::make_unique<AmgPreconditioner>(a, solver_.amg);
  }
  throw ConfigError("unknown preconditioner kind");
}

const LinearOperator& FemSystem::mass_preconditioner() {
  if (!mass_precond_) {
    PhaseTimer timer(stats_.timers.setup);
    mass_precond_ = make_preconditioner(mass_.AII);
  }
  return *mass_precond_;
}

// proj/src/fem_system.cpp:124-145
void FemSystem::shifted_solve(double t, const Vec& z_lin, double gdt, const Vec& rhs, Vec& delta,
                              bool refresh_precond) {
  CsrMatrix shifted;
  {
    PhaseTimer timer(stats_.timers.setup);
    const Vec z_full = lift_full(t, z_lin);
    const CsrMatrix k_full = assemble_stiffness(mesh_, dm_, materials_, z_full);
    ++stats_.assemblies;
    const CsrMatrix k_ii = extract_block(k_full, dm_.free_dofs, dm_.free_dofs);
    shifted = add(1.0, mass_.AII, gdt, k_ii);
    if (refresh_precond || !shifted_precond_) shifted_precond_ = make_preconditioner(shifted);
  }
  PhaseTimer timer(stats_.timers.solve);
  CsrOperator op(shifted);
  PcgResult res = pcg_solve(op, *shifted_precond_, rhs, Vec(), solver_.rel_tol, solver_.max_iter);
  if (!res.converged) throw NumericalError("shifted-system solve failed to converge");
  ++stats_.newton_linear_solves;
  stats_.newton_pcg_iterations += res.iterations;
  delta = std::move(res.x);
}

// proj/src/fem_system.cpp:56-60
Vec FemSystem::lift_full(double t, const Vec& x_free) const {
  Vec full;
  dm_.lift(x_free, excitation_.boundary_values(dm_, t), full);
  return full;
}

// proj/src/fem_system.cpp:62-67
void FemSystem::eval_residual(double t, const Vec& x, Vec& r) {
  PhaseTimer timer(stats_.timers.residual);
  const Vec x_full = lift_full(t, x);
  Vec b_mass = mass_.AIB.apply(excitation_.boundary_rates(dm_, t));
  for (double& e : b_mass) e = -e;
  matfree_.residual(x_full, b_mass, r);
}

// proj/src/fem_system.cpp:69-99
void FemSystem::eval_rhs(double t, const Vec& x, Vec& f) {
  Vec r;
  eval_residual(t, x, r);
  const LinearOperator& precond = mass_preconditioner();
  Vec x0;
  {
    PhaseTimer timer(stats_.timers.estimator);
    x0 = estimator_.next(mass_.AII, r);
  }
  PcgResult res;
  {
    PhaseTimer timer(stats_.timers.solve);
    CsrOperator op(mass_.AII);
    res = pcg_solve(op, precond, r, x0, solver_.rel_tol, solver_.max_iter);
  }
  if (!res.converged)
    throw NumericalError("mass solve failed to converge (relative residual " + std::to_string(res.rel_residual) + ")");
  {
    PhaseTimer timer(stats_.timers.estimator);
    estimator_.feedback(res.x, res.iterations);
  }
  stats_.svd_count = estimator_.stats().svd_count;  // fem_system.cpp:94
  ++stats_.m_solves;
  stats_.pcg_iterations += res.iterations;
  solve_records_.push_back({t, estimator_mode_name(estimator_.mode()), estimator_.current_rank(), res.iterations,
                            res.initial_rel_residual});
  f = std::move(res.x);
}

// proj/src/fem_system.cpp:103-122
void FemSystem::apply_minv_stiffness(double t, const Vec& x_state, const Vec& v, Vec& y) {
  Vec kv_full;
  {
    PhaseTimer timer(stats_.timers.residual);
    const Vec x_full = lift_full(t, x_state);
    Vec v_full;
    dm_.lift(v, Vec(dm_.n_fixed(), 0.0), v_full);
    matfree_.apply(x_full, v_full, kv_full);
  }
  Vec kv;
  dm_.restrict_free(kv_full, kv);
  const LinearOperator& precond = mass_preconditioner();
  PhaseTimer timer(stats_.timers.solve);
  CsrOperator op(mass_.AII);
  PcgResult res = pcg_solve(op, precond, kv, Vec(), solver_.rho_solve_tol, solver_.max_iter);
  ++stats_.rho_solves;
  stats_.rho_pcg_iterations += res.iterations;
  y = std::move(res.x);
}

// ------------------------------------------------------------------ integrators
// proj/src/integrators.cpp:12-18
ControllerDecision step_controller(double err, double dt, int order) {
  if (!std::isfinite(err)) return {false, 0.1 * dt};
  const bool accept = err <= 1.0;
  const double factor = err == 0.0 ? 10.0 : std::clamp(0.8 * std::pow(err, -1.0 / (order + 1)), 0.1, 10.0);
  return {accept, dt * factor};
}
// proj/src/integrators.cpp:20-31
double weighted_rms(const Vec& est, const Vec& x_old, const Vec& x_new, double atol, double rtol) {
  const size_t n = est.size();
  if (n == 0) return 0.0;
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double w = atol + rtol * std::max(std::abs(x_old[i]), std::abs(x_new[i]));
    const double e = est[i] / w;
    acc += e * e;
  }
  return std::sqrt(acc / (double)n);
}
// proj/src/integrators.cpp:33-47
StepAttempt euler_step(IntegratorState& state, OdeSystem& system, double dt) {
  StepAttempt att;
  att.t_start = state.t;
  att.dt = dt;
  Vec f;
  system.eval_rhs(state.t + dt, state.x, f);
  for (size_t i = 0; i < f.size(); ++i) state.x[i] += dt * f[i];
  state.t += dt;
  ++state.stats.accepted;
  ++state.stats.stages;
  att.accepted = true;
  att.stages = 1;
  att.dt_next = dt;
  return att;
}
// proj/src/integrators.cpp:49-75
double estimate_spectral_radius(OdeSystem& system, double t, const Vec& x) {
  const int n = system.size();
  for (int restart = 0; restart < 4; ++restart) {
    std::mt19937 rng(7919u + 31u * (unsigned)restart);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    Vec v(n);
    for (int i = 0; i < n; ++i) v[i] = uni(rng);
    const double nrm = norm(v);
    if (nrm == 0.0) continue;
    for (double& e : v) e /= nrm;
    Vec w;
    double rho = 0.0;
    bool annihilated = false;
    for (int it = 0; it < 15; ++it) {
      system.apply_minv_stiffness(t, x, v, w);
      rho = norm(w);
      if (rho == 0.0) {
        annihilated = true;
        break;
      }
      for (int i = 0; i < n; ++i) v[i] = w[i] / rho;
    }
    if (!annihilated) return 1.2 * rho;
  }
  return 0.0;
}
// proj/src/integrators.cpp:77-84
double spectral_radius_cached(IntegratorState& state, OdeSystem& system, int refresh_every) {
  if (!state.rho.valid || state.rho.age >= refresh_every) {
    state.rho.value = estimate_spectral_radius(system, state.t, state.x);
    state.rho.age = 0;
    state.rho.valid = true;
  }
  return state.rho.value;
}
// proj/src/integrators.cpp:86-133
RkcCoefficients RkcCoefficients::compute(int s) {
  if (s < 2) throw std::invalid_argument("rkc: stage count must be >= 2");
  RkcCoefficients k;
  k.s = s;
  const double eps0 = 2.0 / 13.0;
  k.w0 = 1.0 + eps0 / ((double)s * s);
  k.t_w0.resize(s + 1);
  k.tp_w0.resize(s + 1);
  k.tpp_w0.resize(s + 1);
  k.t_w0[0] = 1.0;
  k.tp_w0[0] = 0.0;
  k.tpp_w0[0] = 0.0;
  k.t_w0[1] = k.w0;
  k.tp_w0[1] = 1.0;
  k.tpp_w0[1] = 0.0;
  for (int j = 2; j <= s; ++j) {
    k.t_w0[j] = 2.0 * k.w0 * k.t_w0[j - 1] - k.t_w0[j - 2];
    k.tp_w0[j] = 2.0 * k.t_w0[j - 1] + 2.0 * k.w0 * k.tp_w0[j - 1] - k.tp_w0[j - 2];
    k.tpp_w0[j] = 4.0 * k.tp_w0[j - 1] + 2.0 * k.w0 * k.tpp_w0[j - 1] - k.tpp_w0[j - 2];
  }
  k.w1 = k.tp_w0[s] / k.tpp_w0[s];
  k.b.resize(s + 1);
  k.a.resize(s + 1);
  k.c.resize(s + 1);
  for (int j = 2; j <= s; ++j) k.b[j] = k.tpp_w0[j] / (k.tp_w0[j] * k.tp_w0[j]);
  k.b[0] = k.b[1] = k.b[2];
  for (int j = 0; j <= s; ++j) k.a[j] = 1.0 - k.b[j] * k.t_w0[j];
  k.c[0] = 0.0;
  for (int j = 2; j <= s; ++j) k.c[j] = (k.tp_w0[s] / k.tpp_w0[s]) * (k.tpp_w0[j] / k.tp_w0[j]);
  k.c[1] = k.c[2] / 4.0;
  k.mu1_tilde = k.b[1] * k.w1;
  k.mu.resize(s + 1);
  k.nu.resize(s + 1);
  k.mu_tilde.resize(s + 1);
  k.gamma_tilde.resize(s + 1);
  for (int j = 2; j <= s; ++j) {
    k.mu[j] = 2.0 * k.b[j] * k.w0 / k.b[j - 1];
    k.nu[j] = -k.b[j] / k.b[j - 2];
    k.mu_tilde[j] = 2.0 * k.b[j] * k.w1 / k.b[j - 1];
    k.gamma_tilde[j] = -k.a[j - 1] * k.mu_tilde[j];
  }
  return k;
}
// proj/src/integrators.cpp:135-144
double RkcCoefficients::amplification(double z) const {
  const double w = w0 + w1 * z;
  double tm2 = 1.0, tm1 = w;
  for (int j = 2; j <= s; ++j) {
    const double t = 2.0 * w * tm1 - tm2;
    tm2 = tm1;
    tm1 = t;
  }
  return a[s] + b[s] * tm1;
}

namespace {
// proj/src/integrators.cpp:148-153
const RkcCoefficients& rkc_coefficients(int s) {
  static std::map<int, RkcCoefficients> cache;
  auto it = cache.find(s);
  if (it == cache.end()) it = cache.emplace(s, RkcCoefficients::compute(s)).first;
  return it->second;
}
// proj/src/integrators.cpp:156-173
void rkc_stages(IntegratorState& state, OdeSystem& system, double dt, const RkcCoefficients& k, Vec& x_new,
                Vec& f0) {
  const double t = state.t;
  const Vec& y0 = state.x;
  const size_t n = y0.size();
  system.eval_rhs(t, y0, f0);
  Vec y_jm2 = y0;
  Vec y_jm1(n);
  const double c1 = k.mu1_tilde * dt;
  for (size_t i = 0; i < n; ++i) y_jm1[i] = y0[i] + c1 * f0[i];
  Vec f, y_j(n);
  for (int j = 2; j <= k.s; ++j) {
    system.eval_rhs(t + k.c[j - 1] * dt, y_jm1, f);
    const double a0 = 1.0 - k.mu[j] - k.nu[j];
    const double mt = k.mu_tilde[j] * dt, gt = k.gamma_tilde[j] * dt;
    for (size_t i = 0; i < n; ++i)
      y_j[i] = a0 * y0[i] + k.mu[j] * y_jm1[i] + k.nu[j] * y_jm2[i] + mt * f[i] + gt * f0[i];
    std::swap(y_jm2, y_jm1);
    std::swap(y_jm1, y_j);
  }
  x_new = std::move(y_jm1);
}
}  // namespace

// proj/src/integrators.cpp:177-225
StepAttempt rkc_step(IntegratorState& state, OdeSystem& system, const RkcOptions& options) {
  StepAttempt att;
  att.t_start = state.t;
  const double rho = spectral_radius_cached(state, system, options.rho_refresh_every);
  att.rho = rho;
  double dt = state.dt;
  int s = 2;
  if (rho > 0.0) {
    s = std::max(2, (int)std::ceil(std::sqrt(dt * rho / 0.653 + 1.0)));
    if (s > options.max_stages) {
      s = options.max_stages;
      dt = 0.95 * RkcCoefficients::stability_boundary(s) / rho;
    }
  }
  att.dt = dt;
  att.stages = s;
  try {
    const RkcCoefficients& k = rkc_coefficients(s);
    Vec x_new, f0, f_new;
    rkc_stages(state, system, dt, k, x_new, f0);
    system.eval_rhs(state.t + dt, x_new, f_new);
    const size_t n = x_new.size();
    Vec est(n);
    const double c = 0.4 * dt;
    for (size_t i = 0; i < n; ++i) est[i] = 0.8 * (state.x[i] - x_new[i]) + c * (f0[i] + f_new[i]);
    att.error = weighted_rms(est, state.x, x_new, options.control.atol, options.control.rtol);
    const ControllerDecision dec = step_controller(att.error, dt, 2);
    bool finite = true;
    for (double v : x_new) finite = finite && std::isfinite(v);
    att.accepted = dec.accept && finite;
    att.dt_next = dec.dt_next;
    state.stats.stages += s;
    if (att.accepted) {
      state.x = std::move(x_new);
      state.t += dt;
      ++state.stats.accepted;
      ++state.rho.age;
    } else {
      ++state.stats.rejected;
      state.rho.valid = false;
    }
  } catch (const NumericalError&) {
    att.accepted = false;
    att.dt_next = 0.5 * dt;
    ++state.stats.rejected;
    state.rho.valid = false;
  }
  state.dt = att.dt_next;
  return att;
}

// proj/src/integrators.cpp:227-235
void rkc_advance_fixed(IntegratorState& state, OdeSystem& system, double dt, int s) {
  const RkcCoefficients& k = rkc_coefficients(s);
  Vec x_new, f0;
  rkc_stages(state, system, dt, k, x_new, f0);
  state.x = std::move(x_new);
  state.t += dt;
  ++state.stats.accepted;
  state.stats.stages += s;
}


// ---------------------------------------------------------------- SDIRK3(2)
// proj/src/integrators.cpp:237-343: stiffly accurate SDIRK3(2), gamma the real
// root of g^3 - 3g^2 + 3g/2 - 1/6; Newton per stage with M + gamma dt K(z).
namespace {
constexpr double kGamma = 0.435866521508459;
constexpr double kSdC[3] = {kGamma, (1.0 + kGamma) / 2.0, 1.0};
constexpr double kB1 = -1.5 * kGamma * kGamma + 4.0 * kGamma - 0.25;
constexpr double kB2 = 1.5 * kGamma * kGamma - 5.0 * kGamma + 1.25;
constexpr double kSdA[3][3] = {{kGamma, 0.0, 0.0}, {(1.0 - kGamma) / 2.0, kGamma, 0.0}, {kB1, kB2, kGamma}};
constexpr double kBhat1 = kGamma / (1.0 - kGamma);
constexpr double kBhat2 = 1.0 - kBhat1;

bool sdirk_stages(IntegratorState& state, OdeSystem& system, double dt, const SdirkOptions& options, Vec& x_new,
                  Vec& est, int& newton_iters) {
  const double t = state.t;
  const double gdt = kGamma * dt;
  const size_t n = state.x.size();
  Vec k[3];
  Vec w, z, g(n), mz, r_ode, delta, zw(n), neg(n);
  newton_iters = 0;
  for (int stage = 0; stage < 3; ++stage) {
    w = state.x;
    for (int j = 0; j < stage; ++j) {
      const double c = dt * kSdA[stage][j];
      for (size_t i = 0; i < n; ++i) w[i] += c * k[j][i];
    }
    const double ts = t + kSdC[stage] * dt;
    z = w;
    double scale = -1.0;
    bool converged = false;
    for (int it = 0;; ++it) {
      system.eval_residual(ts, z, r_ode);
      for (size_t i = 0; i < n; ++i) zw[i] = z[i] - w[i];
      system.mass_apply(zw, mz);
      for (size_t i = 0; i < n; ++i) g[i] = mz[i] - gdt * r_ode[i];
      const double gn = norm(g);
      if (!std::isfinite(gn)) return false;
      if (scale < 0.0) scale = gn;
      if (gn <= options.newton_tol * scale || gn == 0.0) {
        converged = true;
        break;
      }
      if (it >= options.max_newton) break;
      for (size_t i = 0; i < n; ++i) neg[i] = -g[i];
      try {
        system.shifted_solve(ts, z, gdt, neg, delta, stage == 0 && it == 0);
      } catch (const NumericalError&) {
        return false;
      }
      for (size_t i = 0; i < n; ++i) z[i] += delta[i];
      ++newton_iters;
    }
    if (!converged) return false;
    k[stage].resize(n);
    for (size_t i = 0; i < n; ++i) k[stage][i] = (z[i] - w[i]) / gdt;
  }
  x_new = std::move(z);
  est.assign(n, 0.0);
  const double e0 = kSdA[2][0] - kBhat1, e1 = kSdA[2][1] - kBhat2;
  for (size_t i = 0; i < n; ++i) est[i] = dt * (e0 * k[0][i] + e1 * k[1][i] + kGamma * k[2][i]);
  return true;
}
}  // namespace

StepAttempt sdirk_step(IntegratorState& state, OdeSystem& system, const SdirkOptions& options) {
  StepAttempt att;
  att.t_start = state.t;
  att.dt = state.dt;
  Vec x_new, est;
  int newton_iters = 0;
  const bool ok = sdirk_stages(state, system, state.dt, options, x_new, est, newton_iters);
  att.newton_iterations = newton_iters;
  state.stats.newton_iterations += newton_iters;
  if (!ok) {
    att.accepted = false;
    att.dt_next = 0.5 * state.dt;
    ++state.stats.rejected;
    state.dt = att.dt_next;
    return att;
  }
  att.error = weighted_rms(est, state.x, x_new, options.control.atol, options.control.rtol);
  const ControllerDecision dec = step_controller(att.error, state.dt, 3);
  bool finite = true;
  for (double v : x_new) finite = finite && std::isfinite(v);
  att.accepted = dec.accept && finite;
  att.dt_next = dec.dt_next;
  if (att.accepted) {
    state.x = std::move(x_new);
    state.t += state.dt;
    ++state.stats.accepted;
  } else {
    ++state.stats.rejected;
  }
  state.dt = dec.dt_next;
  return att;
}

bool sdirk_advance_fixed(IntegratorState& state, OdeSystem& system, double dt, const SdirkOptions& options) {
  Vec x_new, est;
  int newton_iters = 0;
  if (!sdirk_stages(state, system, dt, options, x_new, est, newton_iters)) return false;
  state.stats.newton_iterations += newton_iters;
  state.x = std::move(x_new);
  state.t += dt;
  ++state.stats.accepted;
  return true;
}

}  // namespace ora
