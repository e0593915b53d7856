// eqs_gpu_shim.hpp: the C++ shim a maintainer adds to the reference `eqsim`
// (proj/include/eqs/) to run its RKC path on the B200 library through the
// C-ABI in include/eqs_b200.h. Compiled against the
// unmodified reference headers by integration/Makefile; the drop-in test
// (integration/dropin_main.cpp) drives the reference's own integrators
// through it.
#pragma once

#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "eqs/errors.hpp"
#include "eqs/excitation.hpp"
#include "eqs/fem_system.hpp"
#include "eqs/materials.hpp"
#include "eqs/ode_system.hpp"
#include "eqs_b200.h"

namespace eqs {

// error codes -> the reference's exception classes (errors.hpp:10-37)
inline void eqs_gpu_check(int rc) {
  if (rc == EQS_OK) return;
  const std::string msg = eqs_last_error();
  switch (rc) {
    case EQS_ERR_CONFIG: throw ConfigError(msg);
    case EQS_ERR_NUMERICAL: throw NumericalError(msg);
    case EQS_ERR_GEOMETRY: throw GeometryError(msg);
    case EQS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case EQS_ERR_PARSE: throw ParseError(msg);
    default: throw std::runtime_error(msg);  // CUDA / other: exit code 2 in run_scenario
  }
}

// excitation.hpp:12-27
inline eqs_waveform to_c(const Waveform& w) {
  eqs_waveform c{};
  if (const auto* s = std::get_if<SinusoidWaveform>(&w)) {
    c.kind = 0;
    c.amplitude = s->amplitude;
    c.frequency = s->frequency;
    c.phase = s->phase;
  } else if (const auto* r = std::get_if<RampWaveform>(&w)) {
    c.kind = 1;
    c.amplitude = r->amplitude;
    c.rise_time = r->rise_time;
  } else {
    c.kind = 2;
    c.value = std::get<ConstantWaveform>(w).value;
  }
  return c;
}

// materials.hpp:10-33
inline eqs_material to_c(int region, const MaterialModel& m) {
  eqs_material c{};
  c.region = region;
  c.eps_r = m.eps_r;
  if (const auto* k = std::get_if<ConstantConductivity>(&m.conductivity)) {
    c.kind = 0;
    c.kappa = k->kappa;
  } else {
    const auto& v = std::get<MicrovaristorConductivity>(m.conductivity);
    c.kind = 1;
    c.kappa_lo = v.kappa_lo;
    c.kappa_hi = v.kappa_hi;
    c.e_switch = v.e_switch;
    c.width = v.width;
  }
  return c;
}

// fem_system.hpp:14-20, amg.hpp:12-18, start_vector.hpp:29-38; the additive
// GPU keys take the defaults the JSON configs get
inline eqs_solver_params to_c(const LinearSolverParams& s, const EstimatorParams& e) {
  eqs_solver_params c{};
  c.precond = s.precond == PrecondKind::Jacobi ? 0 : s.precond == PrecondKind::Ssor ? 1 : 2;
  c.rel_tol = s.rel_tol;
  c.max_iter = s.max_iter;
  c.rho_solve_tol = s.rho_solve_tol;
  c.amg_strength_threshold = s.amg.strength_threshold;
  c.amg_prolongation_omega = s.amg.prolongation_omega;
  c.amg_smoother_sweeps = s.amg.smoother_sweeps;
  c.amg_max_levels = s.amg.max_levels;
  c.amg_coarse_limit = s.amg.coarse_limit;
  c.estimator_mode = static_cast<int>(e.mode);  // Zero, Previous, Spe, PodFixed, PodRolling
  c.spe_window = e.spe_window;
  c.mgs_drop_tol = e.mgs_drop_tol;
  c.amg_coarse_filter = 0.0025;
  c.amg_dense_coarse = 512;
  c.pod_snapshots = e.pod_snapshots;
  c.pod_rank = e.pod_rank;
  c.pod_capacity = e.pod_capacity;
  c.pod_threshold = e.pod_threshold;
  return c;
}

// Drop-in for FemSystem (fem_system.hpp:28-78) behind the OdeSystem
// interface (ode_system.hpp:45-73): host vectors in and out, the system on
// the device. eqs_create copies everything, so nothing borrowed outlives the
// constructor except the dof map (size()).
class GpuFemSystem final : public OdeSystem {
 public:
  GpuFemSystem(const TetMesh& mesh, const DofMap& dm, const MaterialTable& materials,
               const BoundaryExcitation& exc, const LinearSolverParams& solver, const EstimatorParams& est,
               int device = 0)
      : dm_(dm) {
    std::vector<double> nodes;
    std::vector<int> tets, ed;
    nodes.reserve(3 * mesh.nodes.size());
    for (const auto& p : mesh.nodes) nodes.insert(nodes.end(), p.begin(), p.end());
    for (const auto& t : mesh.tets) tets.insert(tets.end(), t.begin(), t.end());
    for (const auto& e : dm.element_dofs) ed.insert(ed.end(), e.begin(), e.begin() + dm.n_local);
    std::vector<eqs_waveform> w;  // by DofMap::set_names index
    for (const auto& name : dm.set_names) w.push_back(to_c(exc.waveforms().at(name)));
    std::vector<eqs_material> m;
    for (const auto& [region, mm] : materials) m.push_back(to_c(region, mm));
    eqs_problem_desc d{};
    d.n_nodes = mesh.n_nodes();
    d.n_tets = mesh.n_tets();
    d.nodes = nodes.data();
    d.tets = tets.data();
    d.region_id = mesh.region_id.data();
    d.order = dm.order;
    d.n_dofs = dm.n_dofs;
    d.element_dofs = ed.data();
    d.n_free = dm.n_free();
    d.free_dofs = dm.free_dofs.data();
    d.n_fixed = dm.n_fixed();
    d.fixed_dofs = dm.fixed_dofs.data();
    d.fixed_set = dm.fixed_set.data();
    d.n_sets = static_cast<int>(w.size());
    d.set_waveforms = w.data();
    d.n_materials = static_cast<int>(m.size());
    d.materials = m.data();
    d.solver = to_c(solver, est);
    d.device = device;
    eqs_gpu_check(eqs_create(&d, &ctx_));
    refresh_stats();
  }
  GpuFemSystem(const GpuFemSystem&) = delete;
  GpuFemSystem& operator=(const GpuFemSystem&) = delete;
  ~GpuFemSystem() override { eqs_destroy(ctx_); }

  int size() const override { return dm_.n_free(); }
  void eval_rhs(double t, const Vec& x, Vec& f) override {  // fem_system.cpp:69-99
    f.resize(size());
    eqs_pcg_result r;
    const int rc = eqs_eval_rhs(ctx_, t, x.data(), f.data(), &r);
    refresh_stats();
    eqs_gpu_check(rc);
  }
  void eval_residual(double t, const Vec& x, Vec& r) override {  // fem_system.cpp:62-67
    r.resize(size());
    eqs_gpu_check(eqs_eval_residual(ctx_, t, x.data(), r.data()));
  }
  void mass_apply(const Vec& v, Vec& y) const override {  // fem_system.cpp:101
    y.resize(size());
    eqs_gpu_check(eqs_mass_apply(ctx_, v.data(), y.data()));
  }
  void apply_minv_stiffness(double t, const Vec& xs, const Vec& v, Vec& y) override {  // :103-122
    y.resize(size());
    const int rc = eqs_apply_minv_stiffness(ctx_, t, xs.data(), v.data(), y.data());
    refresh_stats();
    eqs_gpu_check(rc);
  }
  void shifted_solve(double t, const Vec& z, double gdt, const Vec& rhs, Vec& delta,
                     bool refresh) override {  // fem_system.cpp:124-145
    delta.resize(size());
    const int rc = eqs_shifted_solve(ctx_, t, z.data(), gdt, rhs.data(), delta.data(), refresh ? 1 : 0);
    refresh_stats();
    eqs_gpu_check(rc);
  }
  Vec lift_full(double t, const Vec& x) const {  // fem_system.cpp:56-60
    Vec full(dm_.n_dofs);
    eqs_gpu_check(eqs_lift_full(ctx_, t, x.data(), full.data()));
    return full;
  }
  eqs_ctx* handle() { return ctx_; }

 private:
  void refresh_stats() {  // ode_system.hpp:20-31
    eqs_solve_stats s;
    eqs_gpu_check(eqs_get_stats(ctx_, &s));
    stats_.m_solves = s.m_solves;
    stats_.pcg_iterations = s.pcg_iterations;
    stats_.rho_solves = s.rho_solves;
    stats_.rho_pcg_iterations = s.rho_pcg_iterations;
    stats_.newton_linear_solves = s.newton_linear_solves;
    stats_.newton_pcg_iterations = s.newton_pcg_iterations;
    stats_.precond_setups = s.precond_setups;
    stats_.assemblies = s.assemblies;
    stats_.svd_count = s.svd_count;
    stats_.timers = {s.time_residual, s.time_solve, s.time_setup, s.time_estimator};
  }
  eqs_ctx* ctx_ = nullptr;
  const DofMap& dm_;
};

}  // namespace eqs
