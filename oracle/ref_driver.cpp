// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// C driver over the UNMODIFIED reference sources (/root/reference/proj/src,
// compiled by oracle/Makefile target `ref` against oracle/ref_shim) ->
// oracle/_ref/libeqsref.so. It exists to pin the restatement in oracle/ and
// the GPU path to the reference's own outputs (tests/golden/ fixtures made by
// tests/golden/make_ref_fixtures.py) and to time the reference's CPU path as
// bench.py's `--impl reference` arm. It only calls the reference's public
// API: SimConfig::from_json_text (scenario.cpp:110-211), generate_box_mesh /
// finalize (mesh.cpp:57-154), build_dof_map (dofmap.cpp:22-91),
// BoundaryExcitation, FemSystem (fem_system.cpp), color_elements
// (matfree.cpp:11-38), aggregate / AmgPreconditioner (amg.cpp:49-143),
// estimate_spectral_radius / rkc_advance_fixed / rkc_step / euler_step
// (integrators.cpp) and run_scenario (scenario.cpp:217-383).
//
// The one addition is the benchmark meshes' jitter (an
// additive key of this repository): the same rule as oracle/mesh_dof.cpp
// jitter_box_mesh, applied to the reference's generated mesh, then the
// reference's own TetMesh::finalize().
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>

#include "eqs/amg.hpp"
#include "eqs/errors.hpp"
#include "eqs/fem_system.hpp"
#include "eqs/integrators.hpp"
#include "eqs/matfree.hpp"
#include "eqs/msh_io.hpp"
#include "eqs/scenario.hpp"

using namespace eqs;

namespace {

struct RefCtx {
  SimConfig cfg;
  TetMesh mesh;
  DofMap dm;
  std::unique_ptr<BoundaryExcitation> exc;
  std::unique_ptr<FemSystem> sys;
  IntegratorState state;
  std::unique_ptr<AmgPreconditioner> amg;  // standalone hierarchy for inspection
};

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const NumericalError*>(&e)) return 2;
  if (dynamic_cast<const GeometryError*>(&e)) return 3;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 4;
  return 7;
}

void jitter(TetMesh& m, const BoxSpec& b, double amplitude, unsigned seed) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  const int n[3] = {b.nx, b.ny, b.nz};
  const double h[3] = {b.lx / b.nx, b.ly / b.ny, b.lz / b.nz};
  for (int k = 0; k <= b.nz; ++k)
    for (int j = 0; j <= b.ny; ++j)
      for (int i = 0; i <= b.nx; ++i) {
        const int id = (k * (b.ny + 1) + j) * (b.nx + 1) + i;
        const int idx[3] = {i, j, k};
        double u[3];
        for (int d = 0; d < 3; ++d) u[d] = uni(rng);
        for (int d = 0; d < 3; ++d)
          if (idx[d] > 0 && idx[d] < n[d]) m.nodes[id][d] += amplitude * h[d] * u[d];
      }
  m.finalize();
}

Vec to_vec(const double* p, int n) {
  Vec v(n);
  for (int i = 0; i < n; ++i) v[i] = p[i];
  return v;
}
void from_vec(const Vec& v, double* p) {
  for (Eigen::Index i = 0; i < v.size(); ++i) p[i] = v[i];
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Build mesh, dof map, excitation and FemSystem exactly as run_scenario does
// (scenario.cpp:229-253). jitter > 0 moves interior nodes (box meshes only).
int ref_create(const char* json_text, double jitter_amp, unsigned jitter_seed, void** out) {
  try {
    auto c = std::make_unique<RefCtx>();
    c->cfg = SimConfig::from_json_text(json_text);
    const SimConfig& cfg = c->cfg;
    if (cfg.mesh_file) c->mesh = load_msh(*cfg.mesh_file);
    else if (cfg.box)
      c->mesh = generate_box_mesh(cfg.box->nx, cfg.box->ny, cfg.box->nz, cfg.box->lx, cfg.box->ly,
                                  cfg.box->lz, cfg.box->layers);
    else throw ConfigError("no mesh source in config");
    if (jitter_amp != 0.0 && cfg.box) jitter(c->mesh, *cfg.box, jitter_amp, jitter_seed);
    for (int t = 0; t < c->mesh.n_tets(); ++t)
      if (!cfg.materials.count(c->mesh.region_id[t]))
        throw ConfigError("no material for mesh region " + std::to_string(c->mesh.region_id[t]));
    std::vector<std::string> dirichlet;
    for (const auto& [set, w] : cfg.excitations) dirichlet.push_back(set);
    c->dm = build_dof_map(c->mesh, cfg.order, dirichlet);
    c->exc = std::make_unique<BoundaryExcitation>(BoundaryExcitation{cfg.excitations});
    c->sys = std::make_unique<FemSystem>(c->mesh, c->dm, cfg.materials, *c->exc, cfg.solver,
                                         cfg.estimator, cfg.workers);
    c->state.t = 0;
    c->state.x = Vec::Zero(c->dm.n_free());
    c->state.dt = cfg.dt0;
    *out = c.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_destroy(void* h) { delete static_cast<RefCtx*>(h); }

// sizes: n_nodes, n_tets, n_dofs, n_free, n_fixed, nnz(M_II), n_colors, workers
int ref_sizes(void* h, long* out) {
  auto* c = static_cast<RefCtx*>(h);
  out[0] = c->mesh.n_nodes();
  out[1] = c->mesh.n_tets();
  out[2] = c->dm.n_dofs;
  out[3] = c->dm.n_free();
  out[4] = c->dm.n_fixed();
  out[5] = c->sys->mass_free().nnz();
  out[6] = c->sys->stiffness_operator().n_colors();
  out[7] = c->cfg.workers;
  return 0;
}

// node coordinates [n_nodes x 3] and tets [n_tets x 4] after finalize()
int ref_mesh(void* h, double* nodes, int* tets, int* region) {
  auto* c = static_cast<RefCtx*>(h);
  for (int i = 0; i < c->mesh.n_nodes(); ++i)
    for (int d = 0; d < 3; ++d) nodes[3 * i + d] = c->mesh.nodes[i][d];
  for (int t = 0; t < c->mesh.n_tets(); ++t) {
    for (int d = 0; d < 4; ++d) tets[4 * t + d] = c->mesh.tets[t][d];
    region[t] = c->mesh.region_id[t];
  }
  return 0;
}

int ref_free_dofs(void* h, int* free_dofs) {
  auto* c = static_cast<RefCtx*>(h);
  std::copy(c->dm.free_dofs.begin(), c->dm.free_dofs.end(), free_dofs);
  return 0;
}

// colour of every tet from color_elements (matfree.cpp:11-38)
int ref_colors(void* h, int* color_of_tet) {
  auto* c = static_cast<RefCtx*>(h);
  const auto batches = color_elements(c->dm, c->mesh.n_tets());
  for (size_t k = 0; k < batches.size(); ++k)
    for (int t : batches[k]) color_of_tet[t] = static_cast<int>(k);
  return static_cast<int>(batches.size());
}

// M_II in CSR (assemble_mass + split_dirichlet, fem_system.cpp:33-35)
int ref_mass_free(void* h, int* row_ptr, int* col_idx, double* values) {
  auto* c = static_cast<RefCtx*>(h);
  const CsrMatrix& m = c->sys->mass_free();
  std::copy(m.row_ptr.begin(), m.row_ptr.end(), row_ptr);
  std::copy(m.col_idx.begin(), m.col_idx.end(), col_idx);
  std::copy(m.values.begin(), m.values.end(), values);
  return 0;
}

// aggregate ids of M_II's rows (amg.cpp:49-88, theta from the config)
int ref_aggregate(void* h, int* agg) {
  auto* c = static_cast<RefCtx*>(h);
  const auto a = aggregate(c->sys->mass_free(), c->cfg.solver.amg.strength_threshold);
  std::copy(a.begin(), a.end(), agg);
  return 0;
}

// SA-AMG hierarchy of M_II (amg.cpp:90-143): per level rows, nnz(A), nnz(P)
int ref_amg_levels(void* h, int* n_levels, long* rows, long* nnz_a, long* nnz_p, int max_levels) {
  auto* c = static_cast<RefCtx*>(h);
  try {
    if (!c->amg) c->amg = std::make_unique<AmgPreconditioner>(c->sys->mass_free(), c->cfg.solver.amg);
    *n_levels = c->amg->n_levels();
    for (int l = 0; l < c->amg->n_levels() && l < max_levels; ++l) {
      rows[l] = c->amg->level(l).A.n_rows;
      nnz_a[l] = c->amg->level(l).A.nnz();
      nnz_p[l] = c->amg->level(l).P.nnz();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// level l Galerkin operator values (CSR order) and its sum of |values|
int ref_amg_level_csr(void* h, int l, int* row_ptr, int* col_idx, double* values) {
  auto* c = static_cast<RefCtx*>(h);
  const CsrMatrix& a = c->amg->level(l).A;
  std::copy(a.row_ptr.begin(), a.row_ptr.end(), row_ptr);
  std::copy(a.col_idx.begin(), a.col_idx.end(), col_idx);
  std::copy(a.values.begin(), a.values.end(), values);
  return 0;
}

// y_full = K(x_state) v over all dofs (MatFreeStiffness::apply, matfree.cpp:90-117)
int ref_kx_apply(void* h, const double* x_full, const double* v_full, double* y_full) {
  auto* c = static_cast<RefCtx*>(h);
  try {
    Vec y;
    c->sys->stiffness_operator().apply(to_vec(x_full, c->dm.n_dofs), to_vec(v_full, c->dm.n_dofs), y);
    from_vec(y, y_full);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_mass_apply(void* h, const double* v, double* y) {
  auto* c = static_cast<RefCtx*>(h);
  Vec out;
  c->sys->mass_apply(to_vec(v, c->dm.n_free()), out);
  from_vec(out, y);
  return 0;
}

int ref_eval_residual(void* h, double t, const double* x, double* r) {
  auto* c = static_cast<RefCtx*>(h);
  try {
    Vec out;
    c->sys->eval_residual(t, to_vec(x, c->dm.n_free()), out);
    from_vec(out, r);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_eval_rhs(void* h, double t, const double* x, double* f) {
  auto* c = static_cast<RefCtx*>(h);
  try {
    Vec out;
    c->sys->eval_rhs(t, to_vec(x, c->dm.n_free()), out);
    from_vec(out, f);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_lift_full(void* h, double t, const double* x_free, double* x_full) {
  auto* c = static_cast<RefCtx*>(h);
  from_vec(c->sys->lift_full(t, to_vec(x_free, c->dm.n_free())), x_full);
  return 0;
}

// estimate_spectral_radius (integrators.cpp:49-75), 1.2 x power-iteration value
int ref_spectral_radius(void* h, double t, const double* x, double* rho) {
  auto* c = static_cast<RefCtx*>(h);
  try {
    *rho = estimate_spectral_radius(*c->sys, t, to_vec(x, c->dm.n_free()));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_set_state(void* h, double t, const double* x, double dt) {
  auto* c = static_cast<RefCtx*>(h);
  c->state.t = t;
  c->state.x = to_vec(x, c->dm.n_free());
  c->state.dt = dt;
  c->state.rho = RhoCache{};
  return 0;
}

int ref_get_state(void* h, double* t, double* x, double* dt) {
  auto* c = static_cast<RefCtx*>(h);
  *t = c->state.t;
  if (dt) *dt = c->state.dt;
  if (x) from_vec(c->state.x, x);
  return 0;
}

// rkc_advance_fixed (integrators.cpp:227-235), `steps` times
int ref_rkc_advance_fixed(void* h, double dt, int s, int steps) {
  auto* c = static_cast<RefCtx*>(h);
  try {
    for (int k = 0; k < steps; ++k) rkc_advance_fixed(c->state, *c->sys, dt, s);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// rkc_step (integrators.cpp:177-225) with the config's tolerances; an optional
// pinned rho (> 0) is installed in the cache before the attempt.
// att: t_start, dt, accepted, stages, error, rho, dt_next
int ref_rkc_step(void* h, double pinned_rho, double* att) {
  auto* c = static_cast<RefCtx*>(h);
  try {
    if (pinned_rho > 0) {
      c->state.rho.value = pinned_rho;
      c->state.rho.valid = true;
      c->state.rho.age = 0;
    }
    RkcOptions o;
    o.control = {c->cfg.tolerance, c->cfg.effective_atol()};
    o.max_stages = c->cfg.max_stages;
    const StepAttempt a = rkc_step(c->state, *c->sys, o);
    att[0] = a.t_start;
    att[1] = a.dt;
    att[2] = a.accepted ? 1 : 0;
    att[3] = a.stages;
    att[4] = a.error;
    att[5] = a.rho;
    att[6] = a.dt_next;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_euler_step(void* h, double dt) {
  auto* c = static_cast<RefCtx*>(h);
  try {
    euler_step(c->state, *c->sys, dt);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// SolveStats (ode_system.hpp:20-31) + phase timers:
// m_solves, pcg_iterations, rho_solves, rho_pcg_iterations, newton_linear_solves,
// newton_pcg_iterations, precond_setups, assemblies, svd_count
int ref_stats(void* h, long* out, double* timers) {
  auto* c = static_cast<RefCtx*>(h);
  const SolveStats& s = c->sys->stats();
  const long v[9] = {s.m_solves, s.pcg_iterations, s.rho_solves, s.rho_pcg_iterations,
                     s.newton_linear_solves, s.newton_pcg_iterations, s.precond_setups,
                     s.assemblies, s.svd_count};
  std::memcpy(out, v, sizeof(v));
  if (timers) {
    timers[0] = s.timers.setup;
    timers[1] = s.timers.residual;
    timers[2] = s.timers.solve;
    timers[3] = s.timers.estimator;
  }
  return 0;
}

// full run_scenario (scenario.cpp:217-383): exit code, accepted/rejected steps,
// final t and the final free-dof state (caller buffer of n_free, may be null)
int ref_run_scenario(const char* json_text, const char* out_dir, long* counts, double* final_t,
                     double* final_x, int final_x_len) {
  try {
    const SimConfig cfg = SimConfig::from_json_text(json_text);
    const RunResult r = run_scenario(cfg, out_dir ? out_dir : "");
    counts[0] = r.exit_code;
    counts[1] = r.totals.accepted;
    counts[2] = r.totals.rejected;
    counts[3] = r.totals.stats.m_solves;
    counts[4] = r.totals.stats.pcg_iterations;
    counts[5] = static_cast<long>(r.final_x_free.size());
    *final_t = r.final_t;
    if (final_x && final_x_len == r.final_x_free.size()) from_vec(r.final_x_free, final_x);
    g_err = r.error;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
