// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// extern "C" surface of the CPU restatement, loaded with ctypes by tests/,
// __graft_entry__.smoke() and bench.py's CPU-baseline leg (oracle/pyoracle.py).
#include <cstring>
#include <exception>
#include <string>

#include "oracle.hpp"

using namespace ora;

namespace {
thread_local std::string g_err;

struct Problem {
  SimConfig cfg;
  TetMesh mesh;
  DofMap dm;
  BoundaryExcitation exc;
  std::unique_ptr<FemSystem> sys;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const GeometryError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 4;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 7;
  }
}
Vec vec(const double* p, int n) { return p ? Vec(p, p + n) : Vec(); }
}  // namespace

extern "C" {

const char* ora_last_error() { return g_err.c_str(); }

int ora_create(const char* json_text, int workers, void** out) {
  return guard([&] {
    auto p = std::make_unique<Problem>();
    p->cfg = SimConfig::from_json_text(json_text);
    if (workers > 0) p->cfg.workers = workers;
    p->mesh = build_mesh(p->cfg);
    for (int t = 0; t < p->mesh.n_tets(); ++t)
      if (!p->cfg.materials.count(p->mesh.region_id[t]))
        throw ConfigError("no material for mesh region " + std::to_string(p->mesh.region_id[t]));
    std::vector<std::string> dirichlet;
    for (const auto& [set, w] : p->cfg.excitations) dirichlet.push_back(set);
    p->dm = build_dof_map(p->mesh, p->cfg.order, dirichlet);
    p->exc = BoundaryExcitation{p->cfg.excitations};
    p->sys = std::make_unique<FemSystem>(p->mesh, p->dm, p->cfg.materials, p->exc, p->cfg.solver, p->cfg.estimator,
                                         p->cfg.workers);
    *out = p.release();
  });
}

void ora_destroy(void* h) { delete static_cast<Problem*>(h); }

// sizes: n_nodes, n_tets, n_dofs, n_free, n_fixed, n_local, order, n_colors, nnz(M_II), nnz(M_IB)
int ora_sizes(void* h, long* out) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    out[0] = p->mesh.n_nodes();
    out[1] = p->mesh.n_tets();
    out[2] = p->dm.n_dofs;
    out[3] = p->dm.n_free();
    out[4] = p->dm.n_fixed();
    out[5] = p->dm.n_local;
    out[6] = p->dm.order;
    out[7] = p->sys->stiffness_operator().n_colors();
    out[8] = p->sys->mass_free().nnz();
    out[9] = p->sys->mass_ib().nnz();
  });
}

int ora_get_mesh(void* h, double* nodes, int* tets, int* region) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    for (int n = 0; n < p->mesh.n_nodes(); ++n)
      for (int d = 0; d < 3; ++d) nodes[3 * n + d] = p->mesh.nodes[n][d];
    for (int t = 0; t < p->mesh.n_tets(); ++t) {
      for (int v = 0; v < 4; ++v) tets[4 * t + v] = p->mesh.tets[t][v];
      region[t] = p->mesh.region_id[t];
    }
  });
}

int ora_get_dofs(void* h, int* element_dofs, int* free_dofs, int* fixed_dofs, int* fixed_set) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const int nl = p->dm.n_local;
    for (int t = 0; t < p->mesh.n_tets(); ++t)
      for (int i = 0; i < nl; ++i) element_dofs[(size_t)nl * t + i] = p->dm.element_dofs[t][i];
    std::memcpy(free_dofs, p->dm.free_dofs.data(), sizeof(int) * p->dm.n_free());
    std::memcpy(fixed_dofs, p->dm.fixed_dofs.data(), sizeof(int) * p->dm.n_fixed());
    std::memcpy(fixed_set, p->dm.fixed_set.data(), sizeof(int) * p->dm.n_dofs);
  });
}

int ora_get_colors(void* h, int* color_of_tet) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const auto& b = p->sys->stiffness_operator().color_batches();
    for (size_t c = 0; c < b.size(); ++c)
      for (int t : b[c]) color_of_tet[t] = (int)c;
  });
}

// which: 0 = M_II, 1 = M_IB
int ora_get_mass(void* h, int which, int* row_ptr, int* col_idx, double* values) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const CsrMatrix& m = which == 0 ? p->sys->mass_free() : p->sys->mass_ib();
    std::memcpy(row_ptr, m.row_ptr.data(), sizeof(int) * (m.n_rows + 1));
    std::memcpy(col_idx, m.col_idx.data(), sizeof(int) * m.nnz());
    std::memcpy(values, m.values.data(), sizeof(double) * m.nnz());
  });
}

int ora_kx_apply(void* h, const double* x_state, const double* v, double* y) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const int n = p->dm.n_dofs;
    Vec out;
    p->sys->stiffness_operator().apply(vec(x_state, n), vec(v, n), out);
    std::memcpy(y, out.data(), sizeof(double) * n);
  });
}

int ora_kx_residual(void* h, const double* x_full, const double* b_mass, double* r) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    Vec out;
    p->sys->stiffness_operator().residual(vec(x_full, p->dm.n_dofs), vec(b_mass, p->dm.n_free()), out);
    std::memcpy(r, out.data(), sizeof(double) * p->dm.n_free());
  });
}

// assembled K(x_full) applied to v (the reference's test oracle for the fused kernel)
int ora_assembled_k_apply(void* h, const double* x_full, const double* v, double* y) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const int n = p->dm.n_dofs;
    const CsrMatrix k = assemble_stiffness(p->mesh, p->dm, p->cfg.materials, vec(x_full, n));
    Vec out = k.apply(vec(v, n));
    std::memcpy(y, out.data(), sizeof(double) * n);
  });
}

int ora_eval_residual(void* h, double t, const double* x, double* r) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    Vec out;
    p->sys->eval_residual(t, vec(x, p->dm.n_free()), out);
    std::memcpy(r, out.data(), sizeof(double) * out.size());
  });
}

int ora_eval_rhs(void* h, double t, const double* x, double* f) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    Vec out;
    p->sys->eval_rhs(t, vec(x, p->dm.n_free()), out);
    std::memcpy(f, out.data(), sizeof(double) * out.size());
  });
}

int ora_lift_full(void* h, double t, const double* x, double* full) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    Vec out = p->sys->lift_full(t, vec(x, p->dm.n_free()));
    std::memcpy(full, out.data(), sizeof(double) * out.size());
  });
}

// M_II solve with the configured preconditioner; x0 may be null (zero start)
int ora_mass_solve(void* h, const double* b, const double* x0, double tol, int max_iter, double* x, int* iters,
                   double* rel, int* converged) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const int n = p->dm.n_free();
    const LinearOperator& pc = p->sys->mass_preconditioner();
    CsrOperator op(p->sys->mass_free());
    PcgResult r = pcg_solve(op, pc, vec(b, n), vec(x0, n), tol, max_iter);
    std::memcpy(x, r.x.data(), sizeof(double) * n);
    *iters = r.iterations;
    *rel = r.rel_residual;
    *converged = r.converged ? 1 : 0;
  });
}

int ora_mass_apply(void* h, const double* v, double* y) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    Vec out;
    p->sys->mass_apply(vec(v, p->dm.n_free()), out);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
  });
}

int ora_amg_levels(void* h, int* n_levels, long* rows_nnz /* 2 per level */) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    p->sys->mass_preconditioner();
    const AmgPreconditioner* a = p->sys->amg();
    if (!a) throw ConfigError("preconditioner is not AMG");
    *n_levels = a->n_levels();
    if (rows_nnz)
      for (int l = 0; l < a->n_levels(); ++l) {
        rows_nnz[2 * l] = a->level(l).A.n_rows;
        rows_nnz[2 * l + 1] = a->level(l).A.nnz();
      }
  });
}

int ora_amg_aggregates(void* h, int level, int* agg) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const AmgPreconditioner* a = p->sys->amg();
    if (!a) throw ConfigError("preconditioner is not AMG");
    const auto& v = a->level(level).aggregates;
    std::memcpy(agg, v.data(), sizeof(int) * v.size());
  });
}

int ora_spectral_radius(void* h, double t, const double* x, double* rho) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    *rho = estimate_spectral_radius(*p->sys, t, vec(x, p->dm.n_free()));
  });
}

// fixed-(dt, s) RKC, nsteps times from (t, x); x updated in place
int ora_rkc_advance_fixed(void* h, double t, double* x, double dt, int s, int nsteps) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    IntegratorState st;
    st.t = t;
    st.x = vec(x, p->dm.n_free());
    for (int i = 0; i < nsteps; ++i) rkc_advance_fixed(st, *p->sys, dt, s);
    std::memcpy(x, st.x.data(), sizeof(double) * st.x.size());
  });
}

// one adaptive rkc_step (integrators.cpp:177-225) with the rho cache pinned
// to `rho` (valid, age 0); out = accepted, stages, dt, error, rho, dt_next, t
int ora_rkc_step_pinned(void* h, double t, double* x, double dt, double rho, double rtol, double atol,
                        int max_stages, double* out) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    IntegratorState st;
    st.t = t;
    st.dt = dt;
    st.x = vec(x, p->dm.n_free());
    st.rho.value = rho;
    st.rho.valid = true;
    st.rho.age = 0;
    RkcOptions o;
    o.control.rtol = rtol;
    o.control.atol = atol;
    o.max_stages = max_stages;
    o.rho_refresh_every = 1 << 30;
    const StepAttempt a = rkc_step(st, *p->sys, o);
    std::memcpy(x, st.x.data(), sizeof(double) * st.x.size());
    out[0] = a.accepted;
    out[1] = a.stages;
    out[2] = a.dt;
    out[3] = a.error;
    out[4] = a.rho;
    out[5] = a.dt_next;
    out[6] = st.t;
  });
}

int ora_euler_step(void* h, double t, double* x, double dt) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    IntegratorState st;
    st.t = t;
    st.x = vec(x, p->dm.n_free());
    euler_step(st, *p->sys, dt);
    std::memcpy(x, st.x.data(), sizeof(double) * st.x.size());
  });
}

// stats: m_solves, pcg_iterations, rho_solves, rho_pcg_iterations, precond_setups, assemblies, applies, svd_count
int ora_stats(void* h, long* out, double* timers) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const SolveStats& s = p->sys->stats();
    out[0] = s.m_solves;
    out[1] = s.pcg_iterations;
    out[2] = s.rho_solves;
    out[3] = s.rho_pcg_iterations;
    out[4] = s.precond_setups;
    out[5] = s.assemblies;
    out[6] = p->sys->stiffness_operator().applies();
    out[7] = s.svd_count;
    if (timers) {
      timers[0] = s.timers.residual;
      timers[1] = s.timers.solve;
      timers[2] = s.timers.setup;
      timers[3] = s.timers.estimator;
    }
  });
}

// Full drop-in run (proj/src/scenario.cpp:217-383). Outputs: final free
// vector (caller buffer of n_free, may be null), totals[8] = accepted,
// rejected, stages, m_solves, pcg_iterations, rho_solves, precond_setups,
// n_free; final_t; wall.
int ora_run_scenario(const char* json_text, const char* out_dir, double* x_final, long x_cap, long* totals,
                     double* final_t, double* wall) {
  int rc = guard([&] {
    SimConfig c = SimConfig::from_json_text(json_text);
    RunResult r = run_scenario(c, out_dir ? out_dir : "");
    if (r.exit_code != 0) {
      g_err = r.error;
      throw std::runtime_error(r.error);
    }
    totals[0] = r.accepted;
    totals[1] = r.rejected;
    totals[2] = r.stages;
    totals[3] = r.stats.m_solves;
    totals[4] = r.stats.pcg_iterations;
    totals[5] = r.stats.rho_solves;
    totals[6] = r.stats.precond_setups;
    totals[7] = (long)r.final_x_free.size();
    if (x_final && (long)r.final_x_free.size() <= x_cap)
      std::memcpy(x_final, r.final_x_free.data(), sizeof(double) * r.final_x_free.size());
    *final_t = r.final_t;
    *wall = r.wall_time;
  });
  return rc;
}

// rkc amplification / coefficients for KAT tests
int ora_rkc_coefficients(int s, double* out /* w0, w1, mu1_tilde, c[0..s], mu, nu, mu_t, gamma_t [0..s] */) {
  return guard([&] {
    const RkcCoefficients k = RkcCoefficients::compute(s);
    out[0] = k.w0;
    out[1] = k.w1;
    out[2] = k.mu1_tilde;
    double* o = out + 3;
    for (int j = 0; j <= s; ++j) o[j] = k.c[j];
    o += s + 1;
    for (int j = 0; j <= s; ++j) o[j] = k.mu[j];
    o += s + 1;
    for (int j = 0; j <= s; ++j) o[j] = k.nu[j];
    o += s + 1;
    for (int j = 0; j <= s; ++j) o[j] = k.mu_tilde[j];
    o += s + 1;
    for (int j = 0; j <= s; ++j) o[j] = k.gamma_tilde[j];
  });
}

double ora_rkc_amplification(int s, double z) { return RkcCoefficients::compute(s).amplification(z); }

int ora_random_vec(int n, unsigned seed, double* out) {
  return guard([&] {
    Vec v = random_vec(n, seed);
    std::memcpy(out, v.data(), sizeof(double) * n);
  });
}

double ora_kappa_of_e(double eps_r, int kind, double k0, double k1, double k2, double k3, double e) {
  MaterialModel m;
  m.eps_r = eps_r;
  if (kind == 0) m.conductivity = ConstantConductivity{k0};
  else m.conductivity = MicrovaristorConductivity{k0, k1, k2, k3};
  return kappa_of_e(m, e);
}

// element matrices of one tet (KAT: reference-tet P1 matrix, P2 moment oracle)
int ora_element_laplacian(const double* coords /*12*/, int order, const double* coeff_at_qp, double* S /*n*n*/) {
  return guard([&] {
    std::array<std::array<double, 3>, 4> p;
    for (int v = 0; v < 4; ++v)
      for (int d = 0; d < 3; ++d) p[v][d] = coords[3 * v + d];
    const TetGeometry g = tet_geometry(p);
    double s[10][10];
    element_laplacian(g, order, coeff_at_qp, s);
    const int n = order == 1 ? 4 : 10;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) S[i * n + j] = s[i][j];
  });
}


// StartVectorEstimator public API (proj/include/eqs/start_vector.hpp:52-66) on
// the problem's own estimator and M_II: next(m, b), feedback(x, iterations),
// current_rank(), stats() = {svd_count, appends, spe_fallbacks}.
int ora_estimator_next(void* h, const double* b, double* x0, int* rank) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const int n = p->sys->size();
    const Vec bv(b, b + n);
    const Vec x = p->sys->estimator().next(p->sys->mass_free(), bv);
    std::memcpy(x0, x.data(), sizeof(double) * n);
    if (rank) *rank = p->sys->estimator().current_rank();
  });
}
int ora_estimator_feedback(void* h, const double* x, int iterations) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    p->sys->estimator().feedback(Vec(x, x + p->sys->size()), iterations);
  });
}
int ora_estimator_stats(void* h, long* out3) {
  return guard([&] {
    const auto& st = static_cast<Problem*>(h)->sys->estimator().stats();
    out3[0] = st.svd_count;
    out3[1] = st.appends;
    out3[2] = st.spe_fallbacks;
  });
}
// pod_build (start_vector.cpp:64-71) on k snapshots of length n (row-major
// [k][n]); writes up to `rank` basis vectors [keep][n] and all k singular values.
int ora_pod_build(int n, int k, const double* snaps, int rank, double* basis, int* keep, double* sigma) {
  return guard([&] {
    std::vector<Vec> s(k);
    for (int j = 0; j < k; ++j) s[j].assign(snaps + (size_t)j * n, snaps + (size_t)(j + 1) * n);
    std::vector<double> sv;
    const std::vector<Vec> u = pod_build(s, rank, &sv);
    *keep = (int)u.size();
    for (size_t j = 0; j < u.size(); ++j) std::memcpy(basis + j * n, u[j].data(), sizeof(double) * n);
    if (sigma) std::memcpy(sigma, sv.data(), sizeof(double) * sv.size());
  });
}

// sdirk_advance_fixed (integrators.cpp:329-341), nsteps fixed steps; returns
// NumericalError when a Newton iteration fails
int ora_sdirk_advance_fixed(void* h, double t, double* x, double dt, int nsteps) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    IntegratorState st;
    st.t = t;
    st.x.assign(x, x + p->sys->size());
    for (int i = 0; i < nsteps; ++i)
      if (!sdirk_advance_fixed(st, *p->sys, dt, SdirkOptions{})) throw NumericalError("sdirk: Newton failed");
    std::memcpy(x, st.x.data(), sizeof(double) * st.x.size());
  });
}

// FemSystem::shifted_solve (fem_system.cpp:124-145) on host vectors of n_free
int ora_shifted_solve(void* h, double t, const double* z, double gdt, const double* rhs, double* delta, int refresh) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    const int n = p->sys->size();
    Vec d;
    p->sys->shifted_solve(t, Vec(z, z + n), gdt, Vec(rhs, rhs + n), d, refresh != 0);
    std::memcpy(delta, d.data(), sizeof(double) * n);
  });
}
}  // extern "C"

extern "C" {
// which: 0 = A, 1 = P, 2 = R of level l. Call with null buffers to get sizes.
int ora_amg_level_csr(void* h, int level, int which, int* dims /*rows, cols, nnz*/, int* row_ptr, int* col_idx,
                      double* values) {
  return guard([&] {
    auto* p = static_cast<Problem*>(h);
    p->sys->mass_preconditioner();
    const AmgPreconditioner* a = p->sys->amg();
    if (!a) throw ConfigError("preconditioner is not AMG");
    const AmgLevel& lv = a->level(level);
    const CsrMatrix& m = which == 0 ? lv.A : which == 1 ? lv.P : lv.R;
    dims[0] = m.n_rows;
    dims[1] = m.n_cols;
    dims[2] = m.nnz();
    if (row_ptr) {
      std::memcpy(row_ptr, m.row_ptr.data(), sizeof(int) * (m.n_rows + 1));
      std::memcpy(col_idx, m.col_idx.data(), sizeof(int) * m.nnz());
      std::memcpy(values, m.values.data(), sizeof(double) * m.nnz());
    }
  });
}
}
