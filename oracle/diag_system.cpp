// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// DiagonalSystem surrogate (proj/tests/support/test_helpers.hpp:37-87): exact
// diagonal mass/stiffness solves so the integrators can be checked against
// closed forms (amplification, convergence order, stage choice, rho bracket).
#include <cmath>
#include <cstring>
#include <string>

#include "oracle.hpp"

using namespace ora;

namespace {
thread_local std::string d_err;
struct DiagonalSystem final : OdeSystem {
  Vec mass, stiffness;
  // b(t) = c1 sin(w1 t) + c2 cos(w2 t), same for every component (0 when c1 = c2 = 0)
  double c1 = 0, w1 = 0, c2 = 0, w2 = 0;
  int size() const override { return (int)mass.size(); }
  void eval_residual(double t, const Vec& x, Vec& r) override {
    r.resize(x.size());
    const double b = c1 * std::sin(w1 * t) + c2 * std::cos(w2 * t);
    for (size_t i = 0; i < x.size(); ++i) r[i] = -stiffness[i] * x[i] + b;
  }
  void eval_rhs(double t, const Vec& x, Vec& f) override {
    eval_residual(t, x, f);
    for (size_t i = 0; i < f.size(); ++i) f[i] /= mass[i];
    ++stats_.m_solves;
  }
  void mass_apply(const Vec& v, Vec& y) const override {
    y.resize(v.size());
    for (size_t i = 0; i < v.size(); ++i) y[i] = mass[i] * v[i];
  }
  void apply_minv_stiffness(double, const Vec&, const Vec& v, Vec& y) override {
    y.resize(v.size());
    for (size_t i = 0; i < v.size(); ++i) y[i] = stiffness[i] * v[i] / mass[i];
    ++stats_.rho_solves;
  }
  void shifted_solve(double, const Vec&, double gdt, const Vec& rhs, Vec& delta, bool refresh) override {
    if (refresh) ++stats_.precond_setups;  // test_helpers.hpp:67-72
    delta.resize(rhs.size());
    for (size_t i = 0; i < rhs.size(); ++i) delta[i] = rhs[i] / (mass[i] + gdt * stiffness[i]);
    ++stats_.newton_linear_solves;
  }
};
}  // namespace

extern "C" {
const char* ora_diag_last_error() { return d_err.c_str(); }

void* ora_diag_create(int n, const double* mass, const double* stiff, double c1, double w1, double c2, double w2) {
  auto* d = new DiagonalSystem;
  d->mass.assign(mass, mass + n);
  d->stiffness.assign(stiff, stiff + n);
  d->c1 = c1;
  d->w1 = w1;
  d->c2 = c2;
  d->w2 = w2;
  return d;
}
void ora_diag_destroy(void* h) { delete static_cast<DiagonalSystem*>(h); }

// method: 0 euler, 1 rkc_advance_fixed(s); x in/out, nsteps fixed steps of dt from t
int ora_diag_advance(void* h, int method, int s, double t, double dt, int nsteps, double* x) {
  auto* d = static_cast<DiagonalSystem*>(h);
  try {
    IntegratorState st;
    st.t = t;
    st.x.assign(x, x + d->size());
    for (int i = 0; i < nsteps; ++i) {
      if (method == 0) euler_step(st, *d, dt);
      else if (method == 1) rkc_advance_fixed(st, *d, dt, s);
      else if (!sdirk_advance_fixed(st, *d, dt, SdirkOptions{})) throw NumericalError("sdirk: Newton failed");
    }
    std::memcpy(x, st.x.data(), sizeof(double) * st.x.size());
    return 0;
  } catch (const std::exception& e) {
    d_err = e.what();
    return 7;
  }
}

// one adaptive rkc_step; out[0..6] = accepted, stages, dt, error, rho, dt_next, t
int ora_diag_rkc_step(void* h, double t, double dt, double rtol, double atol, int max_stages, double* x,
                      double* out) {
  auto* d = static_cast<DiagonalSystem*>(h);
  try {
    IntegratorState st;
    st.t = t;
    st.dt = dt;
    st.x.assign(x, x + d->size());
    RkcOptions o;
    o.control.rtol = rtol;
    o.control.atol = atol;
    o.max_stages = max_stages;
    const StepAttempt a = rkc_step(st, *d, o);
    std::memcpy(x, st.x.data(), sizeof(double) * st.x.size());
    out[0] = a.accepted;
    out[1] = a.stages;
    out[2] = a.dt;
    out[3] = a.error;
    out[4] = a.rho;
    out[5] = a.dt_next;
    out[6] = st.t;
    return 0;
  } catch (const std::exception& e) {
    d_err = e.what();
    return 7;
  }
}

// one sdirk_step (integrators.cpp:297-327); out[0..6] = accepted, newton_iterations, dt, error, dt_next, t,
// precond_setups
int ora_diag_sdirk_step(void* h, double t, double dt, double rtol, double atol, double* x, double* out) {
  auto* d = static_cast<DiagonalSystem*>(h);
  try {
    IntegratorState st;
    st.t = t;
    st.dt = dt;
    st.x.assign(x, x + d->size());
    SdirkOptions o;
    o.control.rtol = rtol;
    o.control.atol = atol;
    const StepAttempt a = sdirk_step(st, *d, o);
    std::memcpy(x, st.x.data(), sizeof(double) * st.x.size());
    out[0] = a.accepted;
    out[1] = a.newton_iterations;
    out[2] = a.dt;
    out[3] = a.error;
    out[4] = a.dt_next;
    out[5] = st.t;
    out[6] = (double)d->stats().precond_setups;
    return 0;
  } catch (const std::exception& e) {
    d_err = e.what();
    return 7;
  }
}

double ora_diag_spectral_radius(void* h) {
  auto* d = static_cast<DiagonalSystem*>(h);
  return estimate_spectral_radius(*d, 0.0, Vec(d->size(), 0.0));
}

// step_controller (integrators.cpp:12-18): out = {accept, dt_next}
void ora_step_controller(double err, double dt, int order, double* out) {
  const ControllerDecision c = step_controller(err, dt, order);
  out[0] = c.accept;
  out[1] = c.dt_next;
}
}
