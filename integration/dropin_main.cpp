// Drop-in check: the reference's own integrators (proj/src/integrators.cpp,
// compiled unmodified into oracle/_ref/libeqsref.so) drive the B200 library
// through the C++ shim integration/eqs_gpu_shim.hpp, next to the reference's
// own FemSystem on the same mesh, dof map, materials and excitation, all built
// by the reference (SimConfig, generate_box_mesh, build_dof_map;
// proj/src/scenario.cpp:229-253). Compares eval_rhs, the spectral-radius
// estimate, 10 fixed RKC steps (path B), 3 adaptive rkc_step attempts and
// 2 fixed SDIRK3(2) steps.
//
//   dropin_main [config.json]      (default: the 14^3 three-layer slab cube)
// prints one JSON line; exit code 0 when every relative difference is within
// its gate.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "eqs/integrators.hpp"
#include "eqs/scenario.hpp"
#include "eqs_gpu_shim.hpp"

using namespace eqs;

static const char* kDefaultConfig = R"({
  "name": "dropin_slab",
  "mesh": {"box": {"nx": 14, "ny": 14, "nz": 14, "lx": 1.0, "ly": 1.0, "lz": 1.0,
                   "z_planes": [0.3333333333333333, 0.6666666666666666], "regions": [1, 2, 3]}},
  "order": 1,
  "materials": {
    "1": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}},
    "2": {"eps_r": 12.0, "conductivity": {"kind": "microvaristor", "kappa_lo": 1e-10, "kappa_hi": 3e-6,
                                          "e_switch": 5e5, "width": 5e4}},
    "3": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}}},
  "excitations": {"hv": {"kind": "sinusoid", "amplitude": 3333333.3333333335, "frequency": 50.0},
                  "ground": {"kind": "constant", "value": 0.0}},
  "solver": {"preconditioner": "amg", "rel_tol": 1e-12, "max_iter": 500},
  "estimator": {"mode": "spe", "window": 8}
})";

static double rel(const Vec& a, const Vec& b) { return (a - b).norm() / b.norm(); }

int main(int argc, char** argv) {
  std::string text = kDefaultConfig;
  if (argc > 1) {
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    text = ss.str();
  }
  try {
    const SimConfig cfg = SimConfig::from_json_text(text);
    TetMesh mesh = generate_box_mesh(cfg.box->nx, cfg.box->ny, cfg.box->nz, cfg.box->lx, cfg.box->ly, cfg.box->lz,
                                     cfg.box->layers);
    std::vector<std::string> dirichlet;
    for (const auto& [set, w] : cfg.excitations) dirichlet.push_back(set);
    const DofMap dm = build_dof_map(mesh, cfg.order, dirichlet);
    const BoundaryExcitation exc{cfg.excitations};
    FemSystem ref(mesh, dm, cfg.materials, exc, cfg.solver, cfg.estimator, 4);
    GpuFemSystem gpu(mesh, dm, cfg.materials, exc, cfg.solver, cfg.estimator, 0);
    const int n = dm.n_free();
    Vec x0(n);
    eqs_gpu_check(eqs_random_vec(n, 31u, x0.data()));  // mt19937 uniform(-1, 1), seed 31
    x0 *= 2e4;
    // F(t, x) through both systems
    Vec fr, fg;
    ref.eval_rhs(1e-3, x0, fr);
    gpu.eval_rhs(1e-3, x0, fg);
    const double rel_rhs = rel(fg, fr);
    // spectral radius (integrators.cpp:54-76) on both systems
    const double rho_r = estimate_spectral_radius(ref, 0.0, x0);
    const double rho_g = estimate_spectral_radius(gpu, 0.0, x0);
    // 10 fixed RKC steps, s = 4, dt = 0.2 beta(4) / rho (integrators.cpp:227-235)
    const double dt = 0.2 * RkcCoefficients::stability_boundary(4) / rho_r;
    IntegratorState sr, sg;
    sr.x = x0;
    sg.x = x0;
    for (int k = 0; k < 10; ++k) {
      rkc_advance_fixed(sr, ref, dt, 4);
      rkc_advance_fixed(sg, gpu, dt, 4);
    }
    const double rel_fixed = rel(sg.x, sr.x);
    // adaptive rkc_step (integrators.cpp:177-225) from the same state with the same cached rho
    RkcOptions o;
    o.control.rtol = cfg.tolerance;
    o.control.atol = cfg.effective_atol();
    IntegratorState ar, ag;
    ar.x = sr.x;
    ag.x = sr.x;
    ar.t = ag.t = sr.t;
    ar.dt = ag.dt = dt;
    int same_decisions = 1;
    for (int k = 0; k < 3; ++k) {
      const StepAttempt a = rkc_step(ar, ref, o);
      const StepAttempt b = rkc_step(ag, gpu, o);
      same_decisions &= a.accepted == b.accepted && a.stages == b.stages;
    }
    const double rel_adaptive = rel(ag.x, ar.x);
    // the implicit baseline through the same interface: 2 fixed SDIRK3(2)
    // steps (integrators.cpp:237-296) with Newton on the shifted systems
    IntegratorState ir, ig;  // milder start (the reference's Picard-type Newton needs it; test_gpu_sdirk.py)
    ir.x = x0;
    ir.x *= 0.01;
    ig.x = ir.x;
    const double dts = 5e-5;
    SdirkOptions so;
    bool okr = true, okg = true;
    for (int k = 0; k < 2; ++k) {
      okr = sdirk_advance_fixed(ir, ref, dts, so) && okr;
      okg = sdirk_advance_fixed(ig, gpu, dts, so) && okg;
    }
    const double rel_sdirk = rel(ig.x, ir.x);
    const bool ok = rel_rhs <= 1e-9 && std::fabs(rho_g - rho_r) <= 0.05 * rho_r && rel_fixed <= 1e-9 &&
                    rel_adaptive <= 1e-6 && same_decisions && okr && okg && rel_sdirk <= 1e-7;
    std::printf(
        "{\"n_free\": %d, \"rel_eval_rhs\": %.3e, \"rho_reference\": %.6e, \"rho_gpu\": %.6e, \"dt\": %.6e, "
        "\"rel_10_fixed_rkc_steps\": %.3e, \"rel_3_adaptive_rkc_steps\": %.3e, \"same_accept_and_stages\": %d, "
        "\"gpu_m_solves\": %ld, \"reference_m_solves\": %ld, \"rel_2_fixed_sdirk_steps\": %.3e, "
        "\"sdirk_converged\": [%d, %d], \"sdirk_newton_solves_gpu\": %ld, \"sdirk_newton_solves_reference\": %ld, "
        "\"pass\": %s}\n",
        n, rel_rhs, rho_r, rho_g, dt, rel_fixed, rel_adaptive, same_decisions, gpu.stats().m_solves,
        ref.stats().m_solves, rel_sdirk, (int)okr, (int)okg, gpu.stats().newton_linear_solves, ref.stats().newton_linear_solves,
        ok ? "true" : "false");
    return ok ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\", \"pass\": false}\n", e.what());
    return 2;
  }
}
