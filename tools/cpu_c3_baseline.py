#!/usr/bin/env python
"""Full-size C3 record of the reference's CPU path, with GPU parity at C3.

Runs the UNMODIFIED reference (oracle/_ref/libeqsref.so: proj/src compiled
against the Eigen-API shim; checker / baseline only) on the headline workload
(215^3 jittered cube, 9,984,384 free dofs, SPE(8), AMG-PCG 1e-12) with
workers = all host cores (only the element kernel is threaded, exactly as in
the reference, proj/src/matfree.cpp:105-115):

* setup (FemSystem: mesh, M assembly, colouring; AMG setup on the first solve),
* rho(x0) by estimate_spectral_radius (integrators.cpp:49-75),
* `--steps` rkc_advance_fixed steps (path B, s = 4, dt = 0.9 beta(4)/rho),
* the reference's own responses after those steps to a 1e-12 relative
  perturbation of x0 and to PCG tolerance 1e-13 (its conditioning),

then the B200 path from the same x0 and dt, and writes everything to
profiles/CPU_r2_c3.json (bench.py quotes it as cpu_baseline.c3_full_size_record).

    python tools/cpu_c3_baseline.py [--n 215] [--steps 1] [--no-sens] [--out profiles/CPU_r2_c3.json]
"""
import argparse
import copy
import json
import os
import resource
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (scenario builder, CpuArm, cpu_model)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=215)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--no-sens", action="store_true")
    ap.add_argument("--no-gpu", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "CPU_r2_c3.json"))
    args = ap.parse_args()
    from oracle import pyoracle as po  # random_vec only
    from oracle import pyref as pr

    assert pr.available(), "oracle/_ref/libeqsref.so is not built"
    cores = os.cpu_count() or 1
    cfg = bench.scenario(args.n, 0.1, [0.45, 0.55])
    rec = {"what": "reference CPU path (unmodified proj/src + Eigen-API shim, oracle/_ref) on the full C3 workload",
           "cpu_model": bench.cpu_model(), "cores": cores, "workers": cores, "mesh_cells": args.n,
           "steps": args.steps}

    def emit():
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(rec, f, indent=1)
        print(json.dumps(rec), flush=True)

    t0 = time.perf_counter()
    r = pr.RefProblem(cfg, workers=cores)
    rec["n_free"] = r.n_free
    rec["setup_construct_s"] = time.perf_counter() - t0
    x0 = 2e4 * po.random_vec(r.n_free, 31)
    t0 = time.perf_counter()
    rho = r.spectral_radius(0.0, x0)  # the first solve also builds the AMG hierarchy
    rec["rho"] = rho
    rec["rho_plus_amg_setup_s"] = time.perf_counter() - t0
    st = r.stats()
    rec["amg_setup_s"] = st["timers"]["setup"]
    dt = 0.9 * 0.653 * 15 / rho
    rec["dt"] = dt
    emit()
    s0 = r.stats()
    r.set_state(0.0, x0, dt)
    t0 = time.perf_counter()
    r.rkc_advance_fixed(dt, 4, args.steps)
    wall = time.perf_counter() - t0
    s1 = r.stats()
    xr = r.get_state()[0]
    fe = s1["m_solves"] - s0["m_solves"]
    rec.update({"step_s": wall / args.steps, "steps_per_s": args.steps / wall,
                "value": r.n_free * fe / wall, "unit": "DOF-stage-updates/s",
                "f_evals_per_step": fe / args.steps,
                "pcg_iters_per_solve": (s1["pcg_iterations"] - s0["pcg_iterations"]) / max(1, fe),
                "phase_s": {k: s1["timers"][k] - s0["timers"][k] for k in ("residual", "solve", "estimator")},
                "host_peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6})
    emit()
    del r
    sens = {}
    if not args.no_sens:
        for name, c, xs in (("x0_1e-12", cfg, x0 * (1 + 1e-12)), ("tol_1e-13", None, x0)):
            if c is None:
                c = copy.deepcopy(cfg)
                c["solver"]["rel_tol"] = 1e-13
            p = pr.RefProblem(c, workers=cores)
            p.set_state(0.0, xs, dt)
            p.rkc_advance_fixed(dt, 4, args.steps)
            sens[name] = float(np.linalg.norm(p.get_state()[0] - xr) / np.linalg.norm(xr))
            del p
        rec["reference_responses"] = sens
        emit()
    if not args.no_gpu:
        import paper_1612_09447_b200 as eb
        t0 = time.perf_counter()
        g = eb.FemSystem(cfg, device=0)
        rec["gpu_setup_s"] = time.perf_counter() - t0
        g.set_state(0.0, x0, dt)
        g.rkc_advance_fixed(dt, 4, args.steps)
        xg = g.get_state()[0]
        rel = float(np.linalg.norm(xg - xr) / np.linalg.norm(xr))
        gate = 10.0 * max(list(sens.values()) + [1e-9 / 10])
        rec["gpu_parity"] = {"rel_l2_gpu_vs_reference": rel, "gate": gate, "pass": rel <= gate,
                             "rule": "10x the larger reference response (or 1e-9)"}
        emit()


if __name__ == "__main__":
    main()
