"""Regenerate the reference-made golden fixtures (tests/golden/ref_*.npz).

Every number in these files is an output of the UNMODIFIED reference
(/root/reference/proj/src, compiled by `make -C oracle ref` into
oracle/_ref/libeqsref.so against the Eigen-API shim oracle/ref_shim), driven
through its public API by oracle/ref_driver.cpp (oracle/pyref.py). Run in the
build container, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_ref_fixtures.py

The GPU box and the CPU test suite only read the committed .npz files.

Fixtures
* ref_c1.npz   — SURVEY.md §8d config 1 (36^3 cube, layers 1/3 2/3, SPE(8),
  AMG-PCG 1e-12): setup artefact hashes (mesh, dof map, colouring, M_II,
  aggregates), AMG level sizes, rho(x0), path (B) potentials after 10
  rkc_advance_fixed steps (integrators.cpp:227-235) from x0 = 2e4 random_vec(31)
  at dt = 0.2 and 0.9 beta(4)/rho, and the reference's own responses to a
  1e-12 relative perturbation of x0 and to a PCG tolerance of 1e-13 instead
  of 1e-12 (the trajectory's conditioning at the benchmark step).
* ref_c3s.npz  — the C3 family (jittered +-0.1h, layer z in [0.45, 0.55]) at
  24^3: same artefacts and path (B) at the benchmark step 0.9 beta(4)/rho.
* ref_small.npz — 12^3 cube: full K(x)v (matfree.cpp:90-117) and eval_rhs
  (fem_system.cpp:69-99) vectors, P1/P2 matfree K(x)v on the reference's
  test_matfree setup, 25 adaptive rkc_step attempts with rho pinned
  (integrators.cpp:177-225), 10 euler_step steps, and the final state of
  run_scenario (scenario.cpp:217-383) on the committed slab_nonlinear_rkc_spe
  config cut at t_end = 0.004, with the reference's own response to a 1e-12
  relative change of dt0 (the adaptive trajectory's conditioning).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from helpers import cube, matfree_setup, slab_reference  # noqa: E402
from oracle import pyoracle as po  # noqa: E402  (random_vec only: mt19937 + uniform, test_helpers.hpp:15-21)
from oracle import pyref as pr  # noqa: E402

BETA4 = 0.653 * 15.0


def digest(a) -> str:
    """sha256 of the array's bytes (C order, its own dtype)."""
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def artefacts(r: pr.RefProblem) -> dict:
    nodes, tets, region = r.mesh()
    rp, ci, v = r.mass_free()
    rows, nnz_a, nnz_p = r.amg_levels()
    return {
        "sizes": np.array([r.n_nodes, r.n_tets, r.n_dofs, r.n_free, r.nnz_ii, r.n_colors], dtype=np.int64),
        "sha_nodes": digest(nodes.astype(np.float64)), "sha_tets": digest(tets.astype(np.int32)),
        "sha_region": digest(region.astype(np.int32)), "sha_free": digest(r.free_dofs().astype(np.int32)),
        "sha_colors": digest(r.colors().astype(np.int32)),
        "sha_mass_rowptr": digest(rp), "sha_mass_col": digest(ci), "sha_mass_val": digest(v),
        "sha_aggregates": digest(r.aggregate().astype(np.int32)),
        "amg_rows": np.array(rows, dtype=np.int64), "amg_nnz_a": np.array(nnz_a, dtype=np.int64),
        "amg_nnz_p": np.array(nnz_p, dtype=np.int64),
        "mass_val_sum": float(np.sum(v)), "mass_val_abs_sum": float(np.sum(np.abs(v))),
    }


def path_b(cfg, fracs, perturb_frac=None, steps=10):
    """rho(x0) and path (B) potentials after `steps` fixed RKC steps per dt fraction.
    For `perturb_frac` also the reference's own conditioning: its response to a
    1e-12 relative perturbation of x0 (sens_*) and to tightening the PCG
    stopping rule from 1e-12 to 1e-13 (sens_tol_*: the result is defined by
    the solver tolerance only up to this)."""
    r = pr.RefProblem(cfg)
    out = artefacts(r)
    x0 = 2e4 * po.random_vec(r.n_free, 31)
    rho = r.spectral_radius(0.0, x0)
    out["rho0"] = rho

    def run(c, xs, dt):  # a fresh system per run: no estimator history carried over
        p = pr.RefProblem(c)
        p.set_state(0.0, xs, dt)
        p.rkc_advance_fixed(dt, 4, steps)
        st = p.stats()
        return p.get_state()[0], st["pcg_iterations"] / max(1, st["m_solves"])

    for frac in fracs:
        key = f"b{int(round(frac * 100)):03d}"
        dt = frac * BETA4 / rho
        x, its = run(cfg, x0, dt)
        out[f"x_{key}"] = x
        out[f"dt_{key}"] = dt
        out[f"iters_{key}"] = its
        if perturb_frac is not None and abs(frac - perturb_frac) < 1e-12:
            xp, _ = run(cfg, x0 * (1 + 1e-12), dt)
            out[f"sens_{key}"] = float(np.linalg.norm(xp - x) / np.linalg.norm(x))
            tight = json.loads(json.dumps(cfg))
            tight["solver"]["rel_tol"] = 1e-13
            xt, _ = run(tight, x0, dt)
            out[f"sens_tol_{key}"] = float(np.linalg.norm(xt - x) / np.linalg.norm(x))
        print(f"  {key}: dt {dt:.4e} iters/solve {out[f'iters_{key}']:.2f} |x| {np.linalg.norm(x):.6e}"
              + (f" sens {out[f'sens_{key}']:.2e} sens_tol {out[f'sens_tol_{key}']:.2e}"
                 if f"sens_{key}" in out else ""), flush=True)
    return out


def small():
    out = {}
    cfg = cube(12)
    r = pr.RefProblem(cfg)
    x0 = 2e4 * po.random_vec(r.n_free, 31)
    xf = r.lift_full(1e-3, x0)
    v = po.random_vec(r.n_dofs, 7)
    out["cube12_kx"] = r.kx_apply(xf, v)
    out["cube12_rhs"] = r.eval_rhs(1e-3, x0)
    for order in (1, 2):
        c = matfree_setup(order, True)
        rm = pr.RefProblem(c)
        x = 2.0 * po.random_vec(rm.n_dofs, 101 + order)
        vv = po.random_vec(rm.n_dofs, 202 + order)
        out[f"matfree_p{order}_kx"] = rm.kx_apply(x, vv)
    # adaptive rkc_step with the rho cache pinned (the GPU and the reference
    # then take the same decisions; rho itself is preconditioner-dependent)
    cfg = slab_reference("slab_nonlinear_rkc_spe")
    r = pr.RefProblem(cfg)
    x = np.zeros(r.n_free)
    rho = r.spectral_radius(0.0, x)
    r.set_state(0.0, x, 1e-5)
    att = []
    for _ in range(25):
        a = r.rkc_step(pinned_rho=rho)
        att.append([a["t_start"], a["dt"], float(a["accepted"]), a["stages"], a["error"], a["dt_next"]])
    out["slab_rho_pinned"] = rho
    out["slab_attempts"] = np.array(att)
    out["slab_x25"] = r.get_state()[0]
    # explicit Euler (integrators.cpp:33-47) at the driver's dt rule on 12^3
    cfg = cube(12)
    r = pr.RefProblem(cfg)
    x0 = 2e4 * po.random_vec(r.n_free, 31)
    rho = r.spectral_radius(0.0, x0)
    dt = min(1e-5, 1.8 / rho)
    r.set_state(0.0, x0, dt)
    for _ in range(10):
        r.euler_step(dt)
    out["cube12_euler_dt"] = dt
    out["cube12_euler_x10"] = r.get_state()[0]
    # full drop-in scenario
    cfg = slab_reference("slab_nonlinear_rkc_spe")
    cfg["integrator"]["t_end"] = 0.004
    cfg["output"] = {"metrics_csv": "", "probe_csv": "", "solves_csv": ""}
    n_free = pr.RefProblem(cfg).n_free
    res = pr.run_scenario(cfg, "", n_free=n_free)
    out["scenario_counts"] = np.array([res["exit_code"], res["accepted"], res["rejected"], res["m_solves"],
                                       res["pcg_iterations"]], dtype=np.int64)
    out["scenario_final_t"] = res["final_t"]
    out["scenario_x"] = res["final_x"]
    # the adaptive trajectory's conditioning: response to a 1e-12 relative change of dt0
    cfg["integrator"]["dt0"] *= 1 + 1e-12
    pert = pr.run_scenario(cfg, "", n_free=n_free)
    out["scenario_sens"] = float(np.linalg.norm(pert["final_x"] - res["final_x"]) / np.linalg.norm(res["final_x"]))
    return out


def save(name, d):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **{k: np.asarray(v) for k, v in d.items()})
    print("wrote", path, os.path.getsize(path), "bytes", flush=True)


if __name__ == "__main__":
    print("ref_small", flush=True)
    save("ref_small.npz", small())
    if "--small" in sys.argv:
        sys.exit(0)
    print("ref_c3s (24^3 jittered, C3 family)", flush=True)
    save("ref_c3s.npz", path_b(cube(24, jitter=0.1, planes=(0.45, 0.55)), [0.9], perturb_frac=0.9))
    print("ref_c1 (36^3, config 1)", flush=True)
    save("ref_c1.npz", path_b(cube(36), [0.2, 0.9], perturb_frac=0.9))
