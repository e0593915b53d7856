#!/usr/bin/env python
"""Benchmark of the RKC electro-quasistatic hot path (BASELINE.json metric).

One "step" = one RKC time step, path (B) of SURVEY.md §8d: rkc_advance_fixed
with s = 4 stages and dt = 0.9 beta(4)/rho(x0) on the C3 workload (215^3
jittered unit cube, 9,984,384 free dofs, nonlinear microvaristor layer), i.e.
4 F-evaluations, each = fused K(x)x + SPE start vector + AMG-PCG M-solve at
rel_tol 1e-12, plus the fused stage updates.

value = DOF-stage-updates/s = n_free x F-evaluations / device time (whole job,
summed over ranks); steps_per_s is reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4] [--impl b200|reference]

--impl reference times the reference's own CPU implementation of the path:
the unmodified reference sources compiled against an Eigen-API shim
(oracle/_ref/libeqsref.so, built by `make -C oracle ref`; the oracle/ port is
the fallback when that library is absent) on a bounded sample of the same mesh
family, with all host threads for the element kernel exactly like the
reference (PCG/AMG serial, proj/src/matfree.cpp:105).

--gpus N outside torchrun re-launches itself under torch.distributed.run with N
ranks (one per GPU, NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RKC time steps/sec & DOF-updates/sec at 1/2/4/8 B200; % HBM roofline vs CPU"
UNIT = "DOF-stage-updates/s"
S_STAGES = 4

MATERIALS = {
    "1": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}},
    "2": {"eps_r": 12.0, "conductivity": {"kind": "microvaristor", "kappa_lo": 1e-10, "kappa_hi": 3e-6,
                                          "e_switch": 5e5, "width": 5e4}},
    "3": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}},
}

# SURVEY.md §8d configurations (unit cube, hv amplitude scaled from the reference slab)
CONFIGS = {
    "c1": dict(n=36, jitter=0.0, planes=[1 / 3, 2 / 3]),
    "c2": dict(n=99, jitter=0.0, planes=[1 / 3, 2 / 3]),
    "c3": dict(n=215, jitter=0.1, planes=[0.45, 0.55]),
    "c4": dict(n=367, jitter=0.1, planes=[0.45, 0.55]),
    # config 4 weak scaling: 183 x 183 x (183 g) cubic cells on
    # [0,1]^2 x [0,g] for g GPUs (~6.2 M free dofs per GPU), the coating layer
    # repeated in every unit slab and the hv amplitude scaled by g (same fields)
    "c4w": dict(n=183, jitter=0.1, planes=[0.45, 0.55], weak=True),
}
# bounded CPU sample of the same family (same physics/planes/jitter, 48^3 cells)
CPU_SAMPLE = dict(n=48, steps=2)


COARSE_FILTER = None  # --coarse-filter: solver.amg_coarse_filter override (additive key)
VCYCLE_TRUNCATE = None  # --vcycle-truncate: solver.amg_vcycle_truncate override (additive key)
DENSE_COARSE = None  # --dense-coarse: solver.amg_dense_coarse override (additive key)


def scenario(n, jitter, planes, estimator="spe", slabs=1):
    """Unit cube (slabs = 1) or [0,1]^2 x [0,slabs] with n x n x (n slabs)
    cells, the coating layer repeated per unit slab (weak scaling)."""
    zp = [k + p for k in range(slabs) for p in planes]
    regions = [1] + [2, 1] * (slabs - 1) + [2, 3]
    return {
        "name": f"bench_cube{n}" + (f"x{slabs}" if slabs > 1 else ""),
        "mesh": {"box": {"nx": n, "ny": n, "nz": n * slabs, "lx": 1.0, "ly": 1.0, "lz": float(slabs),
                         "z_planes": zp, "regions": regions, "jitter": jitter}},
        "order": 1,
        "materials": MATERIALS,
        "excitations": {"hv": {"kind": "sinusoid", "amplitude": slabs * 4e4 / 0.012, "frequency": 50.0},
                        "ground": {"kind": "constant", "value": 0.0}},
        "solver": dict({"preconditioner": "amg", "rel_tol": 1e-12, "max_iter": 500},
                       **({} if COARSE_FILTER is None else {"amg_coarse_filter": COARSE_FILTER}),
                       **({} if VCYCLE_TRUNCATE is None else {"amg_vcycle_truncate": VCYCLE_TRUNCATE}),
                       **({} if DENSE_COARSE is None else {"amg_dense_coarse": DENSE_COARSE})),
        "estimator": {"mode": estimator, "window": 8},
    }


def host_mem_available():
    """MemAvailable of /proc/meminfo in bytes (0 when unknown)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def ncu_traffic(config_name):
    """DRAM bytes per launch of each timing class from the committed ncu launch
    list of this workload (tools/ncu_traffic.py -> profiles/ncu_traffic_<config>.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{config_name}.json")) as f:
            return json.load(f).get("dram_bytes_per_launch", {})
    except OSError:
        return {}


def fp64_csr_equivalent(g, iters, ms, steps, hbm, other_bytes, dense_rows):
    """SURVEY.md §8d bytes of the same V-cycle passes if every operator were
    fp64 CSR (12 B/entry + 4 B/row) with fp64 vectors, on the reference's
    (unfiltered) Galerkin hierarchy: fine level 4 smoother/residual passes
    (Chebyshev(2) pre and post), coarse levels 2 (Chebyshev(1)), restriction
    and prolongation per level, dense solve of the first level with at most
    `dense_rows` rows. Single-rank contexts only (host copies of P, R)."""
    try:
        L = len(g.amg_levels())
        dims = [[tuple(int(v) for v in _level_dims(g, l, w)) for w in range(3)] for l in range(L)]
    except Exception as e:  # noqa: BLE001 - reported in the line
        return {"unavailable": str(e)}
    total = 0.0
    for l in range(L):
        n_l, _, nnz_a = dims[l][0]
        if n_l <= dense_rows or l == L - 1:
            total += 8.0 * n_l * n_l + 16.0 * n_l
            break
        passes = 4 if l == 0 else 2
        total += passes * (12.0 * nnz_a + 4.0 * (n_l + 1) + 32.0 * n_l)
        nr, nc, nnz_r = dims[l][2]
        total += 12.0 * nnz_r + 4.0 * (nr + 1) + 8.0 * nc + 8.0 * nr
        npr, npc, nnz_p = dims[l][1]
        total += 12.0 * nnz_p + 4.0 * (npr + 1) + 8.0 * npc + 16.0 * npr
    n = dims[0][0][0]
    nnz_m = dims[0][0][2]
    spmv = 12.0 * nnz_m + 4.0 * (n + 1) + 16.0 * n
    per_iter_pcg = spmv + 16.0 * n + 48.0 * n + 16.0 * n + 24.0 * n
    vc_total = iters * total
    step_bytes = (vc_total + iters * per_iter_pcg + other_bytes) / steps
    return {"vcycle_bytes": total, "pcg_iteration_vector_and_spmv_bytes": per_iter_pcg,
            "step_bytes": step_bytes,
            "achieved_full_step": step_bytes * steps / (ms / 1e3) / 1e9,
            "frac_full_step": step_bytes * steps / (ms / 1e3) / 1e9 / hbm,
            "rule": "SURVEY.md §8d fp64-CSR formulas on the reference hierarchy (unfiltered A_l, explicit P/R), "
                    "this V-cycle's pass counts, PCG canonical fused form; K(x)x/RKC/SPE bytes as counted"}


def _level_dims(g, level, which):
    import ctypes as C
    dims = np.zeros(3, dtype=np.int32)
    import paper_1612_09447_b200 as eb
    rc = eb.load_library().eqs_amg_level_csr(g._h, C.c_int(level), C.c_int(which),
                                             dims.ctypes.data_as(C.POINTER(C.c_int)), None, None, None)
    if rc != 0:
        raise RuntimeError(f"eqs_amg_level_csr rc {rc}")
    return dims


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


# ------------------------------------------------------------------ CPU (reference) leg
def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


class CpuArm:
    """The reference's CPU path: oracle/_ref (unmodified reference sources,
    kind "reference") when built, else the oracle/ restatement (kind "port").
    Checker / baseline only, never the measured product."""

    def __init__(self, cfg, cores):
        from oracle import pyref as pr  # checker / baseline only
        if pr.available():
            self.kind, self.p = "reference", pr.RefProblem(cfg, workers=cores)
        else:
            from oracle import pyoracle as po
            self.kind, self.p = "port", po.Problem(cfg, workers=cores)
        self.n_free = self.p.n_free
        self.t = 0.0
        self.x = None

    def spectral_radius(self, x):
        return self.p.spectral_radius(0.0, x)

    def set_state(self, t, x, dt):
        self.t, self.x = t, np.array(x, dtype=np.float64, copy=True)
        if self.kind == "reference":
            self.p.set_state(t, self.x, dt)

    def advance(self, dt, s, steps):
        if self.kind == "reference":
            self.p.rkc_advance_fixed(dt, s, steps)
            self.x, self.t, _ = self.p.get_state()
        else:
            self.x = self.p.rkc_advance_fixed(self.t, self.x, dt, s, steps)
            self.t += steps * dt

    def iters_per_solve(self):
        st = self.p.stats()
        return st["pcg_iterations"] / max(1, st["m_solves"])

    def describe(self, cores):
        what = ("unmodified reference sources (proj/src) compiled against the Eigen-API shim oracle/ref_shim "
                "(oracle/_ref/libeqsref.so, -O3, no -march)" if self.kind == "reference" else
                "oracle/ C++ restatement of the reference (oracle/_ref not built)")
        return (f"{what}; OpenMP element kernel with {cores} threads, serial PCG with the SGS-smoothed SA-AMG V-cycle "
                f"as in the reference (proj/src/matfree.cpp:105-115)")


def sample_x0_dt(arm):
    from oracle import pyoracle as po  # random_vec: mt19937 uniform[-1,1) (test_helpers.hpp:15-21)
    x0 = 2e4 * po.random_vec(arm.n_free, 31)
    rho = arm.spectral_radius(x0)
    return x0, 0.9 * 0.653 * (S_STAGES ** 2 - 1) / rho, rho


def cpu_sample(steps, cores):
    """Time the reference's CPU path on the bounded sample (48^3 cube of the C3
    family) and keep its state for the parity check against the GPU."""
    cfg = scenario(CPU_SAMPLE["n"], 0.1, [0.45, 0.55])
    arm = CpuArm(cfg, cores)
    x0, dt, rho = sample_x0_dt(arm)
    arm.set_state(0.0, x0, dt)
    t0 = time.perf_counter()
    arm.advance(dt, S_STAGES, steps)
    wall = time.perf_counter() - t0
    return {"value": arm.n_free * S_STAGES * steps / wall, "steps_per_s": steps / wall, "arm": arm, "x0": x0,
            "dt": dt, "x": arm.x.copy(), "cfg": cfg, "iters": arm.iters_per_solve(),
            "desc": (f"{arm.describe(cores)}; {CPU_SAMPLE['n']}^3 jittered cube of the C3 family ({arm.n_free} "
                     f"free dofs), {steps} RKC steps path B (s=4, dt=0.9 beta(4)/rho), stepping time only")}


def sample_parity(sample, steps, cores):
    """GPU vs the reference on the CPU sample: same x0, dt and steps; the gate is
    10x the reference's own response to a 1e-12 perturbation of x0 and to a
    PCG tolerance of 1e-13 (tests/test_gpu_ref_parity.py)."""
    import copy

    import paper_1612_09447_b200 as eb
    g = eb.FemSystem(sample["cfg"], device=0)
    g.set_state(0.0, sample["x0"], sample["dt"])
    g.rkc_advance_fixed(sample["dt"], S_STAGES, steps)
    xg = g.get_state()[0]
    g.close()
    xr = sample["x"]
    rel = float(np.linalg.norm(xg - xr) / np.linalg.norm(xr))
    pert = CpuArm(sample["cfg"], cores)
    pert.set_state(0.0, sample["x0"] * (1 + 1e-12), sample["dt"])
    pert.advance(sample["dt"], S_STAGES, steps)
    sens = float(np.linalg.norm(pert.x - xr) / np.linalg.norm(xr))
    tight_cfg = copy.deepcopy(sample["cfg"])
    tight_cfg["solver"]["rel_tol"] = 1e-13
    tight = CpuArm(tight_cfg, cores)
    tight.set_state(0.0, sample["x0"], sample["dt"])
    tight.advance(sample["dt"], S_STAGES, steps)
    sens_tol = float(np.linalg.norm(tight.x - xr) / np.linalg.norm(xr))
    gate = 10.0 * max(sens, sens_tol, 1e-13)
    return {"sample": f"{CPU_SAMPLE['n']}^3 C3-family cube, x0 = 2e4 random_vec(31), {steps} RKC steps path B",
            "against": sample["arm"].kind, "rel_l2_gpu_vs_reference": rel,
            "reference_response_1e-12_x0": sens, "reference_response_tol_1e-13": sens_tol, "gate": gate,
            "pass": rel <= gate}


def c3_cpu_record():
    """The committed full-size C3 measurement of the reference's CPU path
    (tools/cpu_c3_baseline.py -> profiles/CPU_r2_c3.json), if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "CPU_r2_c3.json")) as f:
            return json.load(f)
    except OSError:
        return None


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    cfg = scenario(CPU_SAMPLE["n"], 0.1, [0.45, 0.55])
    arm = CpuArm(cfg, cores)
    x0, dt, _ = sample_x0_dt(arm)
    arm.set_state(0.0, x0, dt)
    for _ in range(args.warmup):
        arm.advance(dt, S_STAGES, 1)
    it0 = arm.p.stats()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        arm.advance(dt, S_STAGES, 1)
    wall = time.perf_counter() - t0
    it1 = arm.p.stats()
    value = arm.n_free * S_STAGES * args.steps / wall
    sample = (f"{CPU_SAMPLE['n']}^3 jittered cube of the C3 family ({arm.n_free} free dofs), RKC path B s=4, "
              f"{args.steps} timed steps after {args.warmup} warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "steps_per_s": args.steps / wall, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cpu sample of {args.config}: {sample}", "n_free": arm.n_free},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": arm.kind, "cpu_model": cpu_model(),
                         "sample": arm.describe(cores) + "; " + sample,
                         "pcg_iters_per_solve": (it1["pcg_iterations"] - it0["pcg_iterations"])
                         / max(1, it1["m_solves"] - it0["m_solves"])},
        "c3_full_size_record": c3_cpu_record(),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 leg
def apply_options(g, args):
    if args.vcycle_values:
        g.set_option(4, {"fp64": 0, "fp32": 1, "bf16": 2}[args.vcycle_values])
    for kv in args.opt or []:  # eqs_set_option keys (include/eqs_b200.h), for sweeps
        k, v = kv.split("=")
        g.set_option(int(k), float(v))


def single_gpu_system(args, estimator=None):
    import torch
    import paper_1612_09447_b200 as eb

    if not torch.cuda.is_available():
        raise RuntimeError("bench.py needs a CUDA device (no CPU fallback)")
    spec = CONFIGS[args.config]
    cfg = scenario(spec["n"], spec["jitter"], spec["planes"], estimator=estimator or args.estimator)
    t0 = time.perf_counter()  # (weak configs: one slab on one GPU)
    g = eb.FemSystem(cfg, device=0)
    apply_options(g, args)
    return g, time.perf_counter() - t0, eb


def run_euler_vs_rkc(args):
    """Config 2: explicit Euler at dt = min(dt0, 1.8/rho)
    (scenario.cpp:286-293) against RKC path B (s = 4, dt = 0.9 beta(4)/rho) on
    the same state, one GPU. Both report simulated seconds per wall second and
    DOF-stage-updates/s (device time, CUDA events)."""
    import ctypes as C
    import torch

    rank, world, _ = dist_env()
    if rank != 0:
        return
    g, t_setup, eb = single_gpu_system(args)
    n = g.n_free
    lib = eb.load_library()
    x0 = np.zeros(n)
    lib.eqs_random_vec(C.c_int(n), C.c_uint(31), x0.ctypes.data_as(C.POINTER(C.c_double)))
    x0 *= 2e4
    g.set_state(0.0, x0, 0.0)
    rho = g.spectral_radius()
    sp = C.c_void_p()
    lib.eqs_get_stream(g._h, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", 0))
    out = {}
    for name, dt, run in (("euler", min(1e-5, 1.8 / rho), lambda dt: g.euler_step(dt)),
                          ("rkc", 0.9 * 0.653 * (S_STAGES ** 2 - 1) / rho,
                           lambda dt: g.rkc_advance_fixed(dt, S_STAGES, 1))):
        g.set_state(0.0, x0, dt)
        for _ in range(args.warmup):
            run(dt)
        st0 = g.stats()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            run(dt)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        st1 = g.stats()
        fe = st1["m_solves"] - st0["m_solves"]
        out[name] = {"dt": dt, "ms_per_step": ms / args.steps, "f_evals_per_step": fe / args.steps,
                     "pcg_iters_per_solve": (st1["pcg_iterations"] - st0["pcg_iterations"]) / max(1, fe),
                     "simulated_s_per_wall_s": dt * args.steps / (ms / 1e3),
                     "dof_stage_updates_per_s": n * fe / (ms / 1e3)}
    line = {"metric": "config 2: Euler vs RKC, simulated seconds per wall second (RKC path B vs Euler at 1.8/rho)",
            "value": out["rkc"]["simulated_s_per_wall_s"], "unit": "simulated s / wall s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "dtype": "f64",
            "data": "synthetic", "rho": rho, "rkc_over_euler": out["rkc"]["simulated_s_per_wall_s"]
            / out["euler"]["simulated_s_per_wall_s"],
            "config": {"workload": f"{args.config} cube, x0 = 2e4*random_vec(31), {n} free dofs",
                       "n_free": n}, "setup_s": t_setup, **out}
    print(json.dumps(line), flush=True)


def run_sdirk_vs_rkc(args):
    """Explicit vs implicit time to t_end (§V, Fig. 2): adaptive RKC
    (rkc_step, tol 1e-2, integrators.cpp:177-225) against adaptive SDIRK3(2)
    (sdirk_step, tol 1e-2, Newton 1e-8, integrators.cpp:297-327) whose shifted
    system M + gamma dt K(z) is re-assembled every Newton iteration and
    preconditioned with the SA-AMG rebuilt on the device once per step (the
    reference's make_preconditioner refresh, fem_system.cpp:124-145), and with
    Jacobi as a third arm. Same state, one GPU, device time (CUDA events)."""
    import ctypes as C
    import torch

    rank, world, _ = dist_env()
    if rank != 0:
        return
    g, t_setup, eb = single_gpu_system(args)
    n = g.n_free
    lib = eb.load_library()
    x0 = np.zeros(n)
    lib.eqs_random_vec(C.c_int(n), C.c_uint(31), x0.ctypes.data_as(C.POINTER(C.c_double)))
    x0 *= 2e4
    sp = C.c_void_p()
    lib.eqs_get_stream(g._h, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", 0))
    t_end, cap = args.t_end, 2000
    out = {}
    for name, step, opt in (("rkc", lambda: g.rkc_step(rtol=1e-2, atol=1e-8), None),
                            ("sdirk_amg", lambda: g.sdirk_step(rtol=1e-2, atol=1e-8, newton_tol=1e-8), 1),
                            ("sdirk_jacobi", lambda: g.sdirk_step(rtol=1e-2, atol=1e-8, newton_tol=1e-8), 0)):
        if opt is not None:
            g.set_option(26, opt)
        g.set_state(0.0, x0, 1e-5)
        st0 = g.stats()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        ev0.record(stream)
        t, acc, rej = 0.0, 0, 0
        while t < t_end and acc + rej < cap:
            a = step()
            acc += a.accepted
            rej += not a.accepted
            t = a.t_start + (a.dt if a.accepted else 0.0)
        ev1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        st1 = g.stats()
        d = {k: st1[k] - st0[k] for k in ("m_solves", "pcg_iterations", "newton_linear_solves",
                                            "newton_pcg_iterations", "precond_setups", "assemblies",
                                            "time_residual", "time_solve", "time_setup", "time_estimator")}
        out[name] = {"t_reached": t, "accepted": acc, "rejected": rej, "device_s": ev0.elapsed_time(ev1) / 1e3,
                     "wall_s": wall, **d}
    line = {"metric": "explicit RKC vs implicit SDIRK3(2): time to t_end (PAPER.md Fig. 2)",
            "value": out["sdirk_amg"]["wall_s"] / out["rkc"]["wall_s"], "unit": "speed-up of RKC over SDIRK+AMG",
            "n_gpus": 1, "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} cube, x0 = 2e4*random_vec(31), {n} free dofs, t_end {t_end}",
                       "n_free": n}, "setup_s": t_setup,
            "rkc_over_sdirk_jacobi": out["sdirk_jacobi"]["wall_s"] / out["rkc"]["wall_s"], **out}
    print(json.dumps(line), flush=True)


def mrhs_rhs(g, n_rhs=40):
    """Config 5 right-hand sides: b_k = M_II x*_k, x*_k = sum_{m=1..3} cos(2 pi m k/40) phi_m,
    phi_m = sin(m pi z) cos(pi x) cos(pi y) at the free dofs."""
    nodes, _, _ = g.mesh()
    _, free, _ = g.dofs()
    xyz = nodes[free]
    phi = [np.sin(m * np.pi * xyz[:, 2]) * np.cos(np.pi * xyz[:, 0]) * np.cos(np.pi * xyz[:, 1]) for m in (1, 2, 3)]
    X = np.stack([sum(np.cos(2 * np.pi * m * k / 40) * phi[m - 1] for m in (1, 2, 3)) for k in range(n_rhs)])
    B = np.stack([g.mass_apply(X[k]) for k in range(n_rhs)])
    return X, B


def run_mrhs(args):
    """Config 5: the 40-RHS sequence solved to 1e-12 with zero / previous /
    SPE(8) / POD start vectors, inputs resident (eqs_mass_solve_sequence)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    g, t_setup, eb = single_gpu_system(args)
    X, B = mrhs_rhs(g)
    n = g.n_free
    res = {}
    # POD modes (start_vector.cpp:111-131): pod_fixed builds its rank-10 basis
    # from the first 8 solutions, pod_rolling keeps a ring of 20 (reference default)
    g.set_option(15, 8)
    for mode, key in (("zero", 0), ("previous", 1), ("spe", 2), ("pod_fixed", 3), ("pod_rolling", 4)):
        g.set_option(12, key)
        g.mass_solve_sequence(B[:4])  # warm-up (graphs, buffers)
        g.set_option(12, key)
        its, ms, Xs = g.mass_solve_sequence(B, want_x=(mode == "spe"))
        res[mode] = {"iters_total": int(its.sum()), "iters_per_solve": float(its.mean()),
                     "iters_per_solve_k_ge_8": float(its[8:].mean()), "ms_total": ms,
                     "solves_per_s": len(its) / (ms / 1e3), "iterations": its.tolist()}
        if Xs is not None:
            res[mode]["max_rel_err"] = float(max(np.linalg.norm(Xs[k] - X[k]) / np.linalg.norm(X[k])
                                                 for k in range(len(X))))
    line = {"metric": "config 5: MRHS sequence (40 RHS, PCG+AMG 1e-12), solves/s with SPE(8) starts",
            "value": res["spe"]["solves_per_s"], "unit": "solves/s", "n_gpus": 1, "higher_is_better": True,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"M_II of {args.config} ({n} free dofs), b_k = M_II x*_k, k = 0..39"},
            "spe_iters_vs_zero": res["spe"]["iters_total"] / res["zero"]["iters_total"],
            "pod_fixed_iters_vs_zero": res["pod_fixed"]["iters_total"] / res["zero"]["iters_total"],
            "pod_rolling_iters_vs_zero": res["pod_rolling"]["iters_total"] / res["zero"]["iters_total"],
            "setup_s": t_setup, **res}
    print(json.dumps(line), flush=True)


def run_b200(args):
    rank, world, local_rank = dist_env()
    if world > 1 and "OMP_NUM_THREADS" not in os.environ:
        # host setup of every rank runs concurrently: share the cores
        os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // world))
    if world > 1 and "EQS_SETUP_CONCURRENCY" not in os.environ:
        # every rank builds the global problem before extracting its partition
        # (~2.5 kB of host memory per global free dof at the peak): bound how
        # many ranks of the node do so at once (capi.cpp SetupGate)
        spec0 = CONFIGS[args.config]
        slabs = world if spec0.get("weak") else 1
        n_glob = (spec0["n"] + 1) ** 2 * (spec0["n"] * slabs - 1)
        avail = host_mem_available()
        k = max(1, int(0.8 * avail / (2.5e3 * n_glob))) if avail else world
        os.environ["EQS_SETUP_CONCURRENCY"] = str(min(world, k))
    import torch
    import paper_1612_09447_b200 as eb

    if not torch.cuda.is_available():
        raise RuntimeError("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    spec = CONFIGS[args.config]
    weak = bool(spec.get("weak"))
    cfg = scenario(spec["n"], spec["jitter"], spec["planes"], estimator=args.estimator, slabs=world if weak else 1)
    t_setup = time.perf_counter()
    if world > 1:
        # one C3 problem partitioned by node ownership over the ranks (strong
        # scaling); halos and dot products over NCCL (csrc/comm.cpp)
        obj = [eb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        g = eb.FemSystem.distributed(cfg, local_rank, world, rank, obj[0])
        owned = g.partition(0)["owned"]
    else:
        g = eb.FemSystem(cfg, device=local_rank)
        owned = None
    apply_options(g, args)
    t_setup = time.perf_counter() - t_setup
    n = g.n_free
    lib = eb.load_library()
    x0 = np.zeros(n)
    import ctypes as C
    lib.eqs_random_vec(C.c_int(n), C.c_uint(31), x0.ctypes.data_as(C.POINTER(C.c_double)))
    x0 *= 2e4
    if owned is not None:
        x0 = np.ascontiguousarray(x0[owned])
    g.set_state(0.0, x0, 0.0)
    rho = g.spectral_radius()
    dt = 0.9 * 0.653 * (S_STAGES ** 2 - 1) / rho
    g.set_state(0.0, x0, dt)
    stream_ptr = C.c_void_p()
    lib.eqs_get_stream(g._h, C.byref(stream_ptr))
    stream = torch.cuda.ExternalStream(stream_ptr.value, device=torch.device("cuda", local_rank))

    for _ in range(args.warmup):
        g.rkc_advance_fixed(dt, S_STAGES, 1)
    st0 = g.stats()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.eqs_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            g.rkc_advance_fixed(dt, S_STAGES, 1)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = lib.eqs_launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    st1 = g.stats()
    # e2e: the same step through the public API with host buffers: every step
    # copies the state in from pinned host memory (H2D) and back out (D2H);
    # measured right after the timed region (same thermal / power-cap state)
    x_host = torch.empty(g.n_own, dtype=torch.float64, pin_memory=True).numpy()
    g.get_state(out=x_host)
    t_host = g.get_state(want_x=False)[1]["t"]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = time.perf_counter()
    e_steps = max(1, min(args.steps, 5))
    for _ in range(e_steps):
        g.set_state(t_host, x_host, dt)
        g.rkc_advance_fixed(dt, S_STAGES, 1)
        t_host = g.get_state(out=x_host)[1]["t"]
    e_wall = time.perf_counter() - e0
    if dist:
        t = torch.tensor([e_wall], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_wall = float(t.item())
    e2e_value = n * S_STAGES * e_steps / e_wall
    # per-class breakdown for the roofline: CUDA events around every kernel
    # class on the library stream, in a second pass of K steps after the
    # timed region (the events add host work, so they stay out of `value`)
    g.timing(True)
    g.timing_reset()
    for _ in range(args.steps):
        g.rkc_advance_fixed(dt, S_STAGES, 1)
    torch.cuda.synchronize()
    timing = g.timing()
    g.timing(False)
    # third pass, graph path: the graph-resident PCG (the timed region's code
    # path) as one event region per solve (class 6), the other classes as above
    g.set_option(24, 1)
    st_g0 = g.stats()
    g.timing(True)
    g.timing_reset()
    for _ in range(args.steps):
        g.rkc_advance_fixed(dt, S_STAGES, 1)
    torch.cuda.synchronize()
    timing_g = g.timing()
    g.timing(False)
    g.set_option(24, 0)
    iters_g = g.stats()["pcg_iterations"] - st_g0["pcg_iterations"]
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    f_evals = st1["m_solves"] - st0["m_solves"]
    iters = st1["pcg_iterations"] - st0["pcg_iterations"]
    value = n * f_evals / (ms / 1e3)  # n = global free dofs: all ranks together

    import resource
    rss_gb = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peaks, peak_kind = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    traffic = ncu_traffic(args.config)
    # roofline of the dominant kernel class (TimeClass in gpu_system.hpp): per-class
    # device time from CUDA events on the library stream, algorithmic bytes per launch
    names = ["stiffness K(x)x", "pcg spmv+vectors", "v-cycle", "rkc stage/error", "spe estimator", "boundary"]
    kernels = {0: "K(x)x blocked stiffness operator (k_kx_block<4> + k_kx_partials)",
               1: "PCG fine-level M_II SpMV+dot (fp64 stencil-coded SELL-S k_sells64<0>; SELL-16 k_sell_red on "
                  "unstructured meshes) and fused x/r update (k_pcg_update)",
               2: "AMG V-cycle: stencil-coded SELL-S (fine level) and packed SELL-P (transfers, coarse levels) bf16 "
                  "smoother/residual/transfer row kernels, dense coarse GEMV"}

    def roof(c, timing=timing):
        if not (timing["launches"][c] and timing["bytes"][c]):
            return None
        avg_ms = timing["ms"][c] / timing["launches"][c]
        per = timing["bytes"][c] / timing["launches"][c]
        ach = per / (avg_ms / 1e3) / 1e9
        tr = traffic.get(names[c])
        return {"kernel": kernels[c], "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                "frac": ach / hbm, "traffic": tr, "traffic_source": f"profiles/ncu_traffic_{args.config}.json"
                if tr else None, "bytes_per_launch": per, "avg_launch_ms": avg_ms,
                "share_of_step": timing["ms"][c] / sum(timing["ms"][:6]),
                "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs"}

    # graph path (what the timed region runs): the whole PCG loop per solve is
    # one event region (class 6); its V-cycle / SpMV+vectors split is the
    # host-loop pass's time ratio, its bytes are the captured body's bytes
    # (iterations x (V-cycle + direction + SpMV + update)), the V-cycle part
    # is iterations x the V-cycle's algorithmic bytes
    n_tets_all = g.n_tets
    v_per = timing["bytes"][2] / max(1, timing["launches"][2])
    host_vp = timing["ms"][1] + timing["ms"][2]
    vshare = timing["ms"][2] / host_vp if host_vp else 0.0
    g_ms = list(timing_g["ms"])
    g_by = list(timing_g["bytes"])
    g_ms[2] = g_ms[2] + vshare * g_ms[6]
    g_ms[1] = g_ms[1] + (1.0 - vshare) * g_ms[6]
    g_by[2] = g_by[2] + iters_g * v_per
    g_by[1] = g_by[1] + max(0.0, g_by[6] - iters_g * v_per)
    g_n = list(timing_g["launches"])
    g_n[2] = g_n[2] + iters_g
    g_n[1] = g_n[1] + 2 * iters_g
    timing_graph = {"ms": g_ms[:6], "bytes": g_by[:6], "launches": g_n[:6]}

    def roof_g(c):
        r = roof(c, timing_graph)
        if r:
            r["time_source"] = ("graph path: CUDA events around each graph-resident PCG solve; its V-cycle share "
                                f"({vshare:.3f}) from the host-loop pass")
        return r

    # the dominant class (largest device time) is the headline roofline
    cls = max(range(3), key=lambda c: timing_graph["ms"][c])
    dom = roof_g(cls)
    others = {names[c]: roof_g(c) for c in range(3) if c != cls}
    # K(x)x: SURVEY.md §8d asks for both fractions (HBM and FP64 pipe). fp64
    # operations per P1 tet of k_kx_block4's residual form (linear material:
    # 9 edge differences, 3 cofactor rows 27, det 5, x differences 3, w 15,
    # |w|^2 5, 1/det 1, kappa/(6 det) 2, y_1..3 18, y_0 3); the peak is the
    # spec-derived B200 vector FP64 rate (148 SMs x 64 FMA/clk x 2 x 1.965 GHz)
    kx = others.get(names[0]) or (dom if cls == 0 else None)
    if kx:
        flops = 88.0 * n_tets_all
        kx["fp64"] = {"flops_per_tet": 88, "achieved_tflops": flops / (kx["avg_launch_ms"] / 1e3) / 1e12,
                      "peak_tflops": 37.2, "frac": flops / (kx["avg_launch_ms"] / 1e3) / 37.2e12,
                      "peak_source": "spec-derived (148 SMs x 64 FP64 FMA/clk x 2 flops x 1.965 GHz), not measured"}
    host_loop = {names[c]: roof(c) for c in range(3)}
    n_tets, nnz_mass, amg_levels = g.n_tets, g.nnz_mass_free, g.amg_levels()
    csr64 = (fp64_csr_equivalent(g, iters_g, ms, args.steps, hbm, g_by[0] + g_by[3] + g_by[4] + g_by[5],
                                 DENSE_COARSE if DENSE_COARSE is not None else 512) if world == 1 else None)
    cpu = parity = None
    if world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        g.close()  # free the C3 system before the sample's GPU parity run
        smp = cpu_sample(CPU_SAMPLE["steps"], cores)
        cpu = {"value": smp["value"], "unit": UNIT, "cores": cores, "kind": smp["arm"].kind,
               "cpu_model": cpu_model(), "pcg_iters_per_solve": smp["iters"], "sample": smp["desc"],
               "c3_full_size_record": c3_cpu_record()}
        parity = sample_parity(smp, CPU_SAMPLE["steps"], cores)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "steps_per_s": 1e3 * args.steps / ms,
        "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated mesh + mt19937 initial state; no dataset)",
        "config": {"workload": (f"{args.config}: {spec['n']}x{spec['n']}x{spec['n'] * world} "
                                f"{'jittered ' if spec['jitter'] else ''}box [0,1]^2x[0,{world}] (weak scaling), "
                                if weak else
                                f"{args.config}: {spec['n']}^3 {'jittered ' if spec['jitter'] else ''}unit cube, ")
                               + f"{n} free dofs, {n_tets} tets, microvaristor layer z in {spec['planes']}, "
                               f"RKC path B s={S_STAGES} dt=0.9*beta(4)/rho (={dt:.4g}s), "
                               f"estimator {args.estimator} + AMG-PCG 1e-12",
                   "estimator": args.estimator,
                   "n_free": n, "n_tets": n_tets, "nnz_mass_free": nnz_mass,
                   "amg_levels": amg_levels,
                   "precision": {
                       "operator_pcg_and_result": "fp64: M_II (fp64 stencil-coded SELL-S, same products and row "
                                                  "order as CsrMatrix::apply), PCG vectors, dots, stopping rule "
                                                  "rel_tol 1e-12, K(x)x, RKC stages",
                       "vcycle_preconditioner": "bf16 matrix values (packed SELL-S/SELL-P; fine-level rows carry "
                                                "their bf16 row-sum correction), fp32 vectors, Chebyshev(2) fine / "
                                                "(1) coarse smoothing instead of SGS, prolongators of levels 0-2 "
                                                "truncated for the V-cycle with the coarser Galerkin operators "
                                                "recomputed "
                                                "(DESIGN.md §4.1-4.2, 4.12-4.13; the reported amg_levels are the "
                                                "reference hierarchy)",
                       "vcycle_truncate": VCYCLE_TRUNCATE if VCYCLE_TRUNCATE is not None else [0.1, 0.15, 0.03],
                       "coarse_filter_eps": COARSE_FILTER if COARSE_FILTER is not None else 0.0025,
                       "dense_coarse_rows": DENSE_COARSE if DENSE_COARSE is not None else 512},
                   "parallelism": (f"node-ownership partition over {world} GPUs (owner-computes K(x)x, halo "
                                   f"SpMV + NCCL allreduce per level, small coarse levels replicated; host setup "
                                   f"{os.environ.get('EQS_SETUP_CONCURRENCY', world)} ranks at a time)")
                   if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (matrices + vectors >> 126 MB), no flush needed"},
        "pcg_iters_per_solve": iters / max(1, f_evals), "f_evals_per_step": f_evals / args.steps,
        "setup_s": t_setup, "rho": rho, "host_peak_rss_gb_rank0": rss_gb,
        "clocks": clocks.summary(),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                "steps": e_steps},
        "gpu_launches": launches,
        "roofline": dom,
        "roofline_other_classes": others,
        "roofline_host_loop": host_loop,
        # whole step: all classes' algorithmic bytes of the
        # graph-path pass / the un-instrumented step time (both K steps)
        "roofline_full_step": {"bound": "hbm", "achieved": sum(timing_graph["bytes"]) / (ms / 1e3) / 1e9,
                               "peak": hbm, "unit": "GB/s",
                               "frac": sum(timing_graph["bytes"]) / (ms / 1e3) / 1e9 / hbm,
                               "frac_vs_8tbs_spec": sum(timing_graph["bytes"]) / (ms / 1e3) / 8e12,
                               "bytes_per_step": sum(timing_graph["bytes"]) / args.steps},
        "bytes_counted_as": ("algorithmic bytes of the stored formats: bf16 SELL-S at 2 B/entry + 1 B/row and "
                             "packed SELL-P at 4 B/entry in the V-cycle, fp64 SELL-S at 8 B/entry for M_II, "
                             "SURVEY.md §8d per-tet/per-dof figures for K(x)x; fp32 V-cycle vectors"),
        "fp64_csr_equivalent": csr64,
        "time_by_class_ms": {names[c]: timing_graph["ms"][c] for c in range(6)},
        "time_by_class_source": ("graph path (third pass of K steps): CUDA events around K(x)x, SPE, RKC and each "
                                 "whole graph-resident PCG solve; PCG split into V-cycle / SpMV+vectors by the "
                                 "host-loop pass (second pass, per-class events)"),
        "time_by_class_host_loop_ms": {names[c]: timing["ms"][c] for c in range(6)},
        "bytes_by_class": {names[c]: timing_graph["bytes"][c] for c in range(6)},
        "cpu_baseline": cpu,
        "parity": parity,
        "parity_rel": parity["rel_l2_gpu_vs_reference"] if parity else None,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--coarse-filter", type=float, default=None,
                    help="solver.amg_coarse_filter (V-cycle coarse-operator filter, DESIGN.md §4)")
    ap.add_argument("--vcycle-truncate", default=None,
                    help="solver.amg_vcycle_truncate: comma-separated per-level prolongator truncation thresholds "
                         "for the V-cycle, or 0 = off (DESIGN.md §4.13; default 0.1,0.15,0.03)")
    ap.add_argument("--dense-coarse", type=int, default=None,
                    help="solver.amg_dense_coarse (dense explicit-inverse solve from the first level with at "
                         "most this many rows, DESIGN.md §4)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the in-run CPU baseline sample")
    ap.add_argument("--estimator", default="spe", choices=["zero", "previous", "spe"],
                    help="MRHS start vectors (proj/src/start_vector.cpp); the reference nonlinear scenario uses spe")
    ap.add_argument("--vcycle-values", default=None, choices=["fp64", "fp32", "bf16"],
                    help="V-cycle matrix value precision (library default when omitted)")
    ap.add_argument("--opt", action="append", help="KEY=VALUE eqs_set_option before the run (repeatable)")
    ap.add_argument("--t-end", type=float, default=1e-3, help="--mode sdirk: simulated interval")
    ap.add_argument("--mode", default="rkc", choices=["rkc", "euler", "mrhs", "sdirk"],
                    help="rkc: the headline line (default); euler: config 2 Euler vs RKC on --config (c2); "
                         "mrhs: config 5 multiple-right-hand-side sequence on --config")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (127.0.0.1 rendezvous)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    global COARSE_FILTER, DENSE_COARSE, VCYCLE_TRUNCATE
    COARSE_FILTER = args.coarse_filter
    if args.vcycle_truncate is not None:
        vt = [float(v) for v in str(args.vcycle_truncate).split(",")]
        VCYCLE_TRUNCATE = 0 if vt == [0.0] else vt
    DENSE_COARSE = args.dense_coarse
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "euler":
        run_euler_vs_rkc(args)
    elif args.mode == "mrhs":
        run_mrhs(args)
    elif args.mode == "sdirk":
        run_sdirk_vs_rkc(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
