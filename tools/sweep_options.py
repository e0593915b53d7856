#!/usr/bin/env python
"""Time RKC path-B steps on one GPU under eqs_set_option variants (one setup,
then per variant: reset the state, warm up, time K steps with CUDA events).

  python tools/sweep_options.py --config c3 --steps 3 --warmup 2 "3=2" "2=4" "2=8" ...

Each argument is a comma-separated list of key=value options applied on top
of the defaults (keys: include/eqs_b200.h eqs_set_option); "default" = none.
Options of one variant are reverted to the defaults listed in DEFAULTS before
the next variant."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402

DEFAULTS = {1: 2, 2: 6.0, 3: 1, 4: 2, 9: 1, 13: 0, 14: 1.1, 19: 1, 20: 1, 21: 1, 28: 0, 29: 0, 30: 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--dense-coarse", type=int, default=None)
    ap.add_argument("--vcycle-truncate", default=None, help="comma-separated per-level thresholds or 0")
    ap.add_argument("--coarse-filter", type=float, default=None)
    ap.add_argument("variants", nargs="*", default=["default"])
    args = ap.parse_args()
    bench.DENSE_COARSE = args.dense_coarse
    if args.vcycle_truncate is not None:
        vt = [float(v) for v in args.vcycle_truncate.split(",")]
        bench.VCYCLE_TRUNCATE = 0 if vt == [0.0] else vt
    bench.COARSE_FILTER = args.coarse_filter
    import torch
    import paper_1612_09447_b200 as eb
    import ctypes as C

    spec = bench.CONFIGS[args.config]
    cfg = bench.scenario(spec["n"], spec["jitter"], spec["planes"])
    t0 = time.perf_counter()
    g = eb.FemSystem(cfg, device=0)
    setup = time.perf_counter() - t0
    n = g.n_free
    lib = eb.load_library()
    x0 = np.zeros(n)
    lib.eqs_random_vec(C.c_int(n), C.c_uint(31), x0.ctypes.data_as(C.POINTER(C.c_double)))
    x0 *= 2e4
    g.set_state(0.0, x0, 0.0)
    rho = g.spectral_radius()
    dt = 0.9 * 0.653 * (bench.S_STAGES ** 2 - 1) / rho
    sp = C.c_void_p()
    lib.eqs_get_stream(g._h, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value, device=torch.device("cuda", 0))
    print(json.dumps({"setup_s": setup, "n_free": n, "rho": rho, "dt": dt}), flush=True)
    for var in args.variants:
        opts = {}
        if var != "default":
            for kv in var.split(","):
                k, v = kv.split("=")
                opts[int(k)] = float(v)
        for k, v in opts.items():
            g.set_option(k, v)
        g.set_option(12, 2)  # fresh SPE history
        g.set_state(0.0, x0, dt)
        for _ in range(args.warmup):
            g.rkc_advance_fixed(dt, bench.S_STAGES, 1)
        st0 = g.stats()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            g.rkc_advance_fixed(dt, bench.S_STAGES, 1)
        e1.record(stream)
        torch.cuda.synchronize()
        st1 = g.stats()
        fe = st1["m_solves"] - st0["m_solves"]
        print(json.dumps({"variant": var, "ms_per_step": e0.elapsed_time(e1) / args.steps,
                          "pcg_iters_per_solve": (st1["pcg_iterations"] - st0["pcg_iterations"]) / max(1, fe)}),
              flush=True)
        for k in opts:
            g.set_option(k, DEFAULTS.get(k, 0))


if __name__ == "__main__":
    main()
