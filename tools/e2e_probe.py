#!/usr/bin/env python
"""Break the bench's end-to-end step (set_state from pinned host memory,
rkc_advance_fixed, get_state into pinned host memory) into its parts with
host timers and CUDA events (C3 by default)."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import bench  # noqa: E402
import paper_1612_09447_b200 as eb  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
spec = bench.CONFIGS[cfg_name]
g = eb.FemSystem(bench.scenario(spec["n"], spec["jitter"], spec["planes"]), device=0)
n = g.n_free
lib = eb.load_library()
x0 = np.zeros(n)
lib.eqs_random_vec(C.c_int(n), C.c_uint(31), x0.ctypes.data_as(C.POINTER(C.c_double)))
x0 *= 2e4
g.set_state(0.0, x0, 0.0)
rho = g.spectral_radius()
dt = 0.9 * 0.653 * 15 / rho
g.set_state(0.0, x0, dt)
for _ in range(3):
    g.rkc_advance_fixed(dt, 4, 1)
x_host = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
t_host = g.get_state(out=x_host)[1]["t"]
torch.cuda.synchronize()
rows = []
for _ in range(5):
    a = time.perf_counter()
    g.set_state(t_host, x_host, dt)
    b = time.perf_counter()
    g.rkc_advance_fixed(dt, 4, 1)
    torch.cuda.synchronize()
    c = time.perf_counter()
    t_host = g.get_state(out=x_host)[1]["t"]
    d = time.perf_counter()
    rows.append((b - a, c - b, d - c))
r = np.array(rows) * 1e3
print("ms per step: set_state %.2f  advance %.2f  get_state %.2f  total %.2f" % tuple(list(r.mean(0)) + [r.sum(1).mean()]))
t0 = time.perf_counter()
for _ in range(5):
    g.rkc_advance_fixed(dt, 4, 1)
torch.cuda.synchronize()
print("device-resident advance only: %.2f ms per step" % ((time.perf_counter() - t0) * 1e3 / 5))
