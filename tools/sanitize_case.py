#!/usr/bin/env python
"""Small end-to-end case for compute-sanitizer (racecheck /
memcheck / synccheck on the hot kernels):

  compute-sanitizer --tool racecheck python tools/sanitize_case.py
  compute-sanitizer --tool memcheck  python tools/sanitize_case.py

Runs the blocked K(x)x (shared-memory products, k_kx_block + k_kx_partials),
the coloured and two-pass modes, a mass solve with the AMG V-cycle, two RKC
steps with the SPE estimator (graph-resident PCG) and, when asked, the P2
blocked kernel. Sizes are small so racecheck finishes in minutes; the kx block
size is lowered so the case has many blocks and block-boundary partials."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1612_09447_b200 as eb  # noqa: E402
from helpers import cube  # noqa: E402


def run(order, n):
    cfg = cube(n, jitter=0.1, order=order, planes=(0.45, 0.55))
    g = eb.FemSystem(cfg, device=0)
    if os.environ.get("SAN_NOGRAPH") == "1":  # host-driven PCG, no V-cycle graph, no PDL
        for key in (8, 20, 21):
            g.set_option(key, 0)
    if os.environ.get("SAN_NOPDL") == "1":  # graphs on, programmatic dependent launch off
        g.set_option(21, 0)
    if os.environ.get("SAN_NOLOOP") == "1":  # V-cycle graphs + PDL on, no conditional (WHILE) PCG graph
        g.set_option(20, 0)
    rng = np.random.default_rng(5)
    x = 2e4 * rng.standard_normal(g.n_dofs)
    v = rng.standard_normal(g.n_dofs)
    outs = []
    for mode in (0, 1, 2):  # blocked, coloured, two-pass gather (eqs_set_option 0)
        g.set_option(0, mode)
        outs.append(g.kx_apply(x, v))
    g.set_option(0, 0)
    spread = max(np.abs(o - outs[0]).max() for o in outs) / np.abs(outs[0]).max()
    b = rng.standard_normal(g.n_free)
    xs, _ = g.mass_solve(b)
    g.set_state(0.0, 1e3 * rng.standard_normal(g.n_free), 1e-5)
    g.rkc_advance_fixed(1e-5, 4, 2)
    xf, _ = g.get_state()
    print(f"order {order} n {n}: n_free {g.n_free}, kx modes spread {spread:.2e}, "
          f"|x_solve| {np.linalg.norm(xs):.3e}, |x_rkc| {np.linalg.norm(xf):.3e}")
    g.close()


if __name__ == "__main__":
    os.environ.setdefault("EQS_KX_BLOCK_TETS", "256")
    run(1, int(os.environ.get("SAN_N", "10")))
    if os.environ.get("SAN_P2", "1") == "1":
        run(2, 4)
