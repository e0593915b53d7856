import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, bench
import paper_1612_09447_b200 as eb
from oracle import pyoracle as po
n = int(sys.argv[1])
cfg = bench.scenario(n, 0.0, [1/3, 2/3])
g = eb.FemSystem(cfg, device=0)
z = 2e4 * po.random_vec(g.n_free, 31); rhs = po.random_vec(g.n_free, 6)
for k in range(3):
    t = time.perf_counter(); d = g.shifted_solve(1e-3, z, 0.4358 * 2e-4, rhs, refresh_precond=True); t1 = time.perf_counter()
    d = g.shifted_solve(1e-3, z, 0.4358 * 2e-4, rhs, refresh_precond=False); t2 = time.perf_counter()
    print(f"refresh+solve {t1-t:.3f} s, solve only {t2-t1:.3f} s", flush=True)
print(g.stats())
