import sys, time, os
sys.path.insert(0, '/root/repo')
import bench
for n in [int(a) for a in sys.argv[1:]]:
    t0 = time.perf_counter()
    cfg = bench.scenario(n, 0.1, [0.45, 0.55])
    arm = bench.CpuArm(cfg, os.cpu_count())
    x0, dt, rho = bench.sample_x0_dt(arm)
    arm.set_state(0.0, x0, dt)
    t1 = time.perf_counter()
    arm.advance(dt, 4, 1)
    t2 = time.perf_counter()
    arm.advance(dt, 4, 1)
    t3 = time.perf_counter()
    print(f"n {n} free {arm.n_free} setup {t1-t0:.1f} s step {t2-t1:.2f} / {t3-t2:.2f} s -> {arm.n_free*4/(t3-t2):.3e} DOF-stage/s iters {arm.iters_per_solve():.1f}", flush=True)
