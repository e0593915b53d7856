"""SDIRK3(2) implicit baseline on the GPU backend:
sdirk_step / sdirk_advance_fixed (proj/src/integrators.cpp:237-343) with the
Newton matrix M + gamma dt K(z) assembled on the device every iteration
(fem_system.cpp:124-145), against the oracle's restatement."""
import numpy as np
import pytest

from helpers import cube, slab_reference
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

eb = pytest.importorskip("paper_1612_09447_b200")

LINEAR = {"1": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}},
          "2": {"eps_r": 12.0, "conductivity": {"kind": "constant", "kappa": 3e-6}},
          "3": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}}}


@pytest.mark.parametrize("order,dt", [(1, 5e-5), (2, 2e-4)])
def test_sdirk_fixed_steps_match_oracle(order, dt):
    """Nonlinear microvaristor cube, x0 = 200 random_vec(31): 3 fixed SDIRK
    steps (P2 at 2e-4 needs several Newton iterations per stage; larger steps
    make the reference's Picard-type Newton fail, for the oracle as well)."""
    cfg = cube(8 if order == 1 else 4, jitter=0.1, order=order)
    g, o = eb.FemSystem(cfg), po.Problem(cfg)
    n = g.n_free
    x0 = 200 * po.random_vec(n, 31)
    g.set_state(0.0, x0, dt)
    g.sdirk_advance_fixed(dt, 3)
    xg, info = g.get_state()
    xo = o.sdirk_advance_fixed(0.0, x0, dt, 3)
    rel = np.linalg.norm(xg - xo) / np.linalg.norm(xo)
    assert rel <= 1e-7, rel
    assert abs(info["t"] - 3 * dt) <= 1e-15
    sg, so = g.stats(), o.stats()
    assert sg["assemblies"] == so["assemblies"] >= 10  # one K assembly per Newton iteration, plus M


@pytest.mark.parametrize("order", [1, 2])
def test_shifted_solve_matches_oracle(order):
    """(M_II + gdt K_II(z)) delta = rhs through eqs_shifted_solve (the
    OdeSystem::shifted_solve a reference sdirk_step calls through the shim)."""
    cfg = cube(8 if order == 1 else 4, jitter=0.1, order=order)
    g, o = eb.FemSystem(cfg), po.Problem(cfg)
    n = g.n_free
    z = 3e4 * po.random_vec(n, 5)
    rhs = po.random_vec(n, 6)
    gdt = 0.435866521508459 * 2e-4
    dg = g.shifted_solve(1e-3, z, gdt, rhs)
    do = o.shifted_solve(1e-3, z, gdt, rhs)
    assert np.linalg.norm(dg - do) <= 1e-9 * np.linalg.norm(do)
    assert g.stats()["newton_linear_solves"] == 1


def test_sdirk_linear_one_newton_iteration_per_stage():  # test_integrators.cpp:192-203 on the FEM system
    cfg = cube(8, jitter=0.1, materials=LINEAR)
    g = eb.FemSystem(cfg)
    x0 = 200 * po.random_vec(g.n_free, 31)
    g.set_state(0.0, x0, 1e-5)
    s0 = g.stats()
    att = g.sdirk_step()
    s1 = g.stats()
    assert att.accepted
    assert att.newton_iterations == 3
    assert s1["precond_setups"] - s0["precond_setups"] == 1  # refreshed once per step
    assert s1["newton_linear_solves"] - s0["newton_linear_solves"] == 3


def test_sdirk_adaptive_step_matches_oracle_controller():
    """One adaptive step: accept decision and dt_next follow the order-3
    controller on the same error estimate (integrators.cpp:310-326)."""
    cfg = cube(4, jitter=0.1, order=2)
    g, o = eb.FemSystem(cfg), po.Problem(cfg)
    x0 = 200 * po.random_vec(g.n_free, 31)
    g.set_state(0.0, x0, 2e-4)
    att = g.sdirk_step(rtol=1e-2, atol=1e-8)
    xo = o.sdirk_advance_fixed(0.0, x0, 2e-4, 1)
    if att.accepted:
        xg, _ = g.get_state()
        assert np.linalg.norm(xg - xo) <= 1e-7 * np.linalg.norm(xo)
    acc, dt_next = po.step_controller(att.error, 2e-4, 3)
    assert bool(acc) == att.accepted
    assert abs(dt_next - att.dt_next) <= 1e-12 * dt_next


def test_sdirk_scenario_runs():  # proj/configs/slab_nonlinear_sdirk.json (acceptance C7/C8 table row)
    cfg = slab_reference("slab_nonlinear_sdirk")
    cfg["output"] = {"metrics_csv": "", "probe_csv": "", "solves_csv": ""}
    cfg["max_steps"] = 60  # additive key: bounded run (the full 0.02 s run takes ~100 s)
    r = eb.run_scenario(cfg)
    assert r["exit_code"] == 0, r.get("error")
    assert r["accepted"] + r["rejected"] == 60 and r["final_t"] > 0
    st = r["stats"]
    assert st["newton_linear_solves"] > 0 and st["newton_pcg_iterations"] > 0
    assert st["precond_setups"] >= r["accepted"]  # one refresh per attempted step (+1 for the mass AMG)
    assert np.isfinite(r["x"]).all()


@pytest.mark.parametrize("jitter", [0.1, 0.0])
def test_shifted_amg_matches_jacobi_with_fewer_iterations(jitter):
    """The shifted system (M_II + gdt K_II(z)) preconditioned with the SA-AMG
    rebuilt on the device (make_preconditioner -> AmgPreconditioner,
    fem_system.cpp:38-46, amg.cpp:90-143; option 26 = 1, the default) and with
    Jacobi (option 26 = 0): same solution to the solver tolerance, and the AMG
    needs far fewer PCG iterations, as the reference's per-step AMG would."""
    cfg = cube(20, jitter=jitter)
    z = 3e4 * po.random_vec(cube_free(cfg), 5)
    rhs = po.random_vec(cube_free(cfg), 6)
    gdt = 0.435866521508459 * 2e-4
    out = {}
    for amg in (1, 0):
        g = eb.FemSystem(cfg)
        g.set_option(26, amg)
        d = g.shifted_solve(1e-3, z, gdt, rhs)
        out[amg] = (d, g.stats()["newton_pcg_iterations"])
        g.close()
    (d_amg, it_amg), (d_jac, it_jac) = out[1], out[0]
    assert np.linalg.norm(d_amg - d_jac) <= 1e-9 * np.linalg.norm(d_jac)
    assert it_amg * 3 <= it_jac, (it_amg, it_jac)


def test_sdirk_steps_with_shifted_amg_match_jacobi():
    """Two fixed SDIRK steps: AMG- and Jacobi-preconditioned Newton solves give
    the same potentials (Newton tolerance 1e-8, PCG 1e-12) and Newton counts."""
    cfg = cube(12, jitter=0.1)
    x0 = 200 * po.random_vec(cube_free(cfg), 31)
    res = {}
    for amg in (1, 0):
        g = eb.FemSystem(cfg)
        g.set_option(26, amg)
        g.set_state(0.0, x0, 5e-5)
        g.sdirk_advance_fixed(5e-5, 2)
        res[amg] = (g.get_state()[0], g.stats()["assemblies"], g.stats()["precond_setups"])
        g.close()
    assert np.linalg.norm(res[1][0] - res[0][0]) <= 1e-8 * np.linalg.norm(res[0][0])
    assert res[1][1] == res[0][1] and res[1][2] == res[0][2]


def test_shifted_solve_graph_loop_matches_host_loop():
    """Shifted AMG solves through pcg_dev (graph-resident loop, fp32 V-cycle
    of the shifted hierarchy; option 27 = 1, default) against the
    host-driven fp64 V-cycle loop (option 27 = 0): same update to the solver
    tolerance, and the oracle's shifted solve."""
    cfg = cube(16, jitter=0.1)
    n = cube_free(cfg)
    z = 3e4 * po.random_vec(n, 5)
    rhs = po.random_vec(n, 6)
    gdt = 0.435866521508459 * 2e-4
    res = {}
    for graph in (1, 0):
        g = eb.FemSystem(cfg)
        g.set_option(27, graph)
        d = g.shifted_solve(1e-3, z, gdt, rhs)
        d2 = g.shifted_solve(1e-3, z, gdt, 2 * rhs, refresh_precond=False)  # captured graph reused
        res[graph] = (d, d2, g.stats()["newton_pcg_iterations"])
        g.close()
    do = po.Problem(cfg).shifted_solve(1e-3, z, gdt, rhs)
    for graph in (1, 0):
        assert np.linalg.norm(res[graph][0] - do) <= 1e-9 * np.linalg.norm(do)
        assert np.linalg.norm(res[graph][1] - 2 * do) <= 1e-9 * np.linalg.norm(2 * do)
    assert abs(res[1][2] - res[0][2]) <= 4


def cube_free(cfg):
    n = cfg["mesh"]["box"]["nx"]
    return (n + 1) ** 2 * (n - 1)  # z = 0 and z = 1 planes are Dirichlet
