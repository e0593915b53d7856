"""Pin the CPU oracle to the reference's own known-answer tests.

Each test cites the reference test it ports. These run without a GPU; they
establish that the oracle the GPU path is compared against reproduces the
reference's documented behaviour.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla

from helpers import cube, matfree_setup
from oracle import pyoracle as po

EPS0 = 8.8541878128e-12


# ----------------------------------------------------------------- elements / materials
def test_reference_tet_p1_matrix():  # proj/tests/test_fem.cpp:202-212
    S = po.element_laplacian([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], 1, [1.0])
    assert S[0, 0] == pytest.approx(0.5, rel=1e-15)
    for j in (1, 2, 3):
        assert S[0, j] == pytest.approx(-1 / 6, rel=1e-15)
    assert S[1, 1] == pytest.approx(1 / 6, rel=1e-15)
    assert abs(S[1, 2]) <= 1e-15


SKEWED = np.array([[0.1, 0.0, -0.2], [1.3, 0.2, 0.1], [0.2, 1.1, 0.05], [-0.3, 0.4, 0.9]])  # test_fem.cpp:73-75
EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def _grad_lambda(p):
    J = (p[1:] - p[0]).T  # columns e1 e2 e3
    G = np.linalg.inv(J)  # rows grad lambda_1..3
    g = np.vstack([-G.sum(axis=0), G])
    vol = np.linalg.det(J) / 6.0
    return g, vol


def _moment_oracle(p, order, coeff):
    """proj/tests/test_fem.cpp:29-67 (exact barycentric moments)."""
    g, vol = _grad_lambda(p)
    n = 4 if order == 1 else 10
    const = np.zeros((n, 3))
    lin = np.zeros((n, 4, 3))
    if order == 1:
        const[:4] = g
    else:
        for i in range(4):
            const[i] = -g[i]
            lin[i, i] = 4 * g[i]
        for e, (a, b) in enumerate(EDGES):
            lin[4 + e, a] = 4 * g[b]
            lin[4 + e, b] = 4 * g[a]
    S = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            v = const[i] @ const[j] * vol
            for q in range(4):
                v += (const[i] @ lin[j, q] + const[j] @ lin[i, q]) * vol / 4
            for q in range(4):
                for r in range(4):
                    v += lin[i, q] @ lin[j, r] * (vol / 10 if q == r else vol / 20)
            S[i, j] = coeff * v
    return S


@pytest.mark.parametrize("order", [1, 2])
def test_element_matrix_matches_moment_oracle(order):  # test_fem.cpp:237-244
    S = po.element_laplacian(SKEWED, order, [0.7] * 4)
    ref = _moment_oracle(SKEWED, order, 0.7)
    assert np.abs(S - ref).max() <= 1e-13 * np.abs(ref).max()
    rows = np.abs(S.sum(axis=1)) / np.abs(S).sum(axis=1)  # test_fem.cpp:214-227 row sums vanish
    assert rows.max() <= 1e-14


def test_kappa_midpoint_and_limits():  # test_fem.cpp:95-102
    mv = {"eps_r": 12.0, "conductivity": {"kind": "microvaristor", "kappa_lo": 1e-10, "kappa_hi": 1e-4,
                                          "e_switch": 5e5, "width": 5e4}}
    assert po.kappa_of_e(mv, 5e5) == pytest.approx(math.sqrt(1e-10 * 1e-4), rel=1e-12)
    assert 1e-10 <= po.kappa_of_e(mv, 0.0) <= 1.001e-10
    const = {"eps_r": 2.0, "conductivity": {"kind": "constant", "kappa": 1e-3}}
    assert po.kappa_of_e(const, 0.0) == 1e-3 and po.kappa_of_e(const, 1e7) == 1e-3


# ----------------------------------------------------------------- RKC coefficients / integrators
def _oracle_amplification(s, z):  # test_integrators.cpp:14-39
    eps0 = 2.0 / 13.0
    w0 = 1.0 + eps0 / (s * s)
    t, tp, tpp = [1.0, w0], [0.0, 1.0], [0.0, 0.0]
    for j in range(2, s + 1):
        t.append(2 * w0 * t[j - 1] - t[j - 2])
        tp.append(2 * t[j - 1] + 2 * w0 * tp[j - 1] - tp[j - 2])
        tpp.append(4 * tp[j - 1] + 2 * w0 * tpp[j - 1] - tpp[j - 2])
    w1 = tp[s] / tpp[s]
    bs = tpp[s] / (tp[s] * tp[s])
    a_s = 1.0 - bs * t[s]
    arg = w0 + w1 * z
    um2, um1 = 1.0, arg
    for _ in range(2, s + 1):
        um2, um1 = um1, 2 * arg * um1 - um2
    return a_s + bs * um1


@pytest.mark.parametrize("s", [2, 5, 13])
def test_rkc_stage_recurrence_matches_amplification(s):  # test_integrators.cpp:117-129
    beta = 0.653 * (s * s - 1)
    for i in range(20):
        z = -beta * (i + 0.5) / 20
        sys_ = po.DiagonalSystem([1.0], [-z])
        x = sys_.advance("rkc", [1.0], 1.0, 1, s=s)
        assert abs(x[0] - _oracle_amplification(s, z)) <= 1e-12


@pytest.mark.parametrize("s", [2, 5, 13, 40])
def test_rkc_coefficients(s):  # test_integrators.cpp:131-140
    k = po.rkc_coefficients(s)
    assert k["c"][s] == pytest.approx(1.0, rel=1e-13)
    assert k["c"][1] == pytest.approx(k["c"][2] / 4, rel=1e-13)
    for z in (-0.1, -1.0, -0.5 * 0.653 * (s * s - 1)):
        assert po.rkc_amplification(s, z) == pytest.approx(_oracle_amplification(s, z), rel=1e-12)


@pytest.mark.parametrize("s", [2, 5, 10, 20])
def test_damped_stability(s):  # test_integrators.cpp:142-151
    beta = 0.653 * (s * s - 1)
    worst = max(abs(po.rkc_amplification(s, -beta * i / 10000)) for i in range(0, 10001, 7))
    assert worst <= 1.0 + 1e-12


def test_step_controller():  # test_integrators.cpp:53-71
    acc, dt = po.step_controller(1.0, 2.0, 2)
    assert acc and dt == pytest.approx(1.6)
    acc, dt = po.step_controller(0.0, 1.0, 2)
    assert acc and dt == pytest.approx(10.0)
    assert not po.step_controller(4.0, 1.0, 1)[0]
    assert po.step_controller(1e9, 1.0, 2)[1] == pytest.approx(0.1)
    prev = math.inf
    for err in (0.01, 0.1, 0.5, 1.0, 2.0, 10.0, 1e4):
        d = po.step_controller(err, 1.0, 2)[1]
        assert d <= prev
        prev = d


def test_convergence_orders():  # test_integrators.cpp:153-190
    k, a, b = 1.0, 3.0, 7.0

    def exact(t):
        p1 = (k * math.sin(a * t) - a * math.cos(a * t)) / (k * k + a * a)
        p2 = 0.5 * (k * math.cos(b * t) + b * math.sin(b * t)) / (k * k + b * b)
        return p1 + p2 - (-a / (k * k + a * a) + 0.5 * k / (k * k + b * b)) * math.exp(-k * t)

    for method, order, tol in (("euler", 1.0, 0.1), ("rkc", 2.0, 0.15), ("sdirk", 3.0, 0.2)):
        errs = []
        for dt in (1 / 40, 1 / 80, 1 / 160, 1 / 320):
            sys_ = po.DiagonalSystem([1.0], [k], c1=1.0, w1=a, c2=0.5, w2=b)
            x = sys_.advance(method, [0.0], dt, int(round(1 / dt)), s=5)
            errs.append(abs(x[0] - exact(1.0)))
        xs = -np.arange(4.0)
        slope = np.polyfit(xs, np.log2(errs), 1)[0]
        assert abs(slope - order) <= tol


def test_sdirk_linear_one_newton_per_stage():  # test_integrators.cpp:192-203
    sys_ = po.DiagonalSystem([1.0, 1.0, 1.0], [1.0, 5.0, 9.0])
    _, att = sys_.sdirk_step(po.random_vec(3, 2), 0.05)
    assert att["accepted"]
    assert att["newton_iterations"] == 3
    assert att["precond_setups"] == 1


def test_embedded_error_scales_like_dt3():  # test_integrators.cpp:205-234 (sdirk branch)
    est = []
    for dt in (0.02, 0.01, 0.005, 0.0025):
        sys_ = po.DiagonalSystem([1.0], [3.0], c2=1.0, w2=2.0)  # drive cos(2t)
        _, att = sys_.sdirk_step([1.0], dt, rtol=0.0, atol=1.0)
        assert att["accepted"]
        est.append(att["error"])
    slope = np.polyfit(-np.arange(4.0), np.log2(est), 1)[0]
    assert abs(slope - 3.0) <= 0.3


def test_spectral_radius_diag():  # test_integrators.cpp:73-85
    kk = np.arange(1.0, 11.0)
    rho = po.DiagonalSystem(np.ones(10), kk).spectral_radius()
    assert 10.0 <= rho <= 12.0
    rho2 = po.DiagonalSystem(np.ones(10), 2 * kk).spectral_radius()
    assert rho2 == pytest.approx(2 * rho, rel=1e-2)


def test_stage_choice_and_cap():  # test_integrators.cpp:236-265
    kk = np.array([10.0, 40.0, 90.0, 160.0, 250.0, 400.0])
    sys_ = po.DiagonalSystem(np.ones(6), kk)
    _, a = sys_.rkc_step(po.random_vec(6, 3), 0.5, atol=1e4)
    assert a["accepted"]
    z = a["dt"] * a["rho"]
    assert 0.653 * (a["stages"] ** 2 - 1) >= z
    if a["stages"] > 2:
        assert 0.653 * ((a["stages"] - 1) ** 2 - 1) < z
    sys2 = po.DiagonalSystem(np.ones(2), [1e8, 3e7])
    _, a = sys2.rkc_step(np.ones(2), 10.0, atol=1e9, max_stages=10)
    assert a["stages"] == 10 and a["dt"] <= 0.653 * 99 / a["rho"]


# ----------------------------------------------------------------- fused operator / FEM
@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("nonlinear", [False, True])
def test_fused_equals_assembled(order, nonlinear):  # test_matfree.cpp:40-58 (acceptance C1)
    o = po.Problem(matfree_setup(order, nonlinear))
    x = 2.0 * po.random_vec(o.n_dofs, 101 + order)
    v = po.random_vec(o.n_dofs, 202 + order)
    y, ref = o.kx_apply(x, v), o.assembled_k_apply(x, v)
    assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()


def _dense_k(o, x_full):
    n = o.n_dofs
    return np.column_stack([o.assembled_k_apply(x_full, np.eye(n)[i]) for i in range(n)])


def test_dc_residual_vanishes():  # test_matfree.cpp:106-127
    o = po.Problem(matfree_setup(1, False))
    _, fr, fx, fs = o.dofs()
    K = _dense_k(o, np.zeros(o.n_dofs))
    kii, kib = K[np.ix_(fr, fr)], K[np.ix_(fr, fx)]
    xb = np.array([1.0 if fs[d] == 1 else 0.0 for d in fx])  # set index 1 = "hv" (map order)
    b = -kib @ xb
    xi = np.linalg.solve(kii, b)
    xfull = np.zeros(o.n_dofs)
    xfull[fr], xfull[fx] = xi, xb
    r = o.kx_residual(xfull, np.zeros(o.n_free))
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(b)
    assert np.linalg.norm(o.kx_residual(np.zeros(o.n_dofs), np.zeros(o.n_free))) == 0.0


def test_colouring_is_conflict_free():  # test_matfree.cpp:129-144
    o = po.Problem(matfree_setup(2, False))
    ed = o.dofs()[0]
    col = o.colors()
    for c in range(col.max() + 1):
        d = ed[col == c].ravel()
        assert len(d) == len(np.unique(d))


def test_spectral_radius_brackets_generalized_eigenvalue():  # test_integrators.cpp:267-284
    cfg = {"mesh": {"box": {"nx": 3, "ny": 3, "nz": 3, "lx": 0.01, "ly": 0.01, "lz": 0.02, "z_planes": [0.01],
                            "regions": [1, 2]}},
           "materials": {"1": {"eps_r": 2.0, "conductivity": {"kind": "constant", "kappa": 1e-8}},
                         "2": {"eps_r": 5.0, "conductivity": {"kind": "constant", "kappa": 5e-9}}},
           "excitations": {"ground": {"kind": "constant", "value": 0.0},
                           "hv": {"kind": "sinusoid", "amplitude": 1e4, "frequency": 50.0}}}
    o = po.Problem(cfg)
    rho = o.spectral_radius(0.0, np.zeros(o.n_free))
    _, fr, _, _ = o.dofs()
    K = _dense_k(o, o.lift_full(0.0, np.zeros(o.n_free)))[np.ix_(fr, fr)]
    rp, ci, v = o.mass(0)
    M = np.zeros((o.n_free, o.n_free))
    for i in range(o.n_free):
        M[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    lam = sla.eigh(K, M, eigvals_only=True).max()
    assert lam <= rho <= 1.25 * lam


def test_energy_decays_undriven():  # test_integrators.cpp:286-329
    for nonlinear in (False, True):
        mats = {"1": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}},
                "2": {"eps_r": 12.0, "conductivity": ({"kind": "microvaristor", "kappa_lo": 1e-10, "kappa_hi": 3e-6,
                                                       "e_switch": 5e5, "width": 5e4} if nonlinear else
                                                      {"kind": "constant", "kappa": 3e-7})},
                "3": {"eps_r": 3.0, "conductivity": {"kind": "constant", "kappa": 1e-9}}}
        cfg = {"mesh": {"box": {"nx": 4, "ny": 4, "nz": 8, "lx": 0.006, "ly": 0.006, "lz": 0.012,
                                "z_planes": [0.004, 0.008], "regions": [1, 2, 3]}},
               "materials": mats,
               "excitations": {"ground": {"kind": "constant", "value": 0.0}, "hv": {"kind": "constant", "value": 0.0}}}
        o = po.Problem(cfg)
        x = 2e4 * po.random_vec(o.n_free, 31)
        rho = o.spectral_radius(0.0, x)
        dt = 0.9 * 0.653 * 24 / rho
        energy = x @ o.mass_apply(x)
        for _ in range(20):
            x = o.rkc_advance_fixed(0.0, x, dt, 5)
            e = x @ o.mass_apply(x)
            assert e <= energy * (1 + 1e-10)
            energy = e


def test_amg_pcg_converges_mesh_independently():  # acceptance C9 (acceptance_main.cpp:321-352)
    its = []
    for n in (6, 12, 24):
        o = po.Problem(cube(n))
        b = o.mass_apply(po.random_vec(o.n_free, 5))
        _, it, rel, conv = o.mass_solve(b, tol=1e-12)
        assert conv and rel <= 1e-12
        its.append(it)
    assert max(its) <= 1.5 * min(its)


def test_scenario_runs_and_counts():  # acceptance C5 + test_scenario.cpp:120-131 flavour
    from helpers import slab_reference
    cfg = slab_reference("smoke")
    r = po.run_scenario(cfg, x_cap=1000)
    assert r["precond_setups"] == 1
    assert abs(r["final_t"] - 5e-4) <= 1e-15
