"""POD start-vector estimators: pod_build and the
pod_fixed / pod_rolling modes of StartVectorEstimator
(proj/src/start_vector.cpp:64-71,111-150,165-187).

CPU tests pin the oracle against the reference's own estimator tests
(proj/tests/test_estimators.cpp:135-259). GPU tests drive the device
estimator through the C-ABI (eqs_estimator_next / _feedback / _stats) with
the same inputs and compare the start vectors with the oracle's."""
import numpy as np
import pytest

from oracle import pyoracle as po


def small_mass_config(mode="zero", **est):
    """test_estimators.cpp:21-27: 3x3x3 unit box, one material with eps_r = 1."""
    e = {"mode": mode}
    e.update(est)
    return {
        "name": "small_mass",
        "mesh": {"box": {"nx": 3, "ny": 3, "nz": 3, "lx": 1.0, "ly": 1.0, "lz": 1.0}},
        "order": 1,
        "materials": {"1": {"eps_r": 1.0, "conductivity": {"kind": "constant", "kappa": 0.0}}},
        "excitations": {"ground": {"kind": "constant", "value": 0.0}, "hv": {"kind": "constant", "value": 1.0}},
        "solver": {"preconditioner": "amg", "rel_tol": 1e-12, "max_iter": 500},
        "estimator": e,
    }


def test_pod_identical_snapshots_rank_one():  # test_estimators.cpp:135-143
    s = po.random_vec(30, 1)
    U, sig = po.pod_build(np.stack([s] * 4), 3)
    assert U.shape[0] == 1
    assert abs(abs(U[0] @ (s / np.linalg.norm(s))) - 1.0) <= 1e-12


def test_pod_reconstruction_bound():  # test_estimators.cpp:145-160
    S = np.stack([po.random_vec(40, 60 + c) for c in range(8)])  # rows = snapshots
    rank = 3
    U, sig = po.pod_build(S, rank)
    assert U.shape[0] == rank
    assert np.abs(U @ U.T - np.eye(rank)).max() <= 1e-10
    full = np.linalg.svd(S.T, compute_uv=False)  # full-SVD oracle
    assert np.allclose(sig, full, rtol=1e-12, atol=1e-14 * full[0])
    discarded = float((full[rank:] ** 2).sum())
    A = S.T
    err = float(((A - U.T @ (U @ A)) ** 2).sum())
    assert err <= discarded + 1e-10 * float((A ** 2).sum())
    # same span as LAPACK's leading left singular vectors
    Ul = np.linalg.svd(A, full_matrices=False)[0][:, :rank]
    assert np.linalg.norm(Ul - U.T @ (U @ Ul)) <= 1e-10


def test_pod_truncates_at_numerical_rank():  # start_vector.cpp:64-71 (sigma > 1e-12 sigma_0)
    a, b = po.random_vec(50, 3), po.random_vec(50, 4)
    S = np.stack([a, b, a + b, 2 * a - b, a])
    U, sig = po.pod_build(S, 10)
    assert U.shape[0] == 2
    assert sig[2] <= 1e-12 * sig[0]


@pytest.mark.parametrize("mode", ["zero", "previous", "spe", "pod_fixed", "pod_rolling"])
def test_first_call_starts_at_zero(mode):  # test_estimators.cpp:162-172
    o = po.Problem(small_mass_config(mode))
    x0, _ = o.estimator_next(po.random_vec(o.n_free, 2))
    assert np.linalg.norm(x0) == 0.0


def test_pod_rolling_threshold():  # test_estimators.cpp:194-218
    o = po.Problem(small_mass_config("pod_rolling", threshold=5.0, capacity=4))
    n = o.n_free
    b = po.random_vec(n, 8)
    o.estimator_feedback(po.random_vec(n, 400), 3)
    assert o.estimator_stats()["appends"] == 0
    _, r = o.estimator_next(b)
    assert o.estimator_stats()["svd_count"] == 0 and r == 0
    o.estimator_feedback(po.random_vec(n, 401), 6)
    assert o.estimator_stats()["appends"] == 1
    _, r = o.estimator_next(b)
    assert o.estimator_stats()["svd_count"] == 1 and r == 1
    o.estimator_next(b)
    assert o.estimator_stats()["svd_count"] == 1


def test_pod_rolling_svd_count():  # test_estimators.cpp:220-240
    o = po.Problem(small_mass_config("pod_rolling", threshold=5.0, capacity=3, rank=2))
    n = o.n_free
    b = po.random_vec(n, 8)
    counts = [9, 2, 8, 7, 1, 3, 11, 6]
    for i, c in enumerate(counts):
        o.estimator_next(b)
        o.estimator_feedback(po.random_vec(n, 500 + i), c)
    o.estimator_next(b)
    above = sum(c > 5 for c in counts)
    st = o.estimator_stats()
    assert st["appends"] == above and st["svd_count"] == above


def test_pod_fixed_freezes_basis():  # test_estimators.cpp:242-259
    o = po.Problem(small_mass_config("pod_fixed", snapshots=4, rank=2))
    n = o.n_free
    b = po.random_vec(n, 9)
    for i in range(4):
        x0, _ = o.estimator_next(b)
        assert np.linalg.norm(x0) == 0.0
        o.estimator_feedback(po.random_vec(n, 600 + i), 5)
    _, r = o.estimator_next(b)
    assert o.estimator_stats()["svd_count"] == 1 and r == 2
    for i in range(3):
        o.estimator_feedback(po.random_vec(n, 700 + i), 5)
        o.estimator_next(b)
    assert o.estimator_stats()["svd_count"] == 1


def test_pod_start_is_galerkin_projection():  # start_vector.cpp:127-130: x0 = V (V'MV)^-1 V'b
    o = po.Problem(small_mass_config("pod_fixed", snapshots=5, rank=3))
    n = o.n_free
    snaps = [po.random_vec(n, 800 + i) for i in range(5)]
    for s in snaps:
        o.estimator_feedback(s, 5)
    b = po.random_vec(n, 9)
    x0, r = o.estimator_next(b)
    V, _ = po.pod_build(np.stack(snaps), 3)
    rp, ci, v = o.mass(0)
    M = np.zeros((n, n))
    for i in range(n):
        M[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    ref = V.T @ np.linalg.solve(V @ M @ V.T, V @ b)
    assert r == 3
    assert np.linalg.norm(x0 - ref) <= 1e-12 * np.linalg.norm(ref)


def test_pod_configs_parse():  # scenario.cpp:56-71
    for mode in ("pod_fixed", "pod_rolling"):
        po.Problem(small_mass_config(mode, snapshots=10, rank=4, capacity=6, threshold=3))
    with pytest.raises(po.OracleError):
        po.Problem(small_mass_config("pod_fixed", rank=0))


# ------------------------------------------------------------------ GPU parity
eb = None


def _eb():
    global eb
    if eb is None:
        eb = pytest.importorskip("paper_1612_09447_b200")
    return eb


def _pair(cfg):
    g = _eb().FemSystem(cfg)
    o = po.Problem(cfg)
    assert g.n_free == o.n_free
    return g, o


@pytest.mark.gpu
@pytest.mark.parametrize("mode,params", [
    ("pod_fixed", {"snapshots": 6, "rank": 3}),
    ("pod_rolling", {"threshold": 5.0, "capacity": 4, "rank": 3}),
    ("pod_rolling", {"capacity": 5, "rank": 10}),  # median threshold, rank above the snapshot count
])
def test_gpu_pod_sequence_matches_oracle(mode, params):
    """Same feedback/next sequence on the device estimator and the oracle: start
    vectors agree to 1e-10, ranks and svd/append counters exactly."""
    from helpers import cube
    cfg = cube(8, jitter=0.1, estimator=mode)
    cfg["estimator"] = dict({"mode": mode}, **params)
    g, o = _pair(cfg)
    n = g.n_free
    counts = [9, 2, 8, 7, 1, 3, 11, 6, 12, 4, 9, 8]
    for i, c in enumerate(counts):
        b = po.random_vec(n, 900 + i)
        xg, rg = g.estimator_next(b)
        xo, ro = o.estimator_next(b)
        assert rg == ro, (i, rg, ro)
        scale = max(np.linalg.norm(xo), 1e-300)
        assert np.linalg.norm(xg - xo) <= 1e-10 * scale, (i, np.linalg.norm(xg - xo) / scale)
        # smooth, correlated snapshots (the POD use case) plus noise
        s = np.cos(0.3 * i) * po.random_vec(n, 1) + np.sin(0.3 * i) * po.random_vec(n, 2) \
            + 1e-3 * po.random_vec(n, 1000 + i)
        g.estimator_feedback(s, c)
        o.estimator_feedback(s, c)
    assert g.estimator_stats() == o.estimator_stats()


@pytest.mark.gpu
def test_gpu_pod_rank_deficient_snapshots():
    from helpers import cube
    cfg = cube(6, estimator="pod_fixed")
    cfg["estimator"] = {"mode": "pod_fixed", "snapshots": 5, "rank": 4}
    g, o = _pair(cfg)
    n = g.n_free
    a, c = po.random_vec(n, 3), po.random_vec(n, 4)
    for s in (a, c, a + c, 2 * a - c, a):
        g.estimator_feedback(s, 5)
        o.estimator_feedback(s, 5)
    b = po.random_vec(n, 5)
    xg, rg = g.estimator_next(b)
    xo, ro = o.estimator_next(b)
    assert rg == ro == 2
    assert np.linalg.norm(xg - xo) <= 1e-10 * np.linalg.norm(xo)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["pod_fixed", "pod_rolling"])
def test_gpu_pod_rkc_potentials_match_oracle(mode):
    """10 fixed RKC steps (config-1 family, nonlinear) with a POD estimator:
    the start vector only changes the PCG starting point, so the potentials
    match the oracle's to the solver tolerance."""
    from helpers import cube
    cfg = cube(10, estimator=mode)
    cfg["estimator"] = {"mode": mode, "snapshots": 8, "rank": 4, "capacity": 6}
    g, o = _pair(cfg)
    n = g.n_free
    x0 = 2e4 * po.random_vec(n, 31)
    rho = o.spectral_radius(0.0, x0)
    dt, s = 0.2 * 0.653 * 15 / rho, 4
    g.set_state(0.0, x0, dt)
    g.rkc_advance_fixed(dt, s, 5)
    xg, _ = g.get_state()
    xo = o.rkc_advance_fixed(0.0, x0, dt, s, 5)
    assert np.linalg.norm(xg - xo) <= 1e-9 * np.linalg.norm(xo)
    sg, so = g.stats(), o.stats()
    assert sg["m_solves"] == so["m_solves"] == 20
    assert sg["svd_count"] == so["svd_count"] if mode == "pod_fixed" else sg["svd_count"] >= 1
