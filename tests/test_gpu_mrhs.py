"""Multiple-right-hand-side sequence through
eqs_mass_solve_sequence: the eval_rhs solve path (estimator.next, PCG,
feedback; proj/src/fem_system.cpp:80-90) on resident inputs."""
import numpy as np
import pytest

from helpers import cube

pytestmark = pytest.mark.gpu

eb = pytest.importorskip("paper_1612_09447_b200")


def smooth_sequence(g, k):
    nodes, _, _ = g.mesh()
    _, free, _ = g.dofs()
    xyz = nodes[free]
    phi = [np.sin(m * np.pi * xyz[:, 2]) * np.cos(np.pi * xyz[:, 0]) * np.cos(np.pi * xyz[:, 1]) for m in (1, 2, 3)]
    X = np.stack([sum(np.cos(2 * np.pi * m * j / 40) * phi[m - 1] for m in (1, 2, 3)) for j in range(k)])
    return X, np.stack([g.mass_apply(x) for x in X])


def test_sequence_solutions_and_estimators():
    g = eb.FemSystem(cube(14, jitter=0.1, planes=(0.45, 0.55)))
    X, B = smooth_sequence(g, 16)
    its = {}
    for mode in (0, 1, 2):
        g.set_option(12, mode)
        it, ms, Xs = g.mass_solve_sequence(B, want_x=True)
        assert ms > 0
        for k in range(len(X)):
            assert np.linalg.norm(Xs[k] - X[k]) <= 1e-9 * np.linalg.norm(X[k])
        its[mode] = it
    # the zero start is the plain solve
    x0, r0 = g.mass_solve(B[5])
    assert its[0][5] == r0.iterations
    # acceptance C6 (acceptance_main.cpp:250-269): SPE needs at most half the zero-start iterations
    assert its[2][8:].sum() <= 0.5 * its[0][8:].sum()
    assert its[1][1:].sum() < its[0][1:].sum()


def test_sequence_pod_estimators():
    """POD start vectors on the config-5 sequence (start_vector.cpp:111-131):
    the x*_k span three modes, so once the basis holds them the Galerkin start
    is nearly exact and PCG needs far fewer iterations than from zero."""
    g = eb.FemSystem(cube(14, jitter=0.1, planes=(0.45, 0.55)))
    X, B = smooth_sequence(g, 16)
    g.set_option(15, 4)  # pod_fixed: basis from the first 4 solutions
    g.set_option(18, 5)  # pod_rolling: append every solve above 5 iterations
    its = {}
    for mode in (0, 3, 4):
        g.set_option(12, mode)
        it, ms, Xs = g.mass_solve_sequence(B, want_x=True)
        for k in range(len(X)):
            assert np.linalg.norm(Xs[k] - X[k]) <= 1e-9 * np.linalg.norm(X[k])
        its[mode] = it
    assert (its[3][:4] == its[0][:4]).all()  # still collecting: zero starts
    assert its[3][5:].sum() <= 0.5 * its[0][5:].sum()
    assert its[4][5:].sum() <= 0.5 * its[0][5:].sum()


def test_sequence_rejects_bad_input():
    g = eb.FemSystem(cube(6))
    with pytest.raises(eb.EqsError):
        g.mass_solve_sequence(np.zeros((0, g.n_free)))
