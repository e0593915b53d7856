"""Device Galerkin products of the SA-AMG setup (SURVEY.md §8f rank 1,
csrc/k_spgemm.cu): the hierarchy a GPU context builds (smoothed prolongator
and R A P on the device) is bit-identical to the oracle's restatement of
proj/src/amg.cpp:90-143 and csr.cpp:133-166."""
import os

import numpy as np
import pytest

from helpers import cube, slab_reference
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

eb = pytest.importorskip("paper_1612_09447_b200")


def compare(g, o):
    n_levels = len(o.amg_levels())
    assert g.amg_levels() == o.amg_levels()
    for lvl in range(n_levels):
        if lvl + 1 < n_levels:
            assert np.array_equal(g.amg_aggregates(lvl), o.amg_aggregates(lvl))
        for which in ((0, 1, 2) if lvl + 1 < n_levels else (0,)):
            a, b = po.amg_level_csr(o, lvl, which), g.amg_level_csr(lvl, which)
            assert a[:2] == b[:2]
            for x, y in zip(a[2:], b[2:]):
                assert np.array_equal(x, y), (lvl, which)


@pytest.mark.parametrize("cfg", [cube(12, jitter=0.1), cube(4, jitter=0.1, order=2),
                                 slab_reference("slab_nonlinear_rkc_spe"), cube(20, jitter=0.15)],
                         ids=lambda c: c.get("name", "cfg"))
def test_device_hierarchy_bit_exact(cfg):
    compare(eb.FemSystem(cfg), po.Problem(cfg))


def test_device_hierarchy_bit_exact_many_batches(monkeypatch):
    monkeypatch.setenv("EQS_SPGEMM_BATCH", "5000")  # hundreds of row batches per product
    cfg = cube(14, jitter=0.1)
    compare(eb.FemSystem(cfg), po.Problem(cfg))


def compare_contexts(g, h):
    assert g.amg_levels() == h.amg_levels()
    n_levels = len(h.amg_levels())
    for lvl in range(n_levels):
        if lvl + 1 < n_levels:
            assert np.array_equal(g.amg_aggregates(lvl), h.amg_aggregates(lvl)), lvl
        for which in ((0, 1, 2) if lvl + 1 < n_levels else (0,)):
            a, b = h.amg_level_csr(lvl, which), g.amg_level_csr(lvl, which)
            assert a[:2] == b[:2]
            for x, y in zip(a[2:], b[2:]):
                assert np.array_equal(x, y), (lvl, which)


@pytest.mark.parametrize("cfg", [cube(40, jitter=0.1), cube(9, jitter=0.2, order=2), cube(31, jitter=0.0)],
                         ids=["cube40_jitter", "cube9_p2", "cube31_plain"])
def test_device_aggregation_matches_host_build(cfg):
    """Whole-level device setup (k_amgsetup.cu: strength graph, 3-pass greedy
    aggregation in rounds, P_tent, lambda_max, R = P^T) against the host-only
    build of the same hierarchy (amg.cpp:15-143 restated in host_setup.cpp)."""
    compare_contexts(eb.FemSystem(cfg), eb.FemSystem.partition_host(cfg, 1, 0))


@pytest.mark.parametrize("cfg", [cube(12, jitter=0.1), cube(5, jitter=0.1, order=2),
                                 slab_reference("slab_nonlinear_rkc_spe")], ids=["cube12", "cube5_p2", "slab"])
def test_device_colouring_bit_exact(cfg):
    """color_elements (matfree.cpp:11-38) in device waves (k_setup.cu) against
    the oracle's sequential greedy loop."""
    g, o = eb.FemSystem(cfg), po.Problem(cfg)
    assert np.array_equal(g.colors(), o.colors())
    assert g.colors().max() + 1 == o.n_colors


@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_device_partition_matches_host_plan(nranks):
    """partition_free_dofs with the device radix sort (virtual ranks on one
    GPU) against the host-only plan of the same ranks."""
    cfg = cube(14, jitter=0.1)
    group = eb.FemSystem.virtual_group(cfg, nranks)
    for r, g in enumerate(group):
        h = eb.FemSystem.partition_host(cfg, nranks, r)
        for level in (0, 1):
            a, b = g.partition(level), h.partition(level)
            assert np.array_equal(a["owner"], b["owner"]), (r, level)
            assert np.array_equal(a["owned"], b["owned"]) and np.array_equal(a["ghosts"], b["ghosts"])
