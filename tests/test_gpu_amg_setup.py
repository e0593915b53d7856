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
