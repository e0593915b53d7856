"""The partitioned path across real OS processes (one GPU box, one GPU).

Two / three processes each own one node-ownership partition
(csrc/host_partition.cpp) and exchange halos and allreduce dot products
through the host-staged shared-memory backend (eqs_create_distributed_shm,
csrc/comm.cpp ShmComm). NCCL refuses several ranks on one GPU, so this is the
multi-process data plane that can run under `gpurun`; the NCCL backend runs
the same partition/halo/allreduce sequence with another transport.

Gates: bit-identical to the same partitions as virtual ranks in one process
(both sum the rank partials in rank order), and the single-partition
potentials to 1e-9 (the fp32 V-cycle vectors' partial coarse restrictions
are summed per rank, SURVEY.md §8e / tests/test_gpu_distributed.py).
"""
import os
import threading
import uuid

import numpy as np
import pytest

from helpers import cube
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

eb = pytest.importorskip("paper_1612_09447_b200")

CFG = cube(12, jitter=0.1, planes=(0.45, 0.55), estimator="spe")
STEPS = 3


def _rank_main(rank, world, name, x0, dt, out):
    g = eb.FemSystem.distributed_shm(CFG, 0, world, rank, name)
    owned = g.partition(0)["owned"]
    g.set_state(0.0, x0[owned], dt)
    rho = g.spectral_radius()
    g.rkc_advance_fixed(dt, 4, STEPS)
    out[rank] = (owned, g.get_state()[0], rho, g.stats()["pcg_iterations"])
    g.close()


def _virtual(world, x0, dt):
    ctxs = eb.FemSystem.virtual_group(CFG, world)
    res = [None] * world

    def work(r):
        c = ctxs[r]
        owned = c.partition(0)["owned"]
        c.set_state(0.0, x0[owned], dt)
        rho = c.spectral_radius()
        c.rkc_advance_fixed(dt, 4, STEPS)
        res[r] = (owned, c.get_state()[0], rho, c.stats()["pcg_iterations"])

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return res


@pytest.mark.parametrize("world,gate", [(2, None), (3, None), (3, "1")])
def test_processes_match_virtual_ranks_and_single_partition(world, gate, monkeypatch):
    """gate "1": EQS_SETUP_CONCURRENCY=1, the ranks' host setups run one at a
    time (capi.cpp SetupGate) before the collective device build."""
    import torch.multiprocessing as mp

    if gate:
        monkeypatch.setenv("EQS_SETUP_CONCURRENCY", gate)  # inherited by the spawned ranks

    single = eb.FemSystem(CFG)
    x0 = 2e4 * po.random_vec(single.n_free, 31)
    single.set_state(0.0, x0, 0.0)
    dt = 0.2 * 0.653 * 15 / single.spectral_radius()
    single.set_state(0.0, x0, dt)
    single.rkc_advance_fixed(dt, 4, STEPS)
    xs = single.get_state()[0]

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    name = f"/eqs_gpu_{uuid.uuid4().hex[:12]}"
    procs = [ctx.Process(target=_rank_main, args=(r, world, name, x0, dt, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    virt = _virtual(world, x0, dt)
    x = np.zeros(single.n_free)
    for r in range(world):
        owned, xr, rho, its = out[r]
        vo, vx, vrho, vits = virt[r]
        assert np.array_equal(owned, vo)
        assert np.array_equal(xr, vx), f"rank {r}: process and virtual-rank results differ"
        assert rho == vrho and its == vits
        x[owned] = xr
    assert np.linalg.norm(x - xs) <= 1e-9 * np.linalg.norm(xs)
