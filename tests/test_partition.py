"""Node-ownership partition, host logic without a GPU.

The plan must be a deterministic function of the problem, bit-identical to an
independent CPU recomputation, and consistent across ranks (what rank r sends
to q is exactly q's ghosts owned by r, in q's order). The world-size-2 test
runs two gloo processes that exchange their halo lists.
"""
import copy
import os
import socket

import numpy as np
import pytest

from helpers import cube, slab_reference
from oracle import pyoracle as po

import paper_1612_09447_b200 as eb


def recompute_fine_owner(cfg, nranks):
    """numpy restatement of partition_free_dofs (csrc/host_partition.cpp)."""
    o = po.Problem(cfg)
    nodes, tets, _ = o.mesh()
    _, free, _, _ = o.dofs()
    lo, hi = nodes.min(axis=0), nodes.max(axis=0)
    ext = hi - lo
    axis = 2
    for k in (1, 0):
        if ext[k] > ext[axis]:
            axis = k
    coord = nodes[free, axis]  # P1: dofs are nodes
    order = np.argsort(coord, kind="stable")
    owner = np.empty(len(free), dtype=np.int64)
    owner[order] = (np.arange(len(free)) * nranks) // len(free)
    return owner


def coarse_owner(fine_owner, agg):
    first = {}
    for i, a in enumerate(agg):
        first.setdefault(int(a), i)
    return np.array([fine_owner[first[j]] for j in range(len(first))])


def with_replication(cfg, rows):
    cfg = copy.deepcopy(cfg)
    cfg.setdefault("solver", {})["amg_replicate_rows"] = rows
    return cfg


CFGS = [cube(10), with_replication(cube(10), 0), with_replication(cube(8, jitter=0.1, planes=(0.45, 0.55)), 200),
        slab_reference("slab_nonlinear_rkc_spe")]


def expected_rep_level(sizes, rows):
    """First coarse level with at most `rows` rows, else the coarsest (csrc/host_partition.cpp)."""
    if len(sizes) == 1:
        return 1
    return next((l for l in range(1, len(sizes)) if sizes[l] <= rows), len(sizes) - 1)


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: f'{c.get("name", "cfg")}-rep{c.get("solver", {}).get("amg_replicate_rows", "default")}')
@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_partition_bit_exact_and_consistent(cfg, nranks):
    plans = [eb.FemSystem.partition_host(cfg, nranks, r) for r in range(nranks)]
    ref = recompute_fine_owner(cfg, nranks)
    n_levels = plans[0].partition_levels
    sizes = [plans[0].partition(l)["n_global"] for l in range(n_levels)]
    rep = expected_rep_level(sizes, cfg.get("solver", {}).get("amg_replicate_rows", 32768))
    for lvl in range(n_levels):
        parts = [p.partition(lvl) for p in plans]
        owner = parts[0]["owner"]
        for part in parts[1:]:
            assert np.array_equal(part["owner"], owner)  # every rank computes the same plan
        if lvl == 0:
            assert np.array_equal(owner, ref)
        else:
            agg = plans[0].amg_aggregates(lvl - 1)
            assert np.array_equal(owner, coarse_owner(plans[0].partition(lvl - 1)["owner"], agg))
        if lvl >= rep:  # replicated: whole level on every rank, no halo
            for pr in parts:
                assert pr["replicated"]
                assert np.array_equal(pr["owned"], np.arange(pr["n_global"]))
                assert len(pr["ghosts"]) == 0 and not pr["sends"]
            continue
        assert not any(pr["replicated"] for pr in parts)
        owned = np.concatenate([p["owned"] for p in parts])
        assert np.array_equal(np.sort(owned), np.arange(parts[0]["n_global"]))  # a partition
        for r, pr in enumerate(parts):
            assert np.all(owner[pr["owned"]] == r)
            assert np.all(owner[pr["ghosts"]] != r)
            for q, pq in enumerate(parts):
                if q == r:
                    continue
                expect = pq["ghosts"][owner[pq["ghosts"]] == r]  # q's ghosts owned by r, q's order
                got = pr["sends"].get(q, np.zeros(0, dtype=np.int32))
                assert np.array_equal(got, expect)
    # owner computes: every tet with an owned free dof is local to that owner
    tets_total = sum(p.partition(0)["n_local_tets"] for p in plans)
    assert tets_total >= plans[0].n_tets


def _gloo_worker(rank, world, port, cfg, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = eb.FemSystem.partition_host(cfg, world, rank)
        mine = plan.partition(0)
        payload = {"ghosts": mine["ghosts"].tolist(), "owner": mine["owner"].tolist(),
                   "sends": {q: v.tolist() for q, v in mine["sends"].items()}}
        allp = [None] * world
        dist.all_gather_object(allp, payload)
        ok = allp[0]["owner"] == payload["owner"]
        for q in range(world):
            if q == rank:
                continue
            expect = [g for g in allp[q]["ghosts"] if payload["owner"][g] == rank]
            ok = ok and payload["sends"].get(q, []) == expect
        out[rank] = bool(ok)
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo_halo_lists_agree():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gloo_worker, args=(2, port, cube(8, jitter=0.1), out), nprocs=2, join=True)
    assert out[0] and out[1]


def _shm_worker(rank, world, port, name, cfg, out):
    """One OS process per rank: the partition plan's numeric halo exchange and
    the dot-product allreduce through the shared-memory transport of
    eqs_create_distributed_shm (host buffers, no GPU), checked against the
    global vector and against a gloo allreduce of the same partials."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = eb.eqs.ShmComm(name, world, rank)
    try:
        plan = eb.FemSystem.partition_host(cfg, world, rank).partition(0)
        owner, owned, ghosts = plan["owner"], plan["owned"], plan["ghosts"]
        g = np.sin(0.37 * np.arange(owner.size)) * 1e3  # the global vector
        sends = {q: g[ids] for q, ids in plan["sends"].items()}
        recv_counts = {q: int(np.sum(owner[ghosts] == q)) for q in range(world) if q != rank}
        got = comm.exchange(sends, recv_counts)
        ok = True
        for q, vals in got.items():
            ok = ok and np.array_equal(vals, g[ghosts[owner[ghosts] == q]])
        # allreduce: rank-order sum of the owned partial dots (deterministic)
        part = np.array([float(np.dot(g[owned], g[owned])), float(owned.size)])
        tot = comm.allreduce(part)
        allp = [None] * world
        dist.all_gather_object(allp, part.tolist())
        expect = np.zeros(2)
        for p in allp:
            expect += np.array(p)
        ok = ok and np.array_equal(tot, expect) and tot[1] == owner.size
        t = torch.tensor(part)
        dist.all_reduce(t)  # gloo: the same sum up to summation order
        ok = ok and abs(float(t[0]) - tot[0]) <= 1e-12 * tot[0] and np.isclose(tot[0], np.dot(g, g), rtol=1e-12)
        comm.barrier()
        out[rank] = bool(ok)
    finally:
        comm.close()
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shm_transport_halo_and_allreduce_multiprocess(world):
    import uuid

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    name = f"/eqs_test_{uuid.uuid4().hex[:12]}"
    mp.spawn(_shm_worker, args=(world, port, name, cube(8, jitter=0.1), out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))
