"""Multi-rank host logic on CPU (gloo, world size 2): shard coverage and the node-shard reduce."""
import itertools
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_02670_b200.parallel import node_groups, shard


@pytest.mark.parametrize("world,S,L", [(1, 1, 55), (2, 1, 259), (8, 1, 259), (8, 256, 212), (8, 3, 10),
                                      (4, 16, 112), (3, 2, 7), (8, 64, 687)])
def test_shards_cover_every_unit_once(world, S, L):
    seen = np.zeros((S, L), dtype=int)
    roots = 0
    for r in range(world):
        sh = shard(world, r, S, L)
        if not sh.active:
            continue
        (s0, s1), (l0, l1) = sh.sample_range, sh.node_range
        seen[s0:s1, l0:l1:sh.node_stride] += 1
        roots += sh.is_root
    assert np.all(seen == 1)
    assert roots == shard(world, 0, S, L).n_sample_shards
    # round-robin node shards: their sizes differ by at most one node
    sizes = [len(range(*shard(world, r, S, L).node_range, shard(world, r, S, L).node_stride))
             for r in range(world) if shard(world, r, S, L).active]
    assert max(sizes) - min(sizes) <= 1
    for ranks in node_groups(world, S, L):
        assert shard(world, ranks[0], S, L).is_root


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, S, L, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_02670_b200.parallel import make_groups, reduce_partial
    groups = make_groups(world, S, L)
    sh = shard(world, rank, S, L)
    # stand-in for grf_sample(node_range=...): node l contributes (l+1) * (s+1) to sample s
    s0, s1 = sh.sample_range
    l0, l1 = sh.node_range
    part = torch.zeros(s1 - s0, 4, dtype=torch.float64)
    for s in range(s0, s1):
        part[s - s0] = sum((l + 1) * (s + 1) for l in range(l0, l1, sh.node_stride))
    res = reduce_partial(part, sh, groups)
    if res is not None:
        out[rank] = (s0, s1, res.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("S,L", [(1, 9), (2, 9), (3, 5)])
def test_gloo_node_shard_reduce(S, L):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), S, L, out), nprocs=world, join=True)
    full = {s: sum((l + 1) * (s + 1) for l in range(L)) for s in range(S)}
    got = {}
    for s0, s1, arr in out.values():
        for s in range(s0, s1):
            got[s] = arr[s - s0, 0]
    assert got == {s: float(v) for s, v in full.items()}


@pytest.mark.parametrize("world,S,L", [(1, 1, 55), (2, 1, 259), (8, 1, 259), (8, 256, 212), (8, 3, 10),
                                      (4, 16, 112), (3, 2, 7), (8, 64, 687), (5, 2, 3)])
def test_library_shard_matches_host_logic(world, S, L):
    """grf_dist_shard (the C ABI's copy of the sharding rule) agrees with parallel.shard."""
    from paper_2605_02670_b200.grf import dist_shard
    for r in range(world):
        sh = shard(world, r, S, L)
        srange, nrange, root, active, is_root, pl = dist_shard(world, r, S, L)
        assert active == sh.active and is_root == sh.is_root and pl == sh.n_node_shards == sh.node_stride
        if sh.active:
            assert srange == sh.sample_range and nrange == sh.node_range
            assert root == sh.group_index * sh.n_node_shards
