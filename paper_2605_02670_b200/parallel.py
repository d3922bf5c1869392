"""Multi-GPU sharding of the (quadrature node) x (sample) units.

Every (l, s) pair is an independent vertex system; a sample's field is the sum over l of the
node solutions (PAPER.md P313-324).  One process per GPU:

* samples first: P_s = min(world, S) contiguous sample ranges -- no data-path collective;
* then nodes: the P_l = world // P_s ranks sharing a sample range split the quadrature nodes
  round-robin (shard li takes nodes li, li + P_l, ...: grf_options.node_begin / node_stride --
  the PCG cost varies with l, P162-165, and strided shards balance it), and their partial sums
  are reduced to the range's root with one NCCL reduce over NVLink (torch.distributed group).

The library call for the local part is ``Graph.sample(..., node_range=...)``; the reduce is
``torch.distributed.reduce`` on a per-sample-range sub-group (NCCL on GPUs, gloo in the CPU
tests of this module).
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Tuple


@dataclasses.dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    n_sample_shards: int
    n_node_shards: int
    sample_range: Tuple[int, int]   # [s0, s1) of the call's samples
    node_range: Tuple[int, int]     # nodes l0, l0 + node_stride, ... < l1 of 0..L-1
    node_stride: int
    group_index: int                # which sample range (ranks with equal index share it)
    is_root: bool                   # receives the reduced sum for its sample range
    active: bool                    # False for ranks left over when world > P_s * P_l


def _split(n: int, parts: int, i: int) -> Tuple[int, int]:
    base, extra = divmod(n, parts)
    lo = i * base + min(i, extra)
    return lo, lo + base + (1 if i < extra else 0)


def shard(world: int, rank: int, n_samples: int, n_nodes: int) -> Shard:
    if not (0 <= rank < world) or n_samples < 1 or n_nodes < 1:
        raise ValueError("bad shard arguments")
    ps = min(world, n_samples)
    pl = max(1, min(world // ps, n_nodes))
    active = rank < ps * pl
    gi, li = (rank // pl, rank % pl) if active else (0, 0)
    return Shard(rank, world, ps, pl, _split(n_samples, ps, gi) if active else (0, 0),
                 (li, n_nodes) if active else (0, 0), pl, gi, active and li == 0, active)


def node_groups(world: int, n_samples: int, n_nodes: int):
    """Rank lists that share a sample range (one reduce group each)."""
    s0 = shard(world, 0, n_samples, n_nodes)
    pl = s0.n_node_shards
    return [list(range(g * pl, (g + 1) * pl)) for g in range(s0.n_sample_shards)]


def make_groups(world: int, n_samples: int, n_nodes: int):
    """torch.distributed sub-groups for the node-shard reductions (call on every rank, same order)."""
    import torch.distributed as dist
    return [dist.new_group(ranks) if len(ranks) > 1 else None
            for ranks in node_groups(world, n_samples, n_nodes)]


def reduce_partial(partial, sh: Shard, groups) -> Optional[object]:
    """Sum the node-shard partial sums of a sample range onto its root rank (NCCL reduce)."""
    import torch.distributed as dist
    if not sh.active:
        return None
    g = groups[sh.group_index]
    if g is None:
        return partial
    root = sh.group_index * sh.n_node_shards
    dist.reduce(partial, dst=root, op=dist.ReduceOp.SUM, group=g)
    return partial if sh.is_root else None


def sample_dist(graph, kappa, beta, k, seed, n_samples, groups=None, **opts):
    """This rank's share of a grf_sample call: returns (shard, u or None).

    u is the full field for the rank's sample range on the range's root rank, else None.
    """
    import torch.distributed as dist

    from .grf import plan_info
    world, rank = dist.get_world_size(), dist.get_rank()
    km, kp, _, _ = plan_info(beta, k)
    L = km + kp + 1
    sh = shard(world, rank, n_samples, L)
    if groups is None:
        groups = make_groups(world, n_samples, L)
    if not sh.active:
        return sh, None
    s0, s1 = sh.sample_range
    u = graph.sample(kappa, beta, k, seed=seed + s0, n_samples=s1 - s0, node_range=sh.node_range,
                     node_stride=sh.node_stride, **opts)
    return sh, reduce_partial(u, sh, groups)
