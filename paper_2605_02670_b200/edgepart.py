"""Edge-partitioned sampling helpers -- argument marshalling over the C ABI.

The partition itself (recursive coordinate bisection of the edge midpoints weighted by DOF
weight, or breadth-first runs of equal DOF weight) and everything a part needs from the whole
graph (local mesh, global DOF ids, whole-graph vertex masses and degrees, ownership, halo
lists) are computed inside the library (grf_partition_edges, grf_graph_create_part); this module
only moves ids around:

    G = Graph.from_metric_graph(g, h)
    edge_part, info = partition(G, n_parts, xy=g.coords)     # grf_partition_edges
    parts = make_parts(G, edge_part, n_parts)                # grf_graph_create_part per part
    us = sample_edgepart(parts, kappa, beta, k, ...)         # grf_sample_edgepart
    u = gather(parts, [x.cpu().numpy() for x in us], G.n_dofs)
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from .grf import Graph


def partition(G: Graph, n_parts: int, xy=None):
    """(edge_part [E] int32, info) from grf_partition_edges."""
    return G.partition(n_parts, xy=xy)


def make_parts(G: Graph, edge_part, n_parts: int, which: Optional[Sequence[int]] = None) -> List[Graph]:
    """Graph handles of the parts `which` (default: all) of the partition (grf_graph_create_part)."""
    ids = range(n_parts) if which is None else which
    return [Graph.part_of(G, edge_part, n_parts, q) for q in ids]


def gather(parts: List[Graph], fields, n_dofs: int) -> np.ndarray:
    """Assemble part-local fields [S, N_q] into the whole graph's DOF order [S, N]
    (grf_graph_part_dofs gives each local DOF's global index)."""
    S = fields[0].shape[0]
    out = np.full((S, n_dofs), np.nan)
    for p, f in zip(parts, fields):
        out[:, p.part_dofs()] = f
    return out
