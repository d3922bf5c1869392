"""TEST HELPER (CPU, numpy): a reference edge partition for the host-logic tests of the
edge-partitioned NN-PCG (tests/test_edgepart.py, gloo ranks, no GPU).  The product computes
the same things inside the library (grf_partition_edges / grf_graph_create_part, include/grf.h);
tests/test_edgepart_gpu.py checks the library's partition against the invariants below.

Which edges each part holds, the part-local numbering, and what a part needs from the whole
graph:

* edges are ordered by a breadth-first traversal of the vertex graph from vertex 0 (an edge
  takes the visit rank of its earlier-visited end) and cut into contiguous runs of equal
  DOF weight n_e = max(1, ceil(l_e / h)) (P123) -- parts are connected-ish and balanced;
* a part is the subgraph of its edges and every vertex they touch (local ids ascending in
  global id, local edges in ascending global id); vertices touched by several parts are
  interface vertices, numbered in ascending global id; each vertex is owned by the lowest
  part that touches it;
* the whole graph's lumped vertex masses (P137-145, summed in ascending edge id, edge_u
  end before edge_v end -- the library's order, so the noise is bit-identical) and degrees
  d_v (incident edge ends, P261), and the global DOF offsets of the edges (DOF order S97).
"""
from __future__ import annotations

import dataclasses
from collections import deque
from typing import List

import numpy as np


@dataclasses.dataclass
class Part:
    index: int
    edges: np.ndarray          # global edge ids held by this part (ascending)
    vertices: np.ndarray       # global vertex ids of the local vertices (ascending)
    edge_u: np.ndarray         # local endpoint ids
    edge_v: np.ndarray
    length: np.ndarray
    edge_goff: np.ndarray      # global DOF index of each local edge's first interior node
    vertex_mass: np.ndarray    # whole-graph lumped mass of each local vertex
    vertex_degree: np.ndarray  # whole-graph incident edge ends (int32)
    vertex_owned: np.ndarray   # uint8
    vertex_iface: np.ndarray   # interface id or -1 (int64)
    n_interface: int
    global_n_interior: int

    @property
    def n_vertices(self) -> int:
        return int(len(self.vertices))

    @property
    def n_edges(self) -> int:
        return int(len(self.edges))

    def dof_gid(self, h: float) -> np.ndarray:
        """Global DOF index of every local DOF (local interiors in local edge order, then vertices)."""
        n_el = element_counts(self.length, h)
        parts = [self.edge_goff[e] + np.arange(n_el[e] - 1) for e in range(self.n_edges)]
        parts.append(self.global_n_interior + self.vertices)
        return np.concatenate([np.asarray(p, dtype=np.int64) for p in parts])


def element_counts(length: np.ndarray, h: float) -> np.ndarray:
    """n_e = max(1, ceil(l_e / h)) in fp64 (P123)."""
    return np.maximum(1, np.ceil(np.asarray(length, dtype=np.float64) / h)).astype(np.int64)


def whole_graph_vertex_data(graph, h):
    """(lumped vertex masses, degrees, N_I, interior offsets) of the whole graph."""
    n_el = element_counts(graph.length, h)
    he = graph.length / n_el
    E = graph.n_edges
    idx = np.empty(2 * E, dtype=np.int64)
    idx[0::2] = graph.edge_u
    idx[1::2] = graph.edge_v
    val = np.repeat(he / 2.0, 2)
    mass = np.zeros(graph.n_vertices)
    np.add.at(mass, idx, val)  # sequential in index order: ascending edge, u end then v end
    deg = np.bincount(idx, minlength=graph.n_vertices).astype(np.int32)
    m = n_el - 1
    goff = np.concatenate([[0], np.cumsum(m)[:-1]]).astype(np.int64)
    return mass, deg, int(m.sum()), goff


def bfs_edge_order(graph) -> np.ndarray:
    """Edges ordered by the BFS visit rank of their earlier-visited end (ties: edge id)."""
    V = graph.n_vertices
    adj = [[] for _ in range(V)]
    for u, v in zip(graph.edge_u.tolist(), graph.edge_v.tolist()):
        adj[u].append(v)
        adj[v].append(u)
    rank = np.full(V, -1, dtype=np.int64)
    nxt = 0
    for root in range(V):
        if rank[root] >= 0:
            continue
        rank[root] = nxt
        nxt += 1
        dq = deque([root])
        while dq:
            a = dq.popleft()
            for b in adj[a]:
                if rank[b] < 0:
                    rank[b] = nxt
                    nxt += 1
                    dq.append(b)
    key = np.minimum(rank[graph.edge_u], rank[graph.edge_v])
    return np.lexsort((np.arange(graph.n_edges), key))


def partition(graph, h: float, n_parts: int) -> List[Part]:
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    E = graph.n_edges
    n_el = element_counts(graph.length, h)
    order = bfs_edge_order(graph)
    w = n_el[order].astype(np.float64)
    cum = np.cumsum(w)
    cuts = np.searchsorted(cum, cum[-1] * np.arange(1, n_parts) / n_parts, side="left")
    bounds = np.concatenate([[0], np.minimum(cuts + 1, E), [E]])
    part_of_edge = np.empty(E, dtype=np.int64)
    for q in range(n_parts):
        part_of_edge[order[bounds[q]:bounds[q + 1]]] = q
    mass, deg, NI, goff = whole_graph_vertex_data(graph, h)
    # parts touching each vertex
    touch = [set() for _ in range(graph.n_vertices)]
    for e in range(E):
        q = int(part_of_edge[e])
        touch[int(graph.edge_u[e])].add(q)
        touch[int(graph.edge_v[e])].add(q)
    iface_vertices = [v for v in range(graph.n_vertices) if len(touch[v]) > 1]
    iface_id = np.full(graph.n_vertices, -1, dtype=np.int64)
    iface_id[iface_vertices] = np.arange(len(iface_vertices))
    owner = np.array([min(t) if t else -1 for t in touch], dtype=np.int64)
    parts = []
    for q in range(n_parts):
        edges = np.flatnonzero(part_of_edge == q)
        verts = np.unique(np.concatenate([graph.edge_u[edges], graph.edge_v[edges]]))
        loc = {int(v): i for i, v in enumerate(verts)}
        eu = np.array([loc[int(v)] for v in graph.edge_u[edges]], dtype=np.int64)
        ev = np.array([loc[int(v)] for v in graph.edge_v[edges]], dtype=np.int64)
        parts.append(Part(q, edges, verts.astype(np.int64), eu, ev, graph.length[edges].astype(np.float64),
                          goff[edges], mass[verts], deg[verts].astype(np.int32),
                          (owner[verts] == q).astype(np.uint8), iface_id[verts], len(iface_vertices), NI))
    return parts


def gather(parts: List[Part], fields, h: float, n_dofs: int) -> np.ndarray:
    """Assemble part-local fields [S, N_q] into the whole graph's DOF order [S, N]."""
    S = fields[0].shape[0]
    out = np.full((S, n_dofs), np.nan)
    for p, f in zip(parts, fields):
        out[:, p.dof_gid(h)] = f
    return out
