"""Oracle Phase 1: mesh and canonical DOF order (PAPER.md P122-123, §3.1).

n_e = ceil(l_e / h) (IEEE ceil of the fp64 quotient),
h_e = l_e / n_e, N_e = n_e + 1, interior count m_e = n_e - 1,
N = |V| + sum_e (N_e - 2) (P123).

DOF order (SPEC S97, P150 "W = [W_I,1 ... W_I,|E|  W_Gamma]"): interior nodes of
e_0 by ascending local x, then e_1, ..., then vertices 0..V-1.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class Mesh:
    n_vertices: int
    edge_u: np.ndarray
    edge_v: np.ndarray
    length: np.ndarray
    h: float
    n_el: np.ndarray      # n_e, elements per edge
    h_e: np.ndarray       # local mesh size
    m_int: np.ndarray     # n_e - 1 interior nodes
    offset: np.ndarray    # global index of first interior node of edge e
    n_interior: int
    n_dofs: int

    @property
    def n_edges(self):
        return len(self.edge_u)

    def vertex_dof(self, v):
        return self.n_interior + v

    def node(self, e, j):
        """Global index of node j (0..n_e) along edge e; j=0 is edge_u, j=n_e is edge_v."""
        if j == 0:
            return self.n_interior + int(self.edge_u[e])
        if j == int(self.n_el[e]):
            return self.n_interior + int(self.edge_v[e])
        return int(self.offset[e]) + j - 1

    def degrees(self):
        """d_v = number of incident edge ENDS (a loop counts twice), SURVEY §8c Q9 / SPEC S33."""
        d = np.zeros(self.n_vertices, dtype=np.int64)
        np.add.at(d, self.edge_u, 1)
        np.add.at(d, self.edge_v, 1)
        return d


def validate(n_vertices, edge_u, edge_v, length, h):
    """Input validation (SPEC S22-29, S42; self-loops accepted per SURVEY §8c Q18)."""
    if n_vertices < 1:
        raise ValueError("n_vertices must be >= 1")
    if not (math.isfinite(h) and h > 0):
        raise ValueError("h must be positive and finite")
    eu = np.asarray(edge_u)
    ev = np.asarray(edge_v)
    ln = np.asarray(length, dtype=np.float64)
    if len(eu) < 1 or len(eu) != len(ev) or len(eu) != len(ln):
        raise ValueError("edge arrays must be non-empty and of equal length")
    if eu.min() < 0 or ev.min() < 0 or eu.max() >= n_vertices or ev.max() >= n_vertices:
        raise ValueError("edge endpoint out of range")
    if not np.all(np.isfinite(ln)) or np.any(ln <= 0):
        raise ValueError("edge lengths must be positive and finite")
    deg = np.zeros(n_vertices, dtype=np.int64)
    np.add.at(deg, eu, 1)
    np.add.at(deg, ev, 1)
    if np.any(deg == 0):
        raise ValueError("isolated vertex (zero lumped mass)")


def build_mesh(graph, h: float) -> Mesh:
    validate(graph.n_vertices, graph.edge_u, graph.edge_v, graph.length, h)
    length = np.asarray(graph.length, dtype=np.float64)
    n_el = np.array([max(1, math.ceil(float(l) / h)) for l in length], dtype=np.int64)
    h_e = length / n_el
    m_int = n_el - 1
    offset = np.zeros(len(length), dtype=np.int64)
    if len(length) > 1:
        offset[1:] = np.cumsum(m_int)[:-1]
    n_interior = int(m_int.sum())
    return Mesh(int(graph.n_vertices), np.asarray(graph.edge_u, dtype=np.int64),
                np.asarray(graph.edge_v, dtype=np.int64), length, float(h), n_el, h_e,
                m_int, offset, n_interior, n_interior + int(graph.n_vertices))


def node_positions(mesh: Mesh):
    """(edge_id or -1, vertex_id or -1, local x) for every DOF (SPEC S110-118, S464)."""
    N = mesh.n_dofs
    edge = np.full(N, -1, dtype=np.int64)
    vert = np.full(N, -1, dtype=np.int64)
    x = np.zeros(N)
    for e in range(mesh.n_edges):
        o, m = int(mesh.offset[e]), int(mesh.m_int[e])
        edge[o:o + m] = e
        x[o:o + m] = np.arange(1, m + 1) * mesh.h_e[e]
    vert[mesh.n_interior:] = np.arange(mesh.n_vertices)
    return edge, vert, x
