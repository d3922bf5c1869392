"""Oracle Phase 2: P1-FEM matrices, assembled element by element (PAPER.md P126-160).

* lumped mass (P137-145): interior M_ii = h_e, vertex M_vv = sum_{e in E_v} h_e/2.
  Vertex sums run in ascending edge id, left end (u) before right end (v)
  (fixed order so the noise is bit-reproducible).
* consistent mass (P129-136): element matrix h_e/6 [[2,1],[1,2]].  Tests only
  (row sums == lumped diagonal, P139-144).
* stiffness (P152-160): element matrix [[1,-1],[-1,1]] / h_e, not lumped.
* operator (SPEC S207): K = kappa^2 M_L + G and
  A^{(l)} = c_I^{(l)} M_L + c_L^{(l)} K.

A loop element (both ends at v, n_e = 1) contributes h/2 + h/2 to M_vv and
nothing to G (its element stiffness sums to zero on the single node).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .mesh import Mesh


def element_nodes(mesh: Mesh):
    """Arrays (left, right, h) over all sum_e n_e elements, edge-major, ascending x."""
    E = mesh.n_edges
    n_el = mesh.n_el
    T = int(n_el.sum())
    edge = np.repeat(np.arange(E), n_el)
    start = np.zeros(E, dtype=np.int64)
    start[1:] = np.cumsum(n_el)[:-1]
    k = np.arange(T) - start[edge]
    off = mesh.offset[edge]
    NI = mesh.n_interior
    left = np.where(k == 0, NI + mesh.edge_u[edge], off + k - 1)
    right = np.where(k == n_el[edge] - 1, NI + mesh.edge_v[edge], off + k)
    return left, right, mesh.h_e[edge]


def lumped_mass(mesh: Mesh) -> np.ndarray:
    """Diagonal of M^lumped (P137-145)."""
    M = np.empty(mesh.n_dofs)
    for e in range(mesh.n_edges):
        o, m = int(mesh.offset[e]), int(mesh.m_int[e])
        M[o:o + m] = mesh.h_e[e] / 2 + mesh.h_e[e] / 2  # two elements share each interior node
    Mv = np.zeros(mesh.n_vertices)
    for e in range(mesh.n_edges):
        half = mesh.h_e[e] / 2
        Mv[mesh.edge_u[e]] += half
        Mv[mesh.edge_v[e]] += half
    M[mesh.n_interior:] = Mv
    return M


def stiffness(mesh: Mesh) -> sp.csr_matrix:
    """G (P152-160) as CSR with duplicates summed."""
    p, q, h = element_nodes(mesh)
    g = 1.0 / h
    rows = np.concatenate([p, q, p, q])
    cols = np.concatenate([p, q, q, p])
    vals = np.concatenate([g, g, -g, -g])
    N = mesh.n_dofs
    return sp.csr_matrix((vals, (rows, cols)), shape=(N, N))


def consistent_mass(mesh: Mesh) -> sp.csr_matrix:
    """Consistent M (P129-136); used by tests as a pin for the lumped diagonal."""
    p, q, h = element_nodes(mesh)
    d = h / 3.0
    o = h / 6.0
    rows = np.concatenate([p, q, p, q])
    cols = np.concatenate([p, q, q, p])
    vals = np.concatenate([d, d, o, o])
    N = mesh.n_dofs
    return sp.csr_matrix((vals, (rows, cols)), shape=(N, N))


def operator(ML: np.ndarray, G: sp.csr_matrix, kappa: float, c_I: float, c_L: float) -> sp.csc_matrix:
    """A^{(l)} = c_I M_L + c_L (kappa^2 M_L + G)  (P76 with SURVEY §8c Q3)."""
    K = sp.diags(kappa * kappa * ML) + G
    return (sp.diags(c_I * ML) + c_L * K).tocsc()
