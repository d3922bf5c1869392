"""DEFINITIONS of the domain-decomposition quantities (no DD algorithm).

Used by the tests to check the CUDA path's intermediate results and to pin the
paper's identities.  Everything is computed from its plain definition with
library solvers (scipy sparse LU, LAPACK banded/dense solves):

* local operator A^{(l,e)} = c_I M^{(e)} + c_L (kappa^2 M^{(e)} + G^{(e)}) on the edge
  nodes [u, interior..., v]; the ends carry only THIS edge's share
  (h_e/2 mass, 1/h_e stiffness)              PAPER.md P166-185, SURVEY §8c Q7
* local Schur S^{(l,e)} = A_GG - A_GI A_II^{-1} A_IG (2x2)   P204-213 [eq:local_reduced_schur]
* global Schur S^{(l)} = A_GG - A_GI A_II^{-1} A_IG (|V|x|V|) P113-116 [eq:global_schur]
* condensed rhs g = W_G - A_GI A_II^{-1} W_I                P116, SURVEY §8c Q6
* NN preconditioner D^{-1} (sum_e R_e^T S_e^{-1} R_e) D^{-1}  P298
* textbook PCG, zero start, stop at ||r||_2 <= rtol ||g||_2  P241-296, SURVEY §8c Q10
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from . import fem


def edge_coefficients(prob, li, e):
    """(a, b, vertex_share): interior diagonal, off-diagonal, per-end vertex share of A^{(l,e)}."""
    cI, cL = prob.plan.c_I[li], prob.plan.c_L[li]
    h = prob.mesh.h_e[e]
    k2 = prob.kappa * prob.kappa
    mass = cI + k2 * cL
    a = mass * h + 2.0 * cL / h
    b = -cL / h
    share = mass * h / 2.0 + cL / h
    return a, b, share


def local_schur(prob, li, e):
    """2x2 S^{(l,e)} over (left end, right end) from its definition."""
    a, b, share = edge_coefficients(prob, li, e)
    m = int(prob.mesh.m_int[e])
    if m == 0:
        return np.array([[share, b], [b, share]])
    ab = np.zeros((3, m))
    ab[0, 1:] = b
    ab[1, :] = a
    ab[2, :-1] = b
    rhs = np.zeros((m, 2))
    rhs[0, 0] = b   # A_IG column of the left end: coupling to interior node 1
    rhs[-1, 1] = b  # right end couples to interior node m
    X = sla.solve_banded((1, 1), ab, rhs)
    AGI = rhs.T
    return np.array([[share, 0.0], [0.0, share]]) - AGI @ X


def _blocks(prob, li):
    A = fem.operator(prob.ML, prob.G, prob.kappa, prob.plan.c_I[li], prob.plan.c_L[li]).tocsr()
    NI = prob.mesh.n_interior
    return A[:NI, :NI].tocsc(), A[:NI, NI:], A[NI:, :NI], A[NI:, NI:]


def global_schur(prob, li):
    """Dense S^{(l)} (tiny graphs only)."""
    AII, AIG, AGI, AGG = _blocks(prob, li)
    if AII.shape[0] == 0:
        return AGG.toarray()
    X = splu(AII).solve(AIG.toarray())
    return AGG.toarray() - AGI @ X


def condensed_rhs(prob, li, W):
    """g [S, V] for noise W [S, N]."""
    AII, AIG, AGI, AGG = _blocks(prob, li)
    NI = prob.mesh.n_interior
    W = np.atleast_2d(W)
    if NI == 0:
        return W[:, NI:].copy()
    w = splu(AII).solve(np.ascontiguousarray(W[:, :NI].T))
    return W[:, NI:] - (AGI @ w).T


def recover_interior(prob, li, W, uG):
    """u_I from A_II u_I = W_I - A_IG u_G   (P306-311 [eq:internal_recovery])."""
    AII, AIG, AGI, AGG = _blocks(prob, li)
    NI = prob.mesh.n_interior
    W = np.atleast_2d(W)
    if NI == 0:
        return np.zeros((W.shape[0], 0))
    rhs = W[:, :NI].T - AIG @ np.atleast_2d(uG).T
    return splu(AII).solve(np.ascontiguousarray(rhs)).T


def nn_preconditioner(prob, li):
    """Dense D^{-1} (sum_e R_e^T S_e^{-1} R_e) D^{-1}   (P298), loops map both ends to v."""
    V = prob.mesh.n_vertices
    d = prob.mesh.degrees().astype(np.float64)
    P = np.zeros((V, V))
    for e in range(prob.mesh.n_edges):
        Se = local_schur(prob, li, e)
        Si = np.linalg.inv(Se)
        ends = (int(prob.mesh.edge_u[e]), int(prob.mesh.edge_v[e]))
        for i in range(2):
            for j in range(2):
                P[ends[i], ends[j]] += Si[i, j]
    Dinv = np.diag(1.0 / d)
    return Dinv @ P @ Dinv


def assembled_schur(prob, li):
    """sum_e R_e^T S_e R_e  (P244 [eq:goal_func_1]); equals global_schur by P242."""
    V = prob.mesh.n_vertices
    S = np.zeros((V, V))
    for e in range(prob.mesh.n_edges):
        Se = local_schur(prob, li, e)
        ends = (int(prob.mesh.edge_u[e]), int(prob.mesh.edge_v[e]))
        for i in range(2):
            for j in range(2):
                S[ends[i], ends[j]] += Se[i, j]
    return S


def pcg(S, g, Minv, rtol=1e-13, max_iter=None):
    """Textbook PCG, x0 = 0, stop when ||r||_2 <= rtol ||g||_2.  Returns (x, iterations)."""
    n = len(g)
    max_iter = n + 10 if max_iter is None else max_iter
    x = np.zeros(n)
    r = g.copy()
    gn = np.linalg.norm(g)
    if gn == 0.0:
        return x, 0
    z = Minv @ r
    p = z.copy()
    rz = r @ z
    for it in range(1, max_iter + 1):
        q = S @ p
        alpha = rz / (p @ q)
        x = x + alpha * p
        r = r - alpha * q
        if np.linalg.norm(r) <= rtol * gn:
            return x, it
        z = Minv @ r
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, max_iter
