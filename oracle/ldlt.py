"""Oracle direct solver for large meshes: sparse LDL^T with a fixed ordering.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Solves the definition's per-node systems

    A^{(l)} x_{l,s} = b_s,   A^{(l)} = c_I^{(l)} M_L + c_L^{(l)} (kappa^2 M_L + G)     (P75-78, P76)

and sums over the quadrature nodes in ascending l (P313-324, SPEC S323), like oracle.solve.apply,
but with the plain C factorization in ldlt.c instead of SuperLU, so that meshes of 1e7 DOFs
(configs 4 and 5) can be solved directly:

* ordering: the edge-interior DOFs first in their natural order, then
  the vertex block in a fill-reducing order of the vertex adjacency graph (minimum degree on
  A + A^T from SuperLU's ordering routine, a library primitive used only to pick the order).
  With the interiors first, eliminating an edge's chain from its edge_u end drags only that
  end vertex along (one fill entry per interior DOF: nnz(L) <= 2 N_I + the vertex block's), so
  the factor stays linear in N;
* the symbolic analysis (elimination tree, column counts) depends only on the pattern and is
  done once per mesh; the numeric factorization runs per node, in parallel threads (ctypes
  releases the GIL; each node has its own factor), and the node solutions are added in ascending
  l as they complete in order.

Pinned in tests/test_oracle_ldlt.py against the SuperLU path of oracle.solve on small graphs.
"""
from __future__ import annotations

import concurrent.futures as cf
import ctypes as C
import os
import subprocess

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ldlt.c")
LIB = os.path.join(HERE, "_build", "libldlt.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile ldlt.c (gcc, no FMA contraction) into oracle/_build/libldlt.so."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        tmp = LIB + f".{os.getpid()}.tmp"
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", tmp, SRC], check=True)
        os.replace(tmp, LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        lib = C.CDLL(build())
        i64p = C.POINTER(C.c_int64)
        f64p = C.POINTER(C.c_double)
        lib.ldlt_symbolic.restype = C.c_int64
        lib.ldlt_symbolic.argtypes = [C.c_int64, i64p, i64p, i64p, i64p, i64p, i64p, i64p]
        lib.ldlt_node_solve.restype = C.c_int64
        lib.ldlt_node_solve.argtypes = [C.c_int64, i64p, i64p, f64p, f64p, C.c_double, C.c_double, C.c_double,
                                        i64p, i64p, i64p, i64p, C.c_int64, f64p, f64p]
        _lib = lib
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def vertex_order(mesh) -> np.ndarray:
    """A fill-reducing elimination order of the vertices: minimum degree on the vertex adjacency
    pattern (each edge couples its two end vertices once its interior is eliminated), taken from
    SuperLU's MMD_AT_PLUS_A column ordering; of that permutation and its inverse the one with
    the smaller factor is kept (only the fill depends on this choice, never the result)."""
    V = mesh.n_vertices
    eu, ev = mesh.edge_u, mesh.edge_v
    rows = np.concatenate([eu, ev, np.arange(V)])
    cols = np.concatenate([ev, eu, np.arange(V)])
    vals = np.concatenate([-np.ones(2 * len(eu)), np.full(V, 4.0 * (2 * len(eu) + 1))])
    A = sp.csc_matrix((vals, (rows, cols)), shape=(V, V))
    lu = splu(A, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0, options=dict(SymmetricMode=True))
    pc = np.asarray(lu.perm_c, dtype=np.int64)
    best, best_nnz = None, None
    for cand in (pc, np.argsort(pc)):
        nnz = _symbolic(A.indptr.astype(np.int64), A.indices.astype(np.int64), cand)[2]
        if best is None or nnz < best_nnz:
            best, best_nnz = cand, nnz
    return best


def _symbolic(Ap, Ai, perm):
    n = len(perm)
    perm = np.ascontiguousarray(perm, dtype=np.int64)
    pinv = np.empty(n, dtype=np.int64)
    pinv[perm] = np.arange(n, dtype=np.int64)
    parent = np.empty(n, dtype=np.int64)
    lnz = np.empty(n, dtype=np.int64)
    flag = np.empty(n, dtype=np.int64)
    tot = _load().ldlt_symbolic(n, _p(Ap, C.c_int64), _p(Ai, C.c_int64), _p(perm, C.c_int64),
                                _p(pinv, C.c_int64), _p(parent, C.c_int64), _p(lnz, C.c_int64),
                                _p(flag, C.c_int64))
    return pinv, parent, int(tot), lnz


class Solver:
    """The per-mesh part of the direct solve: pattern of A (= pattern of G plus the diagonal),
    ordering and symbolic factorization.  `apply` then factors each node's A^{(l)}."""

    def __init__(self, mesh, G: sp.csr_matrix, ML: np.ndarray):
        N = mesh.n_dofs
        Gc = sp.csc_matrix(G)
        Gc.sort_indices()
        self.Ap = np.ascontiguousarray(Gc.indptr, dtype=np.int64)
        self.Ai = np.ascontiguousarray(Gc.indices, dtype=np.int64)
        self.Gx = np.ascontiguousarray(Gc.data, dtype=np.float64)
        # every column must hold its diagonal entry (it carries the mass term of A)
        cols = np.repeat(np.arange(N, dtype=np.int64), np.diff(self.Ap))
        has_diag = np.zeros(N, dtype=bool)
        has_diag[cols[self.Ai == cols]] = True
        if not has_diag.all():
            raise ValueError("stiffness pattern lacks diagonal entries")
        self.ML = np.ascontiguousarray(ML, dtype=np.float64)
        NI = mesh.n_interior
        self.perm = np.concatenate([np.arange(NI, dtype=np.int64), NI + vertex_order(mesh)])
        self.pinv, self.parent, self.nnz, lnz = _symbolic(self.Ap, self.Ai, self.perm)
        self.Lp = np.zeros(N + 1, dtype=np.int64)
        np.cumsum(lnz, out=self.Lp[1:])
        self.N = N

    def node_solve(self, cI, cL, kappa, rhs):
        """x [S, N] = (c_I M_L + c_L (kappa^2 M_L + G))^{-1} rhs [S, N]."""
        rhs = np.ascontiguousarray(np.atleast_2d(rhs), dtype=np.float64)
        x = np.empty_like(rhs)
        rc = _load().ldlt_node_solve(self.N, _p(self.Ap, C.c_int64), _p(self.Ai, C.c_int64),
                                     _p(self.Gx, C.c_double), _p(self.ML, C.c_double), float(cI), float(cL),
                                     float(kappa) ** 2, _p(self.perm, C.c_int64), _p(self.pinv, C.c_int64),
                                     _p(self.parent, C.c_int64), _p(self.Lp, C.c_int64), rhs.shape[0],
                                     _p(rhs, C.c_double), _p(x, C.c_double))
        if rc == -2:
            raise MemoryError("ldlt: factor allocation failed")
        if rc != -1:
            raise np.linalg.LinAlgError(f"ldlt: pivot {rc} not positive (A not SPD?)")
        return x

    def apply(self, plan, kappa, rhs, node_range=None, threads=None):
        """sum_{l in range} (A^{(l)})^{-1} rhs, added in ascending l (SPEC S323)."""
        rhs = np.ascontiguousarray(np.atleast_2d(rhs), dtype=np.float64)
        lo, hi = (0, plan.n_nodes) if node_range is None else node_range
        threads = threads or min(os.cpu_count() or 1, 16)
        u = np.zeros_like(rhs)
        with cf.ThreadPoolExecutor(max_workers=threads) as ex:
            for w0 in range(lo, hi, threads):  # a window of nodes in flight; summed in order
                futs = [ex.submit(self.node_solve, plan.c_I[li], plan.c_L[li], kappa, rhs)
                        for li in range(w0, min(hi, w0 + threads))]
                for f in futs:
                    u += f.result()
        return u
