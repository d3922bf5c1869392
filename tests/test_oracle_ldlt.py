"""Pins for the oracle's C sparse LDL^T solver (oracle/ldlt.c, oracle/ldlt.py).

The LDL^T route (interior-first + minimum-degree-vertex ordering) is checked against a second,
independent direct solver -- scipy's SuperLU with COLAMD, a library LU -- on graphs with loops,
multi-edges, edges without interior nodes and hubs, and against the defining residual
A^{(l)} x = W (P75-78) with the operator assembled by oracle/fem.py.
"""
import numpy as np
import pytest

from oracle import fem, ldlt, noise, solve
from synth import MetricGraph, lattice, rgg_knn, star_of_lattices, tadpole

RAGGED = MetricGraph(4, np.array([0, 0, 1, 1, 2, 3, 2, 0]), np.array([1, 1, 2, 1, 3, 3, 0, 3]),
                     np.array([0.01, 0.019, 0.031, 0.005, 0.9, 0.008, 0.43, 1.37]), "ragged")


def _hub():
    n = 40
    eu = np.concatenate([np.zeros(n, np.int64), [0, 1, 0]])
    ev = np.concatenate([np.arange(1, n + 1), [0, 2, 1]])
    return MetricGraph(n + 1, eu, ev, np.concatenate([np.linspace(0.3, 1.1, n), [0.7, 0.45, 0.9]]), "hub")


@pytest.mark.parametrize("gname,h,kappa,beta,k", [
    ("tadpole", 0.01, 5.0, 0.75, 0.5), ("lattice", 0.05, 10.0, 0.6, 0.3), ("ragged", 0.01, 4.0, 0.8, 0.3),
    ("star", 0.125, 3.0, 0.65, 0.3), ("hub", 0.1, 2.0, 0.7, 0.45), ("rgg", 0.2, 2.0, 0.55, 0.6)])
def test_ldlt_equals_superlu(gname, h, kappa, beta, k):
    g = {"tadpole": tadpole(), "lattice": lattice(4, seed=2), "ragged": RAGGED, "star": star_of_lattices(2, 3),
         "hub": _hub(), "rgg": rgg_knn(300, k=3, scale=300.0 * (300 / 100_000) ** 0.5, seed=1)}[gname]
    prob = solve.setup(g, h, kappa, beta, k)
    W = noise.white_noise(prob.ML, 3, 3)
    a = solve.apply(prob, W, method="ldlt", threads=3)
    b = solve.apply(prob, W, method="superlu")
    assert np.linalg.norm(a - b, axis=1).max() / np.linalg.norm(b, axis=1).min() <= 1e-12
    for li in (0, prob.plan.n_nodes - 1):  # single nodes, both routes, and the defining residual
        x = solve.node_solve(prob, li, W, method="ldlt")
        y = solve.node_solve(prob, li, W, method="superlu")
        assert np.abs(x - y).max() <= 1e-12 * np.abs(y).max()
        A = fem.operator(prob.ML, prob.G, prob.kappa, prob.plan.c_I[li], prob.plan.c_L[li])
        r = (A @ x.T).T - W
        assert (np.linalg.norm(r, axis=1) / np.linalg.norm(W, axis=1)).max() <= 1e-13


def test_ldlt_node_ranges_add_up_and_threads_do_not_matter():
    g = lattice(3, seed=4)
    prob = solve.setup(g, 0.05, 3.0, 0.7, 0.4)
    W = noise.white_noise(prob.ML, 1, 2)
    L = prob.plan.n_nodes
    full = solve.apply(prob, W, threads=1)
    assert np.array_equal(full, solve.apply(prob, W, threads=5))  # summed in ascending l either way
    parts = solve.apply(prob, W, node_range=(0, L // 3)) + solve.apply(prob, W, node_range=(L // 3, L))
    assert np.abs(parts - full).max() <= 1e-14 * np.abs(full).max()


def test_ldlt_fill_is_linear_in_the_interior():
    """Interior-first natural order: each interior DOF has at most 2 off-diagonal factor entries
    (the next chain node and the chain's first vertex), so nnz(L) <= 2 N_I + (vertex block)."""
    g = lattice(6, seed=1)
    prob = solve.setup(g, 0.02, 2.0, 0.6, 0.4)
    s = prob.ldlt()
    NI, V = prob.mesh.n_interior, prob.mesh.n_vertices
    lnz = np.diff(s.Lp)
    assert lnz[:NI].max() <= 2
    assert s.nnz <= 2 * NI + V * (V - 1) // 2
    assert sorted(s.perm[NI:]) == list(range(NI, NI + V)) and np.array_equal(s.perm[:NI], np.arange(NI))


def test_ldlt_rejects_indefinite():
    g = tadpole()
    prob = solve.setup(g, 0.1, 1.0, 0.6, 0.4)
    with pytest.raises(np.linalg.LinAlgError):
        prob.ldlt().node_solve(-1.0, 1e-3, 1.0, np.ones((1, prob.mesh.n_dofs)))


def test_ldlt_builds_from_source(tmp_path, monkeypatch):
    monkeypatch.setattr(ldlt, "LIB", str(tmp_path / "libldlt.so"))
    assert ldlt.build(force=True).endswith("libldlt.so")
