"""Seeded metric-graph generators for the five BASELINE.json configs.

Every generator returns a :class:`MetricGraph` (vertex count + three edge
arrays).  Edge ``e = (u, v, length)`` is oriented: the local coordinate x runs
from 0 at ``u`` to ``length`` at ``v`` (PAPER.md P38, §2.1).  Self-loops
(u == v) and multi-edges are allowed (config 1 is a
tadpole whose first edge is a loop).

Recipes:

* cfg1 ``tadpole``: V={0,1}; e0=(0,0,2.0) loop, e1=(0,1,1.0).
* cfg2/3 ``lattice(32)``: vertex id 32*i+j; edges in row-major vertex order,
  right neighbour then down neighbour (1984 edges); lengths iid
  U[0.5,1.5] from ``numpy.random.default_rng(0).uniform`` in that order.
* cfg4 ``rgg_knn``: 1e5 points ``default_rng(0).uniform(0,1,(n,2))*300``,
  symmetric 3-NN union, components joined by the Euclidean-MST edges that
  connect them (Kruskal over Delaunay edges), lengths = Euclidean distance.
* cfg5 ``star_of_lattices``: hub vertex 0 + 8 unit-length 16x16 lattices,
  the hub joined by a unit edge to corner (0,0) of each lattice.
* NEXT-2 ``barabasi_albert(n, m=2)``: star-seeded preferential attachment,
  |E| = m(n-m) (the paper's variant, derived in SURVEY.md §6 from P476-483).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict

import numpy as np


@dataclasses.dataclass(frozen=True)
class MetricGraph:
    n_vertices: int
    edge_u: np.ndarray  # int64 [E]
    edge_v: np.ndarray  # int64 [E]
    length: np.ndarray  # float64 [E]
    name: str = "graph"
    coords: object = None  # optional float64 [V, 2] vertex positions (geometric graphs: partitioning)

    @property
    def n_edges(self) -> int:
        return int(self.edge_u.shape[0])

    def __post_init__(self):
        object.__setattr__(self, "edge_u", np.ascontiguousarray(self.edge_u, dtype=np.int64))
        object.__setattr__(self, "edge_v", np.ascontiguousarray(self.edge_v, dtype=np.int64))
        object.__setattr__(self, "length", np.ascontiguousarray(self.length, dtype=np.float64))


def _mk(nv, edges, lengths, name):
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    return MetricGraph(int(nv), edges[:, 0].copy(), edges[:, 1].copy(),
                       np.asarray(lengths, dtype=np.float64), name)


# --------------------------------------------------------------------------
# small graphs
# --------------------------------------------------------------------------
def tadpole() -> MetricGraph:
    """Config 1: loop edge of length 2 at vertex 0 plus pendant edge (0,1) of length 1."""
    return _mk(2, [(0, 0), (0, 1)], [2.0, 1.0], "tadpole")


def single_edge(length: float = 1.0) -> MetricGraph:
    return _mk(2, [(0, 1)], [length], "single_edge")


def path_graph(lengths) -> MetricGraph:
    lengths = list(lengths)
    return _mk(len(lengths) + 1, [(i, i + 1) for i in range(len(lengths))], lengths, "path")


def triangle_pendant() -> MetricGraph:
    """SPEC S44 / S512 default test graph: triangle {0,1},{1,2},{2,0} plus pendant {0,3}."""
    return _mk(4, [(0, 1), (1, 2), (2, 0), (0, 3)], [1.0] * 4, "triangle_pendant")


# --------------------------------------------------------------------------
# lattices
# --------------------------------------------------------------------------
def _lattice_edges(n: int, base: int = 0):
    edges = []
    for i in range(n):
        for j in range(n):
            v = base + n * i + j
            if j + 1 < n:
                edges.append((v, v + 1))
            if i + 1 < n:
                edges.append((v, v + n))
    return edges


def lattice(n: int = 32, seed: int = 0, lo: float = 0.5, hi: float = 1.5) -> MetricGraph:
    """Configs 2/3: n x n grid, lengths iid U[lo, hi] in edge order."""
    edges = _lattice_edges(n)
    rng = np.random.default_rng(seed)
    lengths = rng.uniform(lo, hi, size=len(edges))
    return _mk(n * n, edges, lengths, f"lattice{n}x{n}_seed{seed}")


def star_of_lattices(n_lattices: int = 8, side: int = 16) -> MetricGraph:
    """Config 5: hub vertex 0 joined by unit edges to corner (0,0) of n_lattices side x side unit lattices."""
    edges = []
    per = side * side
    for q in range(n_lattices):
        edges.extend(_lattice_edges(side, base=1 + q * per))
    for q in range(n_lattices):
        edges.append((0, 1 + q * per))
    nv = 1 + n_lattices * per
    return _mk(nv, edges, np.ones(len(edges)), f"star{n_lattices}x{side}x{side}")


# --------------------------------------------------------------------------
# random geometric k-NN graph (config 4)
# --------------------------------------------------------------------------
class _DSU:
    def __init__(self, n):
        self.p = np.arange(n, dtype=np.int64)

    def find(self, a):
        p = self.p
        root = a
        while p[root] != root:
            root = p[root]
        while p[a] != root:
            p[a], a = root, p[a]
        return root

    def union(self, a, b):
        ra, rb = self.find(a), self.find(b)
        if ra == rb:
            return False
        if ra < rb:
            self.p[rb] = ra
        else:
            self.p[ra] = rb
        return True


def rgg_knn(n: int = 100_000, k: int = 3, scale: float = 300.0, seed: int = 0) -> MetricGraph:
    """Config 4: symmetric k-NN union + MST bridges between components."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    from scipy.spatial import Delaunay, cKDTree

    rng = np.random.default_rng(seed)
    pts = rng.uniform(0.0, 1.0, (n, 2)) * scale
    tree = cKDTree(pts)
    _, idx = tree.query(pts, k=k + 1)
    a = np.repeat(np.arange(n, dtype=np.int64), k)
    b = idx[:, 1:].reshape(-1).astype(np.int64)
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    key = np.unique(lo * n + hi)
    eu = key // n
    ev = key % n
    # components of the kNN graph
    g = coo_matrix((np.ones(len(eu)), (eu, ev)), shape=(n, n))
    ncomp, labels = connected_components(g, directed=False)
    bu, bv = [], []
    if ncomp > 1:
        tri = Delaunay(pts)
        s = tri.simplices
        de = np.concatenate([s[:, [0, 1]], s[:, [1, 2]], s[:, [0, 2]]]).astype(np.int64)
        de.sort(axis=1)
        dkey = np.unique(de[:, 0] * n + de[:, 1])
        du, dv = dkey // n, dkey % n
        cu, cv = labels[du], labels[dv]
        mask = cu != cv
        du, dv, cu, cv = du[mask], dv[mask], cu[mask], cv[mask]
        dl = np.hypot(*(pts[du] - pts[dv]).T)
        order = np.lexsort((dv, du, dl))
        dsu = _DSU(ncomp)
        joined = 1
        for t in order:
            if dsu.union(int(cu[t]), int(cv[t])):
                bu.append(int(du[t]))
                bv.append(int(dv[t]))
                joined += 1
                if joined == ncomp:
                    break
    eu = np.concatenate([eu, np.asarray(bu, dtype=np.int64)])
    ev = np.concatenate([ev, np.asarray(bv, dtype=np.int64)])
    lengths = np.hypot(*(pts[eu] - pts[ev]).T)
    return MetricGraph(n, eu, ev, lengths, f"rgg{n}_knn{k}_seed{seed}", coords=pts)


# --------------------------------------------------------------------------
# Barabasi-Albert (NEXT-2)
# --------------------------------------------------------------------------
def barabasi_albert(n: int, m: int = 2, seed: int = 0, edge_length: float = 1.0) -> MetricGraph:
    """Star-seeded preferential attachment with |E| = m(n-m)."""
    if not (n > m >= 1):
        raise ValueError("barabasi_albert needs n > m >= 1")
    rng = np.random.default_rng(seed)
    edges = [(0, j) for j in range(1, m + 1)]
    targets = [0] * m + list(range(1, m + 1))  # endpoint multiset: P(v) ~ degree
    for v in range(m + 1, n):
        chosen = set()
        while len(chosen) < m:
            chosen.add(targets[int(rng.integers(len(targets)))])
        for u in sorted(chosen):
            edges.append((u, v))
            targets.extend((u, v))
    return _mk(n, edges, np.full(len(edges), edge_length), f"ba{n}_m{m}_seed{seed}")


# --------------------------------------------------------------------------
# text format (SPEC.md S79): "nv ne" then "u v length" per line, '#' comments
# --------------------------------------------------------------------------
def save_graph(g: MetricGraph, path) -> None:
    with open(path, "w") as f:
        f.write(f"{g.n_vertices} {g.n_edges}\n")
        for u, v, l in zip(g.edge_u, g.edge_v, g.length):
            f.write(f"{int(u)} {int(v)} {float(l)!r}\n")


def load_graph(path) -> MetricGraph:
    rows = []
    with open(path) as f:
        for line in f:
            s = line.split("#", 1)[0].strip()
            if s:
                rows.append(s.split())
    if not rows or len(rows[0]) != 2:
        raise ValueError("graph file: first line must be 'num_vertices num_edges'")
    nv, ne = int(rows[0][0]), int(rows[0][1])
    body = rows[1:]
    if len(body) != ne:
        raise ValueError(f"graph file: expected {ne} edges, found {len(body)}")
    eu, ev, ln = [], [], []
    for r in body:
        if len(r) != 3:
            raise ValueError(f"graph file: malformed edge line {' '.join(r)!r}")
        eu.append(int(r[0]))
        ev.append(int(r[1]))
        ln.append(float(r[2]))
    return MetricGraph(nv, np.array(eu), np.array(ev), np.array(ln), str(path))


# --------------------------------------------------------------------------
# the BASELINE.json configs
# --------------------------------------------------------------------------
CONFIGS: Dict[str, dict] = {
    # configs[0]
    "tadpole": dict(graph="tadpole", h=0.01, kappa=5.0, beta=0.75, k=0.5, seed=0, n_samples=1),
    # configs[1]
    "lattice1": dict(graph="lattice32", h=0.01, kappa=10.0, beta=0.6, k=0.2, seed=0, n_samples=1),
    # configs[2]
    "lattice256": dict(graph="lattice32", h=0.01, kappa=10.0, beta=0.75, k=0.25, seed=0, n_samples=256),
    # configs[3]
    "rgg": dict(graph="rgg", h=0.005, kappa=2.0, beta=0.55, k=0.3, seed=0, n_samples=16),
    # configs[4] (one point of the sweep; the sweep varies beta in {.3,.5,.75,.9}, h=2^-j, j=4..12)
    "star": dict(graph="star", h=2.0 ** -8, kappa=8.0, beta=0.75, k=0.2, seed=0, n_samples=64),
}


def config_graph(name: str) -> MetricGraph:
    g = CONFIGS[name]["graph"] if name in CONFIGS else name
    if g == "tadpole":
        return tadpole()
    if g == "lattice32":
        return lattice(32, seed=0)
    if g == "rgg":
        return rgg_knn()
    if g == "star":
        return star_of_lattices()
    raise KeyError(name)
