"""Seeded synthetic inputs (synth/): shapes of the BASELINE.json workloads."""
import numpy as np

from synth import (barabasi_albert, lattice, load_graph, save_graph, star_of_lattices, tadpole,
                   triangle_pendant)


def test_lattice_shape():
    g = lattice(32, seed=0)
    assert g.n_vertices == 1024 and g.n_edges == 1984
    assert 0.5 <= g.length.min() and g.length.max() <= 1.5
    assert (g.edge_u[0], g.edge_v[0], g.edge_u[1], g.edge_v[1]) == (0, 1, 0, 32)
    assert np.array_equal(g.length, np.random.default_rng(0).uniform(0.5, 1.5, 1984))


def test_star_of_lattices_shape():
    g = star_of_lattices()
    assert g.n_vertices == 2049 and g.n_edges == 3848 and np.all(g.length == 1.0)
    deg = np.bincount(np.concatenate([g.edge_u, g.edge_v]))
    assert deg[0] == 8


def test_tadpole():
    g = tadpole()
    assert g.n_vertices == 2 and list(g.edge_u) == [0, 0] and list(g.edge_v) == [0, 1]


def test_barabasi_albert_edge_count():
    for n in (3, 10, 100):
        g = barabasi_albert(n, 2, seed=1)
        assert g.n_edges == 2 * (n - 2)
        assert np.all(g.edge_u != g.edge_v)
        assert len(np.unique(np.concatenate([g.edge_u, g.edge_v]))) == n


def test_file_roundtrip(tmp_path):
    for g in (tadpole(), triangle_pendant(), lattice(4, seed=3)):
        p = tmp_path / "g.txt"
        save_graph(g, p)
        h = load_graph(p)
        assert h.n_vertices == g.n_vertices
        assert np.array_equal(h.edge_u, g.edge_u) and np.array_equal(h.edge_v, g.edge_v)
        assert np.array_equal(h.length, g.length)
