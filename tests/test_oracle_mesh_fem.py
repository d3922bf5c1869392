"""Pins for oracle/mesh.py and oracle/fem.py (PAPER.md P122-160; SPEC S107-109, S179-190, S202-205)."""
import numpy as np
import pytest

from oracle import fem
from oracle.mesh import build_mesh, node_positions, validate
from synth import MetricGraph, lattice, single_edge, star_of_lattices, tadpole, triangle_pendant


def test_spec_mesh_examples():
    m = build_mesh(single_edge(1.0), 0.3)        # S107
    assert m.n_el[0] == 4 and m.h_e[0] == 0.25 and m.m_int[0] == 3
    m = build_mesh(single_edge(1.0), 1.0)        # S108
    assert m.n_el[0] == 1 and m.m_int[0] == 0 and m.n_dofs == 2
    m = build_mesh(triangle_pendant(), 2.0 ** -2)  # S109
    assert m.n_dofs == 16


def test_tadpole_dof_count():
    m = build_mesh(tadpole(), 0.01)
    assert m.n_dofs == 300            # 2 + 199 + 99
    assert m.n_interior == 298


def test_total_length_preserved():
    for g in (tadpole(), lattice(8), star_of_lattices(2, 4)):
        m = build_mesh(g, 0.013)
        assert np.isclose((m.n_el * m.h_e).sum(), g.length.sum(), rtol=1e-14)
        assert np.all(m.h_e <= 0.013 * (1 + 1e-15))


def test_node_positions():
    m = build_mesh(single_edge(1.0), 0.25)
    edge, vert, x = node_positions(m)
    assert x[0] == 0.25 and x[2] == 0.75    # S116, S118
    assert vert[-1] == 1 and edge[-1] == -1  # S117


def test_validation_errors():
    with pytest.raises(ValueError):
        validate(2, [0], [1], [-2.0], 0.1)   # S46
    with pytest.raises(ValueError):
        validate(2, [0], [2], [1.0], 0.1)
    with pytest.raises(ValueError):
        validate(3, [0], [1], [1.0], 0.1)    # isolated vertex 2
    with pytest.raises(ValueError):
        validate(2, [0], [1], [1.0], 0.0)
    validate(1, [0], [0], [1.0], 0.1)        # self-loop accepted


def test_lumped_mass_examples():
    # S179: interior node on edge h_e = 0.1 -> 0.1
    m = build_mesh(single_edge(1.0), 0.1)
    ML = fem.lumped_mass(m)
    assert np.all(ML[:m.n_interior] == m.h_e[0])
    # S180: degree-3 vertex, incident h_e = 0.25 -> 0.375
    m = build_mesh(triangle_pendant(), 0.25)
    ML = fem.lumped_mass(m)
    assert ML[m.vertex_dof(0)] == 0.375
    # tadpole vertex masses: (0.015, 0.005)
    m = build_mesh(tadpole(), 0.01)
    ML = fem.lumped_mass(m)
    assert np.isclose(ML[m.vertex_dof(0)], 0.015, rtol=1e-15)
    assert np.isclose(ML[m.vertex_dof(1)], 0.005, rtol=1e-15)


def test_total_mass_equals_total_length():
    for g in (tadpole(), lattice(8), star_of_lattices(2, 4)):
        m = build_mesh(g, 0.02)
        assert np.isclose(fem.lumped_mass(m).sum(), g.length.sum(), rtol=1e-13)


def test_lumped_is_consistent_row_sum():
    """P139-144: M^lumped_ii = sum_j M_ij, with M from the consistent stencil P129-136."""
    for g in (tadpole(), lattice(6), triangle_pendant()):
        m = build_mesh(g, 0.07)
        Mc = fem.consistent_mass(m)
        assert np.allclose(np.asarray(Mc.sum(axis=1)).ravel(), fem.lumped_mass(m), rtol=1e-14, atol=0)
    # S181: interior node, h_e = 0.3, consistent -> diagonal 0.2, neighbours 0.05
    m = build_mesh(single_edge(1.2), 0.3)
    Mc = fem.consistent_mass(m).toarray()
    assert np.isclose(Mc[1, 1], 0.2) and np.isclose(Mc[1, 0], 0.05) and np.isclose(Mc[1, 2], 0.05)


def test_stiffness_examples():
    # S188: interior node h_e = 0.5 -> diag 4, off -2
    m = build_mesh(single_edge(1.5), 0.5)
    G = fem.stiffness(m).toarray()
    assert G[0, 0] == 4.0 and G[0, 1] == -2.0 and G[0, m.vertex_dof(0)] == -2.0
    # S189: degree-1 vertex, h_e = 0.25 -> 4
    m = build_mesh(single_edge(1.0), 0.25)
    G = fem.stiffness(m).toarray()
    assert G[m.vertex_dof(0), m.vertex_dof(0)] == 4.0


def test_stiffness_kernel_and_psd():
    for g in (tadpole(), lattice(6), triangle_pendant()):
        m = build_mesh(g, 0.05)
        G = fem.stiffness(m)
        assert np.abs(G @ np.ones(m.n_dofs)).max() < 1e-10 * np.abs(G).max()   # S190
        assert abs(G - G.T).max() == 0
        x = np.random.default_rng(0).standard_normal((m.n_dofs, 20))
        assert np.all(np.einsum("ij,ij->j", x, G @ x) >= -1e-9)                # S205


def test_vertex_stencil_by_adjacency():
    """G_vv = sum_{e in E_v} 1/h_e, G_{v,adj(v,e)} = -1/h_e (P157-158), by walking the mesh."""
    g = MetricGraph(3, np.array([0, 1, 0]), np.array([1, 2, 2]), np.array([0.5, 0.7, 0.33]))
    m = build_mesh(g, 0.1)
    G = fem.stiffness(m).toarray()
    for v in range(3):
        dv = m.vertex_dof(v)
        expect = sum(1.0 / m.h_e[e] for e in range(3) if m.edge_u[e] == v) + \
            sum(1.0 / m.h_e[e] for e in range(3) if m.edge_v[e] == v)
        assert np.isclose(G[dv, dv], expect)
        for e in range(3):
            if m.edge_u[e] == v:
                assert np.isclose(G[dv, m.node(e, 1)], -1.0 / m.h_e[e])
            if m.edge_v[e] == v:
                assert np.isclose(G[dv, m.node(e, int(m.n_el[e]) - 1)], -1.0 / m.h_e[e])
