"""Pins of oracle/refine.py (nested prolongation, noise projection) against SPEC S119-127,
S256-264 and the properties the hat-function definition fixes."""
import numpy as np
import pytest

from oracle import fem
from oracle.mesh import build_mesh
from oracle.refine import prolongation
from synth import MetricGraph, single_edge, star_of_lattices, tadpole


def test_identity_when_meshes_coincide():  # SPEC S125
    m = build_mesh(tadpole(), 0.1)
    assert np.array_equal(prolongation(m, m).toarray(), np.eye(m.n_dofs))


def test_one_edge_midpoint_and_quarter_points():  # SPEC S126-127
    g = single_edge(1.0)
    c1, f2 = build_mesh(g, 1.0), build_mesh(g, 0.5)
    P = prolongation(c1, f2).toarray()
    mid = f2.node(0, 1)
    assert np.array_equal(P[mid, [c1.vertex_dof(0), c1.vertex_dof(1)]], [0.5, 0.5])
    c2, f4 = build_mesh(g, 0.5), build_mesh(g, 0.25)
    P = prolongation(c2, f4).toarray()
    x25 = f4.node(0, 1)  # fine node at x = 0.25
    assert P[x25, c2.vertex_dof(0)] == 0.5 and P[x25, c2.node(0, 1)] == 0.5
    # projection of the noise: coarse endpoint gets W_end + 1/2 W_mid (SPEC S262)
    W = np.zeros(f2.n_dofs)
    W[f2.vertex_dof(0)] = 3.0
    W[mid] = 4.0
    Wc = prolongation(c1, f2).T @ W
    assert Wc[c1.vertex_dof(0)] == 3.0 + 0.5 * 4.0


@pytest.mark.parametrize("jc,jf", [(2, 2), (2, 3), (2, 5), (3, 6)])
def test_partition_of_unity_and_linear_reproduction(jc, jf):
    g = star_of_lattices(2, 3)
    c, f = build_mesh(g, 2.0 ** -jc), build_mesh(g, 2.0 ** -jf)
    P = prolongation(c, f)
    assert np.allclose(P @ np.ones(c.n_dofs), 1.0, rtol=0, atol=1e-15)  # row sums = 1 (SPEC S122)
    # an edge-wise linear function is reproduced exactly: interpolate x along each edge
    xc = np.zeros(c.n_dofs)
    xf = np.zeros(f.n_dofs)
    for e in range(c.n_edges):
        for j in range(1, int(c.n_el[e])):
            xc[c.node(e, j)] = j * c.h_e[e]
        for j in range(1, int(f.n_el[e])):
            xf[f.node(e, j)] = j * f.h_e[e]
    # vertices are 0 in both; the hat interpolant of x on an edge is x wherever both ends are 0-based
    # (restrict the check to interior nodes away from the right end: value there depends on vertex data)
    lin = P @ xc
    for e in range(c.n_edges):
        r = int(f.n_el[e]) // int(c.n_el[e])
        for j in range(1, int(f.n_el[e]) - r):
            assert abs(lin[f.node(e, j)] - xf[f.node(e, j)]) <= 1e-14


def test_projected_lumped_mass_is_exact_for_constants():
    """P^T M_f 1 = M_c 1 on nested meshes (each coarse hat is the P-weighted sum of fine hats,
    and lumped row sums = hat integrals): the projection conserves total mass (SPEC S264)."""
    g = MetricGraph(3, np.array([0, 1, 0]), np.array([1, 2, 2]), np.array([1.0, 0.5, 0.75]))
    c, f = build_mesh(g, 0.25), build_mesh(g, 0.0625)
    P = prolongation(c, f)
    Mf, Mc = fem.lumped_mass(f), fem.lumped_mass(c)
    assert np.allclose(P.T @ Mf, Mc, rtol=1e-14, atol=0)


def test_non_nested_meshes_rejected():
    g = single_edge(1.0)
    with pytest.raises(ValueError):
        prolongation(build_mesh(g, 1 / 3), build_mesh(g, 1 / 4))
