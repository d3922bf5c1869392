"""Edge-partitioned sampling, host logic on CPU: the partition and what each part
needs from the whole graph, and the distributed NN-PCG algorithm of dist.cu run in numpy by
two gloo ranks (halo sums of the interface vertices and dot products over owned vertices by
torch.distributed all_reduce) against the oracle's dense global Schur solve."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dd, fem, solve
from _edgepart_ref import element_counts, gather, partition
from synth import lattice, star_of_lattices, tadpole


@pytest.mark.parametrize("gname,h,P", [("lattice5", 0.05, 2), ("lattice5", 0.05, 3), ("star", 0.25, 4),
                                       ("tadpole", 0.1, 2), ("lattice5", 0.05, 1)])
def test_partition_structure(gname, h, P):
    g = {"lattice5": lattice(5, seed=1), "star": star_of_lattices(3, 3), "tadpole": tadpole()}[gname]
    parts = partition(g, h, P)
    prob = solve.setup(g, h, 2.0, 0.7, 0.5)
    mesh = prob.mesh
    # every edge in exactly one part, parts non-empty
    allE = np.concatenate([p.edges for p in parts])
    assert sorted(allE.tolist()) == list(range(g.n_edges)) and all(p.n_edges > 0 for p in parts)
    # each vertex owned exactly once; interface ids exactly for vertices of several parts
    own = np.zeros(g.n_vertices, int)
    cnt = np.zeros(g.n_vertices, int)
    for p in parts:
        own[p.vertices] += p.vertex_owned
        cnt[p.vertices] += 1
    assert np.all(own == 1)
    n_if = int((cnt > 1).sum())
    for p in parts:
        assert p.n_interface == n_if
        assert np.array_equal(p.vertex_iface >= 0, cnt[p.vertices] > 1)
        # whole-graph data: lumped vertex mass bit-identical to the oracle's, global degrees
        ML = prob.ML
        assert np.array_equal(p.vertex_mass, ML[mesh.n_interior + p.vertices])
        assert np.array_equal(p.vertex_degree, mesh.degrees()[p.vertices])
        # local edges keep their global orientation
        assert np.array_equal(p.vertices[p.edge_u], g.edge_u[p.edges])
        assert np.array_equal(p.vertices[p.edge_v], g.edge_v[p.edges])
    # the parts' global DOF maps cover the whole DOF range; interiors exactly once
    seen = np.zeros(mesh.n_dofs, int)
    for p in parts:
        seen[p.dof_gid(h)] += 1
    assert np.all(seen[:mesh.n_interior] == 1) and np.all(seen[mesh.n_interior:] >= 1)
    # gather puts local values at their global DOFs
    f = [p.dof_gid(h)[None, :].astype(float) for p in parts]
    assert np.array_equal(gather(parts, f, h, mesh.n_dofs)[0], np.arange(mesh.n_dofs, dtype=float))


# ----------------------------------------------------------------------------- distributed PCG on 2 gloo ranks
def _part_operators(prob, part, li):
    """This part's edge contributions to the vertex Schur operator and the NN preconditioner
    (local numbering; the NN step uses the GLOBAL degrees d_v), from the oracle's local Schur blocks."""
    V = part.n_vertices
    S = np.zeros((V, V))
    M = np.zeros((V, V))
    for le, e in enumerate(part.edges):
        Se = dd.local_schur(prob, li, int(e))
        Si = np.linalg.inv(Se)
        ends = (int(part.edge_u[le]), int(part.edge_v[le]))
        for i in range(2):
            for j in range(2):
                S[ends[i], ends[j]] += Se[i, j]
                M[ends[i], ends[j]] += Si[i, j]
    Dinv = np.diag(1.0 / part.vertex_degree)
    return S, Dinv @ M @ Dinv


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = lattice(4, seed=2)
    h, kappa, beta, k = 0.1, 2.0, 0.7, 0.6
    prob = solve.setup(g, h, kappa, beta, k)
    part = partition(g, h, world)[rank]
    li = prob.plan.n_nodes // 2
    rng = np.random.default_rng(5)
    W = rng.standard_normal(prob.mesh.n_dofs)  # a fixed right-hand side (same on both ranks)
    g_full = dd.condensed_rhs(prob, li, W)[0]  # assembled condensed rhs (reference only)
    S, M = _part_operators(prob, part, li)
    iface = part.vertex_iface
    n_if = part.n_interface

    def halo(xp):  # partial values -> totals at interface vertices (sum over ranks)
        buf = torch.zeros(max(n_if, 1), dtype=torch.float64)
        m = iface >= 0
        buf[torch.from_numpy(iface[m])] = torch.from_numpy(xp[m])
        dist.all_reduce(buf)
        y = xp.copy()
        y[m] = buf.numpy()[iface[m]]
        return y

    def dot(a, b):  # over owned vertices, then over ranks
        t = torch.tensor([float(np.sum((a * b)[part.vertex_owned == 1]))], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    # the part's partial condensed rhs (P233-239): W_v on owned vertices, minus the
    # condensation A_GI A_II^{-1} W_I of this part's edges only, each at its two end vertices
    gp = np.where(part.vertex_owned == 1, W[prob.mesh.n_interior + part.vertices], 0.0)
    import scipy.linalg as sla
    for le, e in enumerate(part.edges):
        a, b, _ = dd.edge_coefficients(prob, li, int(e))
        m = int(prob.mesh.m_int[e])
        if m == 0:
            continue
        off = int(prob.mesh.offset[e])
        ab = np.zeros((3, m))
        ab[0, 1:] = b
        ab[1, :] = a
        ab[2, :-1] = b
        w = sla.solve_banded((1, 1), ab, W[off:off + m])
        gp[part.edge_u[le]] -= b * w[0]
        gp[part.edge_v[le]] -= b * w[-1]
    gl = g_full[part.vertices]
    r = halo(gp)
    assert np.allclose(r, gl, rtol=0, atol=1e-14)
    x = np.zeros_like(r)
    z = halo(M @ r)
    p = z.copy()
    rz = dot(r, z)
    gg = dot(r, r)
    for it in range(200):
        q = halo(S @ p)
        alpha = rz / dot(p, q)
        x = x + alpha * p
        r = r - alpha * q
        rr = dot(r, r)
        if rr <= 1e-26 * gg:
            break
        z = halo(M @ r)
        rzn = dot(r, z)
        p = z + (rzn / rz) * p
        rz = rzn
    out[rank] = (part.vertices.copy(), x.copy(), it)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_distributed_schur_pcg_matches_dense_solve():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    g = lattice(4, seed=2)
    h, kappa, beta, k = 0.1, 2.0, 0.7, 0.6
    prob = solve.setup(g, h, kappa, beta, k)
    li = prob.plan.n_nodes // 2
    rng = np.random.default_rng(5)
    W = rng.standard_normal(prob.mesh.n_dofs)
    gv = dd.condensed_rhs(prob, li, W)[0]
    uG = np.linalg.solve(dd.global_schur(prob, li), gv)
    got = np.full(g.n_vertices, np.nan)
    for verts, x, _ in out.values():
        # interface values must agree on every rank that holds them
        ok = ~np.isnan(got[verts])
        assert np.allclose(got[verts][ok], x[ok], rtol=1e-12, atol=1e-15)
        got[verts] = x
    assert np.linalg.norm(got - uG) / np.linalg.norm(uG) <= 1e-11
