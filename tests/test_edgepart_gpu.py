"""Edge-partitioned sampling on the GPU (grf_sample_edgepart) vs the oracle and vs
the whole-graph call.  All parts run in this process (comm = NULL: halo and dot sums on the
device); the NCCL path is exercised with a one-rank communicator."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import solve  # noqa: E402
from paper_2605_02670_b200 import Graph, sample_edgepart  # noqa: E402
from paper_2605_02670_b200.edgepart import gather, make_parts, partition  # noqa: E402
from synth import CONFIGS, config_graph, lattice, star_of_lattices, tadpole  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _rel(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)


def _run_parts(g, h, P, kappa, beta, k, seed, S, xy=None, **opts):
    G = Graph.from_metric_graph(g, h)
    ep, _ = partition(G, P, xy=xy)
    gs = make_parts(G, ep, P)
    us, st = sample_edgepart(gs, kappa, beta, k, seed=seed, n_samples=S, return_stats=True, **opts)
    return gather(gs, [u.cpu().numpy() for u in us], G.n_dofs), st, ep, gs


@pytest.mark.parametrize("gname,h,P,geo", [("lattice5", 0.05, 2, False), ("lattice5", 0.05, 3, True),
                                           ("star", 0.25, 4, False), ("tadpole", 0.1, 2, False),
                                           ("rgg", 0.05, 5, True), ("lattice5", 0.05, 1, False)])
def test_library_partition_structure(gname, h, P, geo):
    """grf_partition_edges + grf_graph_create_part: every edge in exactly one non-empty part; each
    vertex owned once; the parts' global DOF maps (grf_graph_part_dofs) cover the whole graph with
    interiors exactly once; part noise = whole-graph noise at the part's DOFs (so the whole-graph
    vertex masses and global counters are used); balanced DOF weights."""
    from synth import rgg_knn
    g = {"lattice5": lattice(5, seed=1), "star": star_of_lattices(3, 3), "tadpole": tadpole(),
         "rgg": rgg_knn(600, k=3, scale=300.0 * (600 / 100_000) ** 0.5, seed=2)}[gname]
    G = Graph.from_metric_graph(g, h)
    ep, info = partition(G, P, xy=g.coords if geo else None)
    assert ep.shape == (g.n_edges,) and ep.min() >= 0 and ep.max() < P and info["empty_parts"] == 0
    gs = make_parts(G, ep, P)
    seen = np.zeros(G.n_dofs, int)
    for q, Gq in enumerate(gs):
        assert Gq.n_edges == int((ep == q).sum())
        d = Gq.part_dofs()
        seen[d] += 1
        Wq = Gq.noise(7, 2).cpu().numpy()
        assert np.array_equal(Wq.view(np.uint64), G.noise(7, 2).cpu().numpy()[:, d].view(np.uint64))
    NI = G.n_interior
    assert np.all(seen[:NI] == 1) and np.all(seen[NI:] >= 1)
    touched = np.zeros(g.n_vertices, int)
    for q in range(P):
        vs = np.unique(np.concatenate([g.edge_u[ep == q], g.edge_v[ep == q]]))
        touched[vs] += 1
    assert info["n_interface"] == int((touched > 1).sum())
    w = np.bincount(ep, weights=np.maximum(1, np.ceil(g.length / h)), minlength=P)
    assert info["max_part_weight"] == int(w.max()) and w.max() <= 2.0 * w.mean() + np.ceil(g.length / h).max()


@pytest.mark.parametrize("P,S", [(1, 2), (2, 1), (2, 3), (3, 16), (4, 20)])
def test_edgepart_matches_oracle(P, S):
    g = lattice(5, seed=1)
    h, kappa, beta, k = 0.05, 2.0, 0.7, 0.4
    u, st, _, _ = _run_parts(g, h, P, kappa, beta, k, seed=3, S=S)
    assert np.isfinite(u).all()
    picks = sorted({0, S - 1})
    ref, _, _ = solve.sample(g, h, kappa, beta, k, 3, S, samples=picks)
    assert _rel(u[picks], ref).max() <= 1e-9
    assert st["n_unconverged"] == 0 and st["worst_rel_residual"] <= 1e-13


def test_edgepart_noise_and_interfaces_consistent():
    """Interface vertices get the same value on every part that holds them; the parts' noise is the
    whole graph's noise (global Philox counters, whole-graph vertex masses)."""
    g = star_of_lattices(3, 4)
    h = 0.125
    whole = Graph.from_metric_graph(g, h)
    ep, _ = partition(whole, 3)
    gs = make_parts(whole, ep, 3)
    Wall = whole.noise(7, 2).cpu().numpy()
    for G in gs:
        assert np.array_equal(G.noise(7, 2).cpu().numpy().view(np.uint64), Wall[:, G.part_dofs()].view(np.uint64))
    us = sample_edgepart(gs, 3.0, 0.6, 0.35, seed=7, n_samples=2)
    vals = {}
    NI = whole.n_interior
    for G, u in zip(gs, us):
        uu = u.cpu().numpy()
        for i, d in enumerate(G.part_dofs()):
            if d < NI:
                continue
            x = uu[:, i]
            if d in vals:
                assert np.allclose(vals[d], x, rtol=1e-12, atol=1e-14)
            vals[d] = x


def test_edgepart_equals_whole_graph_rgg():
    from synth import rgg_knn
    g = rgg_knn(5000, k=3, scale=300.0 * (5000 / 100_000) ** 0.5, seed=1)
    h, kappa, beta, k = 0.02, 2.0, 0.55, 0.6
    whole = Graph.from_metric_graph(g, h).sample(kappa, beta, k, seed=4, n_samples=16).cpu().numpy()
    for P, geo in ((2, False), (5, True)):
        u, st, _, _ = _run_parts(g, h, P, kappa, beta, k, seed=4, S=16, xy=g.coords if geo else None)
        assert _rel(u, whole).max() <= 1e-10, f"P={P}"


def test_edgepart_nccl_one_rank():
    """The NCCL code path (grf_comm) with a one-rank communicator."""
    import os
    import tempfile

    import torch.distributed as dist

    from paper_2605_02670_b200 import Comm
    # a file rendezvous: no TCP port to collide with the previous test's store (EADDRINUSE)
    fd, path = tempfile.mkstemp(prefix="grf_pg_")
    os.close(fd)
    os.unlink(path)
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=0, world_size=1)
    try:
        comm = Comm()
        g = lattice(4, seed=3)
        h = 0.05
        W = Graph.from_metric_graph(g, h)
        ep, _ = partition(W, 1)
        G = make_parts(W, ep, 1)[0]
        u = sample_edgepart([G], 3.0, 0.7, 0.4, seed=1, n_samples=4, comm=comm)[0].cpu().numpy()
        ref = W.sample(3.0, 0.7, 0.4, seed=1, n_samples=4).cpu().numpy()
        assert _rel(gather([G], [u], ref.shape[1]), ref).max() <= 1e-11
        comm.close()
    finally:
        dist.destroy_process_group()


def test_config4_edge_partitioned_two_parts():
    """configs[3] (1e5 vertices, N = 2.8e7, L = 112, 16 samples) split into 2 edge parts, both on
    this GPU, vs the whole-graph call."""
    import gc
    cfg = CONFIGS["rgg"]
    g = config_graph("rgg")
    G = Graph.from_metric_graph(g, cfg["h"])
    whole = G.sample(cfg["kappa"], cfg["beta"], cfg["k"], seed=0, n_samples=16)[[0, 15]].cpu().numpy()
    del G
    gc.collect()
    torch.cuda.empty_cache()
    u, st, _, _ = _run_parts(g, cfg["h"], 2, cfg["kappa"], cfg["beta"], cfg["k"], seed=0, S=16, xy=g.coords)
    assert st["n_unconverged"] == 0
    assert _rel(u[[0, 15]], whole).max() <= 1e-10


def test_sample_dist_one_rank():
    """grf_sample_dist (sample-then-node sharding in the library) with a one-rank communicator."""
    import os
    import tempfile

    import torch.distributed as dist

    from paper_2605_02670_b200 import Comm
    from paper_2605_02670_b200.grf import sample_dist
    # a file rendezvous: no TCP port to collide with the previous test's store (EADDRINUSE)
    fd, path = tempfile.mkstemp(prefix="grf_pg_")
    os.close(fd)
    os.unlink(path)
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=0, world_size=1)
    try:
        comm = Comm()
        G = Graph.from_metric_graph(lattice(4, seed=3), 0.05)
        u, rng, root = sample_dist(G, comm, 3.0, 0.7, 0.4, seed=2, n_samples=5)
        ref = G.sample(3.0, 0.7, 0.4, seed=2, n_samples=5)
        assert rng == (0, 5) and root
        assert torch.equal(u, ref)
        comm.close()
    finally:
        dist.destroy_process_group()
