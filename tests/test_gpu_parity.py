"""GPU parity: the CUDA path through the C ABI vs the CPU oracle (BASELINE north_star).

Bars (north_star): noise bit-exact; fields <= 1e-9 relative L2 per sample with PCG at
rtol 1e-13.  Intermediate stage: the local Schur blocks of K2 vs their dense definition
(oracle/dd.py) to 1e-12.  Inputs are the seeded synthetic graphs of synth/.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import dd, noise, solve  # noqa: E402
from synth import CONFIGS, MetricGraph, config_graph, lattice, single_edge, star_of_lattices, tadpole  # noqa: E402

FIELD_TOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _graph(g, h):
    from paper_2605_02670_b200 import Graph
    return Graph.from_metric_graph(g, h)


def _rel(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


# ----------------------------------------------------------------------------- noise
def test_noise_bitexact_tadpole():
    G = _graph(tadpole(), 0.01)
    W = G.noise(5, 3).cpu().numpy()
    prob = solve.setup(tadpole(), 0.01, 5.0, 0.75, 0.5)
    ref = noise.white_noise(prob.ML, 5, 3)
    assert np.array_equal(_bits(W), _bits(ref))
    assert np.array_equal(G.lumped_mass(), prob.ML)


def test_noise_bitexact_lattice_256_samples_sampled():
    """Full config-3 noise call (256 x 198325); the oracle recomputes sampled rows / columns."""
    cfg = CONFIGS["lattice256"]
    g = config_graph("lattice256")
    G = _graph(g, cfg["h"])
    W = G.noise(cfg["seed"], cfg["n_samples"])
    prob = solve.setup(g, cfg["h"], cfg["kappa"], cfg["beta"], cfg["k"])
    rng = np.random.default_rng(0)
    rows = [0, 1, 127, 255]
    cols = np.unique(np.concatenate([rng.integers(0, G.n_dofs, 4000), [0, G.n_interior - 1, G.n_interior,
                                                                       G.n_dofs - 1]]))
    Wc = W[:, torch.as_tensor(cols, device=W.device)].cpu().numpy()
    for s in range(0, 256, 15):
        ref = noise.white_noise(prob.ML, cfg["seed"], 256, dofs=cols, samples=[s])[0]
        assert np.array_equal(_bits(Wc[s]), _bits(ref)), f"sample {s}"
    for s in rows:
        ref = noise.white_noise(prob.ML, cfg["seed"], 256, samples=[s])[0]
        assert np.array_equal(_bits(W[s].cpu().numpy()), _bits(ref)), f"row {s}"


def test_noise_large_seed_wraps():
    G = _graph(single_edge(1.0), 0.1)
    seed = 2 ** 64 - 2
    W = G.noise(seed, 4).cpu().numpy()
    prob = solve.setup(single_edge(1.0), 0.1, 1.0, 0.6, 0.3)
    ref = noise.white_noise(prob.ML, seed, 4)
    assert np.array_equal(_bits(W), _bits(ref))


# ----------------------------------------------------------------------------- K2 stage
@pytest.mark.parametrize("gname,h,kappa,beta,k", [("tadpole", 0.01, 5.0, 0.75, 0.5),
                                                  ("lattice4", 0.05, 10.0, 0.6, 0.3),
                                                  ("short", 0.01, 2.0, 0.55, 0.3)])
def test_edge_schur_vs_definition(gname, h, kappa, beta, k):
    g = {"tadpole": tadpole(), "lattice4": lattice(4, seed=2),
         "short": MetricGraph(3, np.array([0, 1, 1, 2]), np.array([1, 2, 2, 2]),
                              np.array([0.004, 0.7, 0.015, 0.33]))}[gname]
    G = _graph(g, h)
    sig = G.edge_schur(kappa, beta, k)
    prob = solve.setup(g, h, kappa, beta, k)
    for li in range(0, prob.plan.n_nodes, max(1, prob.plan.n_nodes // 12)):
        for e in range(g.n_edges):
            S = dd.local_schur(prob, li, e)
            scale = abs(S[0, 0])
            assert abs(sig[li, e, 0] - S[0, 0]) <= 1e-12 * scale
            assert abs(sig[li, e, 1] - S[0, 1]) <= 1e-12 * scale


# ----------------------------------------------------------------------------- fields
def test_config1_tadpole():
    cfg = CONFIGS["tadpole"]
    g = tadpole()
    G = _graph(g, cfg["h"])
    u, st = G.sample(cfg["kappa"], cfg["beta"], cfg["k"], seed=cfg["seed"], n_samples=1, return_stats=True)
    ref, _, _ = solve.sample(g, cfg["h"], cfg["kappa"], cfg["beta"], cfg["k"], cfg["seed"], 1)
    assert _rel(u.cpu().numpy(), ref).max() <= FIELD_TOL
    assert st["n_unconverged"] == 0 and st["iter_max"] <= 2 and st["n_nodes"] == 55


@pytest.mark.parametrize("gname", ["lattice4", "star2", "multi_loop_short", "single"])
def test_per_node_solves(gname):
    """node_range = [l, l+1) returns the single node solve x_l = A_l^{-1} W (c-form, P76)."""
    g, h = {"lattice4": (lattice(4, seed=1), 0.05), "star2": (star_of_lattices(2, 3), 0.125),
            "multi_loop_short": (MetricGraph(3, np.array([0, 0, 1, 1, 2]), np.array([1, 1, 2, 1, 2]),
                                             np.array([0.5, 0.8, 0.004, 0.3, 0.21])), 0.01),
            "single": (single_edge(0.77), 0.01)}[gname]
    kappa, beta, k = 3.0, 0.65, 0.3
    G = _graph(g, h)
    prob = solve.setup(g, h, kappa, beta, k)
    W = noise.white_noise(prob.ML, 9, 2)
    for li in sorted({0, 1, prob.plan.n_nodes // 2, prob.plan.n_nodes - 1}):
        u = G.sample(kappa, beta, k, seed=9, n_samples=2, node_range=(li, li + 1)).cpu().numpy()
        ref = solve.node_solve(prob, li, W)
        assert _rel(u, ref).max() <= 1e-10, f"node {li}"


@pytest.mark.parametrize("precond", ["nn", "jacobi", "none"])
def test_small_graph_all_preconditioners(precond):
    g = lattice(5, seed=3)
    h, kappa, beta, k = 0.02, 2.0, 0.7, 0.35
    G = _graph(g, h)
    u, st = G.sample(kappa, beta, k, seed=1, n_samples=5, precond=precond, return_stats=True)
    ref, _, _ = solve.sample(g, h, kappa, beta, k, 1, 5)
    assert _rel(u.cpu().numpy(), ref).max() <= FIELD_TOL
    assert st["n_unconverged"] == 0 and st["worst_true_rel_residual"] <= 1e-11


@pytest.mark.parametrize("n_samples", [5, 8])
def test_fused_rhs_assembly_small_calls(n_samples):
    """Calls of <= 8 samples: the warp PCG assembles its rhs from the end values itself (K4a fused,
    pcg.cu launch_pcg; 8 = one full octet, the 16-byte run loads; 5 = a partial octet).  Fields vs
    the oracle; the call without statistics (rhs never written) equals the call with them bitwise;
    the same samples from a 9-sample call (separate K4a) agree to rounding."""
    g = lattice(6, seed=2)
    h, kappa, beta, k = 0.04, 3.0, 0.7, 0.3
    G = _graph(g, h)
    u, st = G.sample(kappa, beta, k, seed=3, n_samples=n_samples, return_stats=True)
    u = u.cpu().numpy()
    ref, _, _ = solve.sample(g, h, kappa, beta, k, 3, n_samples)
    assert _rel(u, ref).max() <= FIELD_TOL
    assert st["n_unconverged"] == 0 and st["worst_true_rel_residual"] <= 1e-11
    plain = G.sample(kappa, beta, k, seed=3, n_samples=n_samples).cpu().numpy()
    assert np.array_equal(_bits(u), _bits(plain))
    nine = G.sample(kappa, beta, k, seed=3, n_samples=9).cpu().numpy()
    assert _rel(nine[:n_samples], u).max() <= 1e-12


def test_ragged_and_degenerate_edges():
    """Edges with 0, 1, 2 interior nodes, a loop with n_e = 1, multi-edges; odd sample count."""
    g = MetricGraph(4, np.array([0, 0, 1, 1, 2, 3, 2, 0]), np.array([1, 1, 2, 1, 3, 3, 0, 3]),
                    np.array([0.01, 0.019, 0.031, 0.005, 0.9, 0.008, 0.43, 1.37]))
    h, kappa, beta, k = 0.01, 4.0, 0.8, 0.3
    G = _graph(g, h)
    u = G.sample(kappa, beta, k, seed=4, n_samples=3).cpu().numpy()
    ref, _, _ = solve.sample(g, h, kappa, beta, k, 4, 3)
    assert _rel(u, ref).max() <= FIELD_TOL


def test_single_edge_one_pcg_iteration():
    G = _graph(single_edge(1.0), 0.01)
    _, st = G.sample(3.0, 0.7, 0.4, seed=0, n_samples=2, return_stats=True)
    assert st["iter_max"] <= 2 and st["iter_min"] >= 1
    assert st["n_unconverged"] == 0


def test_seed_convention_and_determinism():
    g = lattice(4, seed=5)
    G = _graph(g, 0.05)
    a = G.sample(5.0, 0.6, 0.3, seed=0, n_samples=6).cpu().numpy()
    b = G.sample(5.0, 0.6, 0.3, seed=3, n_samples=1).cpu().numpy()
    c = G.sample(5.0, 0.6, 0.3, seed=0, n_samples=6).cpu().numpy()
    # the noise is bit-identical; the field's sum over nodes may be grouped differently for a
    # different sample count (the lane mapping depends on it), so it agrees to rounding
    assert np.array_equal(_bits(G.noise(0, 6).cpu().numpy()[3]), _bits(G.noise(3, 1).cpu().numpy()[0]))
    assert _rel(a[3], b[0]) <= 1e-13
    # the same call is bitwise reproducible (fixed-order reductions, no atomics on data)
    assert np.array_equal(_bits(a), _bits(c))


@pytest.mark.parametrize("pcg", ["auto", "global"])
def test_repeat_calls_bitwise_identical(pcg):
    # stress for shared-memory / queue races in the persistent sweep kernels (items fetched one
    # ahead, folds of the previous block, mbarrier phases), the PCG kernels and the chunked host
    # path: ten calls on the config-3 lattice with two sample tiles must agree bit for bit
    G = _graph(lattice(32, seed=0), 0.05)
    ref = G.sample(10.0, 0.75, 0.25, seed=11, n_samples=64, pcg=pcg).cpu().numpy()
    for _ in range(9):
        again = G.sample(10.0, 0.75, 0.25, seed=11, n_samples=64, pcg=pcg).cpu().numpy()
        assert np.array_equal(_bits(ref), _bits(again))
    host = G.sample_host(10.0, 0.75, 0.25, seed=11, n_samples=64, pcg=pcg)
    assert np.array_equal(_bits(ref), _bits(host))


def test_apply_equals_sample_on_noise():
    g = lattice(3, seed=6)
    G = _graph(g, 0.05)
    W = G.noise(2, 3)
    u1 = G.sample(2.0, 0.6, 0.3, seed=2, n_samples=3)
    u2 = G.apply(2.0, 0.6, 0.3, W)
    assert torch.equal(u1, u2)
    u3 = G.apply(2.0, 0.6, 0.3, W.clone(), out=None)
    assert torch.equal(u1, u3)


def test_node_range_partial_sums_add_up():
    """sum over node shards == full sum (the multi-GPU l-sharding identity)."""
    g = lattice(4, seed=7)
    G = _graph(g, 0.05)
    kappa, beta, k = 3.0, 0.7, 0.4
    full = G.sample(kappa, beta, k, seed=1, n_samples=2).cpu().numpy()
    L = solve.setup(g, 0.05, kappa, beta, k).plan.n_nodes
    cuts = [0, L // 3, L // 2, L]
    parts = sum(G.sample(kappa, beta, k, seed=1, n_samples=2, node_range=(a, b)).cpu().numpy()
                for a, b in zip(cuts[:-1], cuts[1:]))
    assert _rel(parts, full).max() <= 1e-13


@pytest.mark.parametrize("n_samples", [2, 70, 100, 256, 257, 1000])
def test_host_output_matches_device(n_samples):
    # n_samples >= 64 runs grf_sample_host in overlapped chunks (70: 38 / 32; 100: 36 / 32 / 32;
    # 256: 64 x 3 / 32 / 32; 257: 64 x 3 / 33 / 32; 1000: 192 x 4 / 168 / 32 / 32): every chunk
    # reseeds with seed + its first sample, so the field is bitwise the one-call field
    g = lattice(3, seed=8)
    G = _graph(g, 0.05)
    a = G.sample(2.0, 0.6, 0.3, seed=7, n_samples=n_samples).cpu().numpy()
    b, st = G.sample_host(2.0, 0.6, 0.3, seed=7, n_samples=n_samples, return_stats=True)
    assert np.array_equal(_bits(a), _bits(b))
    assert st["n_systems"] == n_samples * st["n_nodes"]
    assert st["worst_rel_residual"] <= 1e-13


@pytest.mark.parametrize("n_samples", [2, 70, 256])
def test_pinned_host_output_matches_device(n_samples):
    # a page-locked buffer is mapped into the device: grf_sample_host's last chunk (all of it below
    # 64 samples) is written by the recovery kernels straight into it, the earlier chunks through
    # the staged copies -- bitwise the one-call device field either way
    g = lattice(3, seed=8)
    G = _graph(g, 0.05)
    a = G.sample(2.0, 0.6, 0.3, seed=7, n_samples=n_samples).cpu().numpy()
    host = torch.full((n_samples, G.n_dofs), float("nan"), dtype=torch.float64, pin_memory=True)
    G.sample_into_host(2.0, 0.6, 0.3, 7, n_samples, host)
    assert np.array_equal(_bits(a), _bits(host.numpy()))


@pytest.mark.parametrize("n_samples", [20, 70])
def test_pinned_host_output_long_edges(n_samples):
    # edges longer than the recovery's output tile are folded into u by read-modify-write, which
    # must not run over PCIe: such a last chunk goes through the staged copy (same field)
    g = MetricGraph(5, np.array([0, 1, 2, 0, 3, 3, 2]), np.array([1, 2, 3, 2, 4, 4, 2]),
                    np.array([6.0, 4.5, 1.505, 0.3, 0.02, 0.9, 0.6]))
    G = _graph(g, 0.005)
    a = G.sample(2.0, 0.7, 0.35, seed=6, n_samples=n_samples).cpu().numpy()
    host = torch.full((n_samples, G.n_dofs), float("nan"), dtype=torch.float64, pin_memory=True)
    G.sample_into_host(2.0, 0.7, 0.35, 6, n_samples, host)
    assert np.array_equal(_bits(a), _bits(host.numpy()))


def test_nonfinite_output_is_reported():
    """An infinite right-hand side (grf_apply) gives non-finite fields: the exit check reports them
    (GRF_ENOCONV with statistics) instead of returning silently."""
    from paper_2605_02670_b200 import GrfError
    G = _graph(lattice(3, seed=2), 0.1)
    rhs = torch.zeros((2, G.n_dofs), dtype=torch.float64, device="cuda")
    rhs[1, 3] = float("inf")
    with pytest.raises(GrfError):
        G.apply(2.0, 0.6, 0.3, rhs, return_stats=True)


def test_sample_into_host_checks_its_buffer():
    """grf_sample_host writes n x N doubles into the caller's buffer: a wrong size, dtype or device
    is rejected before the call (no out-of-bounds host write)."""
    G = _graph(lattice(3, seed=2), 0.1)
    for bad in (torch.empty((2, G.n_dofs - 1), dtype=torch.float64),
                torch.empty((2, G.n_dofs), dtype=torch.float32),
                torch.empty((2, G.n_dofs), dtype=torch.float64, device="cuda")):
        with pytest.raises(ValueError):
            G.sample_into_host(2.0, 0.6, 0.3, 0, 2, bad)
    ok = torch.empty((2, G.n_dofs), dtype=torch.float64)
    G.sample_into_host(2.0, 0.6, 0.3, 0, 2, ok)
    assert torch.equal(ok, G.sample(2.0, 0.6, 0.3, seed=0, n_samples=2).cpu())


def test_invalid_arguments():
    from paper_2605_02670_b200 import GrfError
    G = _graph(single_edge(1.0), 0.1)
    for kw in (dict(kappa=0.0, beta=0.6, k=0.3), dict(kappa=1.0, beta=0.2, k=0.3),
               dict(kappa=1.0, beta=0.6, k=-1.0)):
        with pytest.raises(GrfError):
            G.sample(kw["kappa"], kw["beta"], kw["k"], n_samples=1)
    with pytest.raises(GrfError):
        G.sample(1.0, 0.6, 0.3, n_samples=1, node_range=(5, 2))


# ----------------------------------------------------------------------------- BASELINE configs
def test_config2_lattice_one_sample():
    """configs[1] at full size: N = 198325, L = 259 (oracle ~45 s on CPU)."""
    cfg = CONFIGS["lattice1"]
    g = config_graph("lattice1")
    G = _graph(g, cfg["h"])
    u, st = G.sample(cfg["kappa"], cfg["beta"], cfg["k"], seed=cfg["seed"], n_samples=1, return_stats=True)
    ref, _, _ = solve.sample(g, cfg["h"], cfg["kappa"], cfg["beta"], cfg["k"], cfg["seed"], 1)
    assert _rel(u.cpu().numpy(), ref).max() <= FIELD_TOL
    assert st["n_nodes"] == 259 and st["n_unconverged"] == 0


def test_config3_lattice_256_samples_sampled():
    """configs[2] at full size in the bench launch configuration (256 samples in one call);
    the oracle recomputes samples 0, 101, 255 (all 212 nodes)."""
    cfg = CONFIGS["lattice256"]
    g = config_graph("lattice256")
    G = _graph(g, cfg["h"])
    u, st = G.sample(cfg["kappa"], cfg["beta"], cfg["k"], seed=cfg["seed"], n_samples=cfg["n_samples"],
                     return_stats=True)
    assert st["n_nodes"] == 212 and st["n_unconverged"] == 0
    # exit checks: the TRUE residual of every vertex system, no non-finite output,
    # and the per-phase device times
    assert 0.0 < st["worst_true_rel_residual"] <= 1e-11 and st["n_nonfinite"] == 0
    assert all(st["phase_ms"][k] > 0.0 for k in ("noise", "condense", "pcg", "recover"))
    picks = [0, 101, 255]
    ref, _, _ = solve.sample(g, cfg["h"], cfg["kappa"], cfg["beta"], cfg["k"], cfg["seed"], cfg["n_samples"],
                             samples=picks)
    got = u[picks].cpu().numpy()
    assert _rel(got, ref).max() <= FIELD_TOL
    # property at any size: every sample is finite and has the Matern-scale variance
    uu = u.cpu().numpy()
    assert np.isfinite(uu).all()


# ----------------------------------------------------------------------------- global-memory K4
@pytest.mark.parametrize("n_samples", [1, 3, 16, 20, 40])
def test_global_pcg_matches_oracle(n_samples):
    """The global-memory PCG (pcg_global.cu, used for V > 4096) forced on small graphs, for every
    sample mapping (1 / 16 / 32 samples per tile, ragged tile), vs the oracle."""
    g = lattice(5, seed=3)
    h, kappa, beta, k = 0.04, 2.0, 0.7, 0.4
    G = _graph(g, h)
    u, st = G.sample(kappa, beta, k, seed=2, n_samples=n_samples, pcg="global", return_stats=True)
    picks = sorted({0, n_samples // 2, n_samples - 1})
    ref, _, _ = solve.sample(g, h, kappa, beta, k, 2, n_samples, samples=picks)
    assert _rel(u.cpu().numpy()[picks], ref).max() <= FIELD_TOL
    assert st["n_unconverged"] == 0 and st["worst_rel_residual"] <= 1e-13


@pytest.mark.parametrize("precond", ["nn", "jacobi"])
def test_global_pcg_equals_shared(precond):
    g = star_of_lattices(2, 3)
    h, kappa, beta, k = 0.1, 3.0, 0.6, 0.35
    G = _graph(g, h)
    a = G.sample(kappa, beta, k, seed=5, n_samples=4, precond=precond, pcg="shared").cpu().numpy()
    b = G.sample(kappa, beta, k, seed=5, n_samples=4, precond=precond, pcg="global").cpu().numpy()
    assert _rel(b, a).max() <= 1e-11


def test_rgg_5000_per_node_vs_oracle():
    """A 5000-vertex config-4-style graph (V > 4096: the global-memory PCG is selected
    automatically): single-node solves vs the oracle's sparse direct solve."""
    from synth import rgg_knn
    g = rgg_knn(5000, k=3, scale=300.0 * (5000 / 100_000) ** 0.5, seed=1)
    h, kappa, beta, k = 0.02, 2.0, 0.55, 0.6
    G = _graph(g, h)
    prob = solve.setup(g, h, kappa, beta, k)
    W = noise.white_noise(prob.ML, 3, 2)
    L = prob.plan.n_nodes
    for li in (0, L // 2, L - 1):
        u, st = G.sample(kappa, beta, k, seed=3, n_samples=2, node_range=(li, li + 1), return_stats=True)
        ref = solve.node_solve(prob, li, W)
        assert _rel(u.cpu().numpy(), ref).max() <= 1e-10, f"node {li}"
        assert st["n_unconverged"] == 0


def test_config4_rgg_full_size():
    """configs[3] at full size on one GPU in the production launch: 1e5 vertices,
    N = 28 032 313, L = 112, 16 samples in one call (the global-memory PCG; sweep kernels of the
    16-sample mapping).  The oracle (C sparse LDL^T with the interior-first + minimum-degree
    ordering) recomputes samples 0 and 15 over all 112 nodes: fields <= 1e-9
    relative L2, noise bit-exact."""
    cfg = CONFIGS["rgg"]
    g = config_graph("rgg")
    G = _graph(g, cfg["h"])
    u, st = G.sample(cfg["kappa"], cfg["beta"], cfg["k"], seed=cfg["seed"], n_samples=cfg["n_samples"],
                     return_stats=True)
    assert G.n_dofs == 28_032_313
    assert st["n_nodes"] == 112 and st["n_unconverged"] == 0 and st["worst_rel_residual"] <= 1e-13
    assert st["worst_true_rel_residual"] <= 1e-11 and st["n_nonfinite"] == 0
    picks = [0, 15]
    got = u[picks].cpu().numpy()
    del u
    Wg = G.noise(cfg["seed"], cfg["n_samples"])[picks].cpu().numpy()
    del G
    torch.cuda.empty_cache()
    ref, Wref, _ = solve.sample(g, cfg["h"], cfg["kappa"], cfg["beta"], cfg["k"], cfg["seed"], cfg["n_samples"],
                                samples=picks)
    assert np.array_equal(_bits(Wg), _bits(Wref))
    assert np.isfinite(got).all()
    assert _rel(got, ref).max() <= FIELD_TOL


# ----------------------------------------------------------------------------- config 5 (star of lattices)
@pytest.mark.parametrize("beta", [0.3, 0.5, 0.75, 0.9])
def test_config5_star_coarsest_all_betas(beta):
    """configs[4] at h = 2^-4 (N = 59 769), every beta of the sweep (L = 296 / 249 / 331 / 687),
    kappa = 8, k = 0.2, 64 samples in one call; the oracle recomputes samples 0 and 63."""
    g = star_of_lattices(8, 16)
    h, kappa, k = 2.0 ** -4, 8.0, 0.2
    G = _graph(g, h)
    u, st = G.sample(kappa, beta, k, seed=0, n_samples=64, return_stats=True)
    assert st["n_nodes"] == {0.3: 296, 0.5: 249, 0.75: 331, 0.9: 687}[beta]
    assert st["n_unconverged"] == 0
    ref, _, _ = solve.sample(g, h, kappa, beta, k, 0, 64, samples=[0, 63])
    assert _rel(u.cpu().numpy()[[0, 63]], ref).max() <= FIELD_TOL


def test_config5_star_default_level():
    """configs[4] at the CONFIGS level h = 2^-8 (N = 983 289, L = 331, 64 samples in one call);
    the oracle recomputes samples 0, 31 and 63 over all 331 nodes."""
    cfg = CONFIGS["star"]
    g = config_graph("star")
    G = _graph(g, cfg["h"])
    u, st = G.sample(cfg["kappa"], cfg["beta"], cfg["k"], seed=cfg["seed"], n_samples=cfg["n_samples"],
                     return_stats=True)
    assert G.n_dofs == 983_289 and st["n_nodes"] == 331 and st["n_unconverged"] == 0
    picks = [0, 31, 63]
    got = u[picks].cpu().numpy()
    assert bool(torch.isfinite(u).all())
    ref, _, _ = solve.sample(g, cfg["h"], cfg["kappa"], cfg["beta"], cfg["k"], cfg["seed"], cfg["n_samples"],
                             samples=picks)
    assert _rel(got, ref).max() <= FIELD_TOL


def test_config5_star_finest_level():
    """configs[4] at the finest level h = 2^-12 (N = 15 759 609, edges of 4095 interior nodes:
    longer than the recovery kernel's shared-memory output tile) with beta = 0.9 (L = 687, the
    largest rule), 64 samples in one call; the oracle recomputes samples 0 and 63 over all 687
    nodes (a stated subset of the 64 samples; fields <= 1e-9 relative L2)."""
    g = star_of_lattices(8, 16)
    h, kappa, beta, k = 2.0 ** -12, 8.0, 0.9, 0.2
    G = _graph(g, h)
    u, st = G.sample(kappa, beta, k, seed=0, n_samples=64, return_stats=True)
    assert G.n_dofs == 15_759_609 and st["n_nodes"] == 687 and st["n_unconverged"] == 0
    assert bool(torch.isfinite(u).all())
    picks = [0, 63]
    got = u[picks].cpu().numpy()
    del u, G
    torch.cuda.empty_cache()
    ref, _, _ = solve.sample(g, h, kappa, beta, k, 0, 64, samples=picks)
    assert _rel(got, ref).max() <= FIELD_TOL


@pytest.mark.parametrize("n_samples", [20, 40])
def test_long_edges_direct_accumulation(n_samples):
    """Edges with 1199 / 899 / 300 interior nodes (l = 6, 4.5, 1.505 at h = 0.005) next to short
    ones: with >= 17 samples the recovery's shared-memory output tile cannot hold the long edges,
    which then accumulate straight into u (sweep_impl.cuh); fields vs the oracle."""
    g = MetricGraph(5, np.array([0, 1, 2, 0, 3, 3, 2]), np.array([1, 2, 3, 2, 4, 4, 2]),
                    np.array([6.0, 4.5, 1.505, 0.3, 0.02, 0.9, 0.6]))
    h, kappa, beta, k = 0.005, 2.0, 0.7, 0.35
    G = _graph(g, h)
    u, st = G.sample(kappa, beta, k, seed=6, n_samples=n_samples, return_stats=True)
    assert st["n_unconverged"] == 0
    picks = sorted({0, 17, n_samples - 1})
    ref, _, _ = solve.sample(g, h, kappa, beta, k, 6, n_samples, samples=picks)
    assert _rel(u.cpu().numpy()[picks], ref).max() <= FIELD_TOL


# ----------------------------------------------------------------------------- NEXT-1 strong-error study
def test_nested_transfer_kernels_vs_oracle():
    """grf_project_noise / grf_prolong vs the oracle's hat-function matrices (P335, SPEC S119-127)."""
    from oracle.mesh import build_mesh
    from oracle.refine import prolongation
    from paper_2605_02670_b200.study import project_noise, prolong
    g = MetricGraph(4, np.array([0, 0, 1, 2, 3]), np.array([1, 2, 2, 3, 3]),
                    np.array([1.0, 0.5, 0.75, 1.25, 0.5]))  # includes a loop edge (3, 3)
    hc, hf = 0.25, 0.25 / 4
    Gc, Gf = _graph(g, hc), _graph(g, hf)
    P = prolongation(build_mesh(g, hc), build_mesh(g, hf))
    rng = np.random.default_rng(0)
    uc = rng.standard_normal((3, Gc.n_dofs))
    wf = rng.standard_normal((3, Gf.n_dofs))
    up = prolong(Gc, Gf, torch.from_numpy(uc).cuda()).cpu().numpy()
    wc = project_noise(Gf, Gc, torch.from_numpy(wf).cuda()).cpu().numpy()
    assert np.abs(up - (P @ uc.T).T).max() <= 1e-15
    assert np.abs(wc - (P.T @ wf.T).T).max() <= 1e-14
    with pytest.raises(Exception):
        prolong(_graph(g, 0.22), Gf, torch.zeros((1, _graph(g, 0.22).n_dofs), dtype=torch.float64, device="cuda"))


def test_strong_error_study_vs_oracle():
    """The whole study pipeline on a small star of lattices: per-realization squared errors vs
    the oracle's definition (oracle/refine.strong_error)."""
    from oracle.refine import strong_error
    from paper_2605_02670_b200.study import strong_error as gpu_study
    g = star_of_lattices(2, 3)
    kappa, beta, k, ok = 4.0, 0.75, 0.5, 5
    res = gpu_study(g, [2, 3], ok, kappa, beta, k, seed=11, n_samples=4, batch=4)
    Gf = _graph(g, 2.0 ** -ok)
    W = Gf.noise(11, 4).cpu().numpy()
    for j in (2, 3):
        ref = strong_error(g, 2.0 ** -j, 2.0 ** -ok, kappa, beta, k, W)
        assert np.max(np.abs(res["per_sample_sq"][j] - ref) / ref) <= 1e-9


# ----------------------------------------------------------------------------- hubs (CSR operator tables)
def test_hub_graph_csr_tables_vs_oracle():
    """A vertex with 41 incident edge ends (> 32: CSR operator tables, global-memory PCG) plus a
    loop and a multi-edge at the hub, vs the oracle."""
    n_leaf = 40
    eu = np.concatenate([np.zeros(n_leaf, np.int64), [0, 1, 0]])
    ev = np.concatenate([np.arange(1, n_leaf + 1), [0, 2, 1]])
    ln = np.concatenate([np.linspace(0.3, 1.1, n_leaf), [0.7, 0.45, 0.9]])
    g = MetricGraph(n_leaf + 1, eu, ev, ln)
    h, kappa, beta, k = 0.1, 2.0, 0.7, 0.45
    G = _graph(g, h)
    u, st = G.sample(kappa, beta, k, seed=3, n_samples=3, return_stats=True)
    ref, _, _ = solve.sample(g, h, kappa, beta, k, 3, 3)
    assert _rel(u.cpu().numpy(), ref).max() <= FIELD_TOL
    assert st["n_unconverged"] == 0


def test_barabasi_albert_per_node_vs_oracle():
    """The paper's §4.3 workload family (P340-341): Barabasi-Albert m = 2, unit edges, h = 2^-6;
    n = 2000 (hubs of degree > 32 -> CSR tables); single-node solves vs the oracle."""
    from synth import barabasi_albert
    g = barabasi_albert(2000, 2, seed=0)
    h, kappa, beta = 2.0 ** -6, 1.0, 0.75
    k = -1.0 / (beta * np.log(h))  # the paper's step rule (P335)
    G = _graph(g, h)
    prob = solve.setup(g, h, kappa, beta, k)
    assert prob.plan.n_nodes == 131
    W = noise.white_noise(prob.ML, 0, 2)
    for li in (0, 65, 130):
        x = G.sample(kappa, beta, k, seed=0, n_samples=2, node_range=(li, li + 1)).cpu().numpy()
        assert _rel(x, solve.node_solve(prob, li, W)).max() <= 1e-10, f"node {li}"


def test_covariance_vs_oracle():
    """NEXT-4: C = B M_L B from batched grf_apply on unit columns vs the oracle's definition
    (B from oracle.solve.apply on the identity)."""
    from paper_2605_02670_b200.study import covariance
    g = tadpole()
    h, kappa, beta, k = 0.125, 5.0, 0.75, 0.4
    G = _graph(g, h)
    C = covariance(G, kappa, beta, k, batch=7).cpu().numpy()
    prob = solve.setup(g, h, kappa, beta, k)
    B = solve.apply(prob, np.eye(prob.mesh.n_dofs))
    Cref = B @ np.diag(prob.ML) @ B.T
    assert np.abs(C - Cref).max() <= 1e-10 * np.abs(Cref).max()
    assert np.allclose(C, C.T, rtol=0, atol=1e-14 * np.abs(C).max())


# ----------------------------------------------------------------------------- NEXT-3 consistent mass
@pytest.mark.parametrize("gname", ["tadpole", "ragged", "lattice"])
def test_consistent_mass_vs_oracle(gname):
    """Consistent mass in operator and noise (P129-150): noise R xi vs the oracle's dense
    natural-order Cholesky (same xi; different arithmetic order, so to rounding), field to 1e-9."""
    from oracle import consistent
    from oracle.mesh import build_mesh
    g, h = {"tadpole": (tadpole(), 0.05),
            "ragged": (MetricGraph(4, np.array([0, 0, 1, 1, 2, 3, 2, 0]), np.array([1, 1, 2, 1, 3, 3, 0, 3]),
                                   np.array([0.01, 0.019, 0.031, 0.005, 0.9, 0.008, 0.43, 1.37])), 0.01),
            "lattice": (lattice(4, seed=2), 0.05)}[gname]
    kappa, beta, k = 4.0, 0.7, 0.35
    G = _graph(g, h)
    W = G.noise(5, 3, mass="consistent").cpu().numpy()
    Wref = consistent.white_noise(build_mesh(g, h), 5, 3)
    assert np.abs(W - Wref).max() <= 1e-13 * np.abs(Wref).max()
    u, st = G.sample(kappa, beta, k, seed=5, n_samples=3, mass="consistent", return_stats=True)
    ref, _ = consistent.sample(g, h, kappa, beta, k, 5, 3)
    assert _rel(u.cpu().numpy(), ref).max() <= FIELD_TOL
    assert st["n_unconverged"] == 0
    # the consistent field is a different discretization from the lumped one (but close)
    ul = G.sample(kappa, beta, k, seed=5, n_samples=3).cpu().numpy()
    assert _rel(ul, ref).max() > 1e-6
