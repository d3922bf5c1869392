"""Debug: new sweep kernels vs the oracle on multi-item graphs (prints max rel error per case)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import solve
from synth import lattice, rgg_knn, star_of_lattices
from paper_2605_02670_b200 import Graph
torch.cuda.set_device(0)
cases = [
    ("rgg5000", rgg_knn(5000, k=3, scale=300.0 * (5000 / 100_000) ** 0.5, seed=1), 0.02, 2.0, 0.55, 0.6),
    ("lat12_h05", lattice(12, seed=1), 0.05, 2.0, 0.7, 0.4),
    ("lat12_h02", lattice(12, seed=1), 0.02, 2.0, 0.7, 0.4),
    ("lat12_k06", lattice(12, seed=1), 0.05, 2.0, 0.55, 0.6),
    ("star2", star_of_lattices(2, 4), 0.03125, 3.0, 0.6, 0.35),
]
for name, g, h, kappa, beta, k in cases:
    G = Graph.from_metric_graph(g, h)
    for S in (16, 32, 40):
        for pcg in ("auto", "global"):
            u = G.sample(kappa, beta, k, seed=2, n_samples=S, pcg=pcg).cpu().numpy()
            picks = sorted({0, 3, 5, S // 2, S - 1})
            ref, _, _ = solve.sample(g, h, kappa, beta, k, 2, S, samples=picks)
            rel = np.linalg.norm(u[picks] - ref, axis=1) / np.linalg.norm(ref, axis=1)
            print(f"{name:10s} N={G.n_dofs:7d} S={S:3d} pcg={pcg:6s} rel={np.array2string(rel, precision=1)}", flush=True)
