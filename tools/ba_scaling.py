"""NEXT-2: the paper's §4.3 workload on B200 (P340-341, P460-484): Barabasi-Albert graphs (m = 2,
star-seeded, unit edges) with n = 100 .. 50 000 vertices at h = 2^-6; lumped mass; kappa = 1,
beta = 0.75, k = -1/(beta ln h) (the paper's step rule, L = 131 nodes).  Times one GRF sample
(the paper's "full_nrf" task, 1 sample per call) and the noise alone ("noise_only"), and a
16-sample call, with CUDA events (median of 5 after 2 warm-ups).  Linear scaling in N is the
check (the paper's lumped pipeline is ~68k instructions per DOF at every size).

    python tools/ba_scaling.py r01
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_02670_b200 import Graph  # noqa: E402
from synth import barabasi_albert  # noqa: E402

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
torch.cuda.set_device(0)
h, kappa, beta = 2.0 ** -6, 1.0, 0.75
k = -1.0 / (beta * np.log(h))


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


rows = []
for n in (100, 500, 1000, 2000, 5000, 10000, 20000, 50000):
    g = barabasi_albert(n, 2, seed=0)
    G = Graph.from_metric_graph(g, h)
    _, st = G.sample(kappa, beta, k, seed=0, n_samples=1, return_stats=True)
    t1 = timed(lambda: G.sample(kappa, beta, k, seed=0, n_samples=1))
    tn = timed(lambda: G.noise(0, 1))
    t16 = timed(lambda: G.sample(kappa, beta, k, seed=0, n_samples=16))
    L = st["n_nodes"]
    row = {"n": n, "N": G.n_dofs, "N_interior": G.n_interior, "max_degree": int(np.bincount(
        np.concatenate([g.edge_u, g.edge_v])).max()), "L": L, "ms_sample": t1, "ms_noise": tn, "ms_16_samples": t16,
        "iter_mean": st["iter_mean"], "iter_max": st["iter_max"], "iter_total_per_sample": st["iter_mean"] * L,
        "ns_per_dof_sample": 1e6 * t1 / G.n_dofs, "ns_per_dof_16": 1e6 * t16 / (16 * G.n_dofs)}
    rows.append(row)
    print(row, flush=True)
    del G
    torch.cuda.empty_cache()
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump({"h": h, "kappa": kappa, "beta": beta, "k": k, "rows": rows},
          open(os.path.join(ROOT, "profiles", f"{R}_ba_scaling.json"), "w"), indent=1)
with open(os.path.join(ROOT, "profiles", f"{R}_ba_scaling.md"), "w") as f:
    f.write(f"# {R} Barabasi-Albert scaling on B200 (PAPER.md §4.3, P340-341; SURVEY §8f NEXT-2)\n\n")
    f.write("BA(n, m = 2), star-seeded, unit edges, h = 2^-6 (N = 126 (n - 2) interior DOFs + n vertices), "
            f"lumped mass, kappa = 1, beta = 0.75, k = -1/(beta ln h) = {k:.4f}, L = 131 nodes. CUDA-event medians. "
            "Hubs of degree > 32 use the CSR operator tables and the global-memory PCG.\n\n")
    f.write("| n | N | max deg | noise ms | 1 sample ms | ns/DOF (1) | 16 samples ms | ns/DOF/sample (16) | PCG iters mean (max) |\n")
    f.write("|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        f.write(f"| {r['n']} | {r['N']} | {r['max_degree']} | {r['ms_noise']:.3f} | {r['ms_sample']:.2f} | "
                f"{r['ns_per_dof_sample']:.1f} | {r['ms_16_samples']:.2f} | {r['ns_per_dof_16']:.2f} | "
                f"{r['iter_mean']:.1f} ({r['iter_max']}) |\n")
print("written")
