"""NEXT-3 comparison (§4.3 Fig. 2, P462-484): lumped vs consistent mass on the paper's
Barabasi-Albert graphs (m = 2, h = 2^-6, kappa = 1, beta = 0.75, k = -1/(beta ln h)) on B200.
"noise" = W only; "full" = one GRF sample.  The consistent noise needs the natural-order Cholesky
factor of M, built once per graph (host, dense vertex Schur complement: O(V^3)) -- reported
separately as "factor s".  CUDA-event medians of 5 runs after 2 warm-ups.

    python tools/mass_comparison.py r01
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
for n in (100, 500, 1000, 2000, 5000):
    g = barabasi_albert(n, 2, seed=0)
    G = Graph.from_metric_graph(g, h)
    t0 = time.perf_counter()
    G.noise(0, 1, mass="consistent")
    torch.cuda.synchronize()
    factor_s = time.perf_counter() - t0
    row = {"n": n, "N": G.n_dofs, "factor_s": factor_s,
           "noise_lumped_ms": timed(lambda: G.noise(0, 1)),
           "noise_consistent_ms": timed(lambda: G.noise(0, 1, mass="consistent")),
           "full_lumped_ms": timed(lambda: G.sample(kappa, beta, k, seed=0, n_samples=1)),
           "full_consistent_ms": timed(lambda: G.sample(kappa, beta, k, seed=0, n_samples=1, mass="consistent"))}
    rows.append(row)
    print(row, flush=True)
    del G
    torch.cuda.empty_cache()
json.dump({"h": h, "kappa": kappa, "beta": beta, "k": k, "rows": rows},
          open(os.path.join(ROOT, "profiles", f"{R}_mass_comparison.json"), "w"), indent=1)
with open(os.path.join(ROOT, "profiles", f"{R}_mass_comparison.md"), "w") as f:
    f.write(f"# {R} lumped vs consistent mass on B200 (PAPER.md §4.3, Fig. 2; SURVEY §8f NEXT-3)\n\n")
    f.write("BA(n, 2), h = 2^-6, kappa = 1, beta = 0.75, L = 131; one sample per call. The consistent factor "
            "(natural-order Cholesky of M: per-edge chains + dense Cholesky of the vertex Schur complement, "
            "host) is built once per graph.\n\n")
    f.write("| n | N | consistent factor (s, once) | noise lumped ms | noise consistent ms | full lumped ms | "
            "full consistent ms | full ratio C/L |\n|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        f.write(f"| {r['n']} | {r['N']} | {r['factor_s']:.3f} | {r['noise_lumped_ms']:.3f} | "
                f"{r['noise_consistent_ms']:.3f} | {r['full_lumped_ms']:.2f} | {r['full_consistent_ms']:.2f} | "
                f"{r['full_consistent_ms'] / r['full_lumped_ms']:.2f} |\n")
print("written")
