"""Small driver for profiling the global-memory PCG (ncu): a 20k-vertex RGG, 16 samples."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2605_02670_b200 import Graph  # noqa: E402
from synth import rgg_knn  # noqa: E402
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
g = rgg_knn(n, k=3, scale=300.0 * (n / 100_000) ** 0.5, seed=1)
G = Graph.from_metric_graph(g, 0.005)
for _ in range(2):
    u, st = G.sample(2.0, 0.55, 0.3, seed=0, n_samples=16, return_stats=True)
torch.cuda.synchronize()
print(G.n_dofs, st)
