"""Config-4 edge partitions from the library (grf_partition_edges): interface vertices and DOF
balance for 2 / 4 / 8 parts, coordinate bisection vs breadth-first runs -> profiles/<tag>_partition.json.
usage (GPU box): python tools/partition_report.py r02"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_02670_b200 import Graph  # noqa: E402
from synth import CONFIGS, config_graph  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
torch.cuda.set_device(0)
cfg = CONFIGS["rgg"]
g = config_graph("rgg")
G = Graph.from_metric_graph(g, cfg["h"])
out = {"config": "rgg (configs[3])", "n_vertices": g.n_vertices, "n_edges": g.n_edges, "n_dofs": G.n_dofs,
       "partitions": []}
for P in (2, 4, 8):
    for method, xy in (("RCB", g.coords), ("BFS runs", None)):
        ep, info = G.partition(P, xy=xy)
        counts = [int((ep == q).sum()) for q in range(P)]
        total = G.n_interior + g.n_edges  # sum of the DOF weights n_e
        out["partitions"].append(dict(parts=P, method=method, edges_per_part=counts, **info,
                                      weight_imbalance=info["max_part_weight"] * P / total))
        print(P, method, info, flush=True)
os.makedirs("gpurun_out", exist_ok=True)  # copied into profiles/ by hand (gpurun returns gpurun_out/ only)
json.dump(out, open(f"gpurun_out/{tag}_partition.json", "w"), indent=1)
