"""NEXT-4: covariance-error study on B200 (§4.2, P337-338):
the covariance C_h = B_h M_L B_h (B_h = sum_l A_l^{-1}, from batched grf_apply on unit columns)
on coarse meshes h = 2^-3 .. 2^-6, upsampled (P C_h P^T) and compared with the overkill
covariance (h = 2^-8) in the lumped-mass L2(Gamma x Gamma) norm.  Graph: the config-1 tadpole;
kappa = 5, k = 0.2.  Theory: rate min(4 beta - 1/2, 2).

    python tools/covariance_study.py r01
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2605_02670_b200.study import covariance_error  # noqa: E402
from synth import tadpole  # noqa: E402

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
torch.cuda.set_device(0)
levels, ok = [3, 4, 5, 6], 8
rows = []
for beta in (0.3, 0.5, 0.75, 0.9):
    t0 = time.perf_counter()
    r = covariance_error(tadpole(), levels, ok, 5.0, beta, 0.2)
    r["seconds"] = time.perf_counter() - t0
    rows.append((beta, r))
    print(beta, r["rate"], r["theory_rate"], r["cov_err"], flush=True)
json.dump({"graph": "tadpole", "kappa": 5.0, "k": 0.2, "levels": levels, "ok_level": ok,
           "results": {str(b): r for b, r in rows}}, open(os.path.join(ROOT, "profiles", f"{R}_covariance_error.json"), "w"),
          indent=1)
with open(os.path.join(ROOT, "profiles", f"{R}_covariance_error.md"), "w") as f:
    f.write(f"# {R} covariance-error study on B200 (PAPER.md §4.2, P337-338; SURVEY §8f NEXT-4)\n\n")
    f.write("Config-1 tadpole graph, kappa = 5, k = 0.2; C_h = B_h M_L B_h from batched grf_apply on the "
            "identity columns; error ||C_ok - P C_h P^T|| in the overkill lumped-mass L2(Gamma x Gamma) norm, "
            f"overkill h = 2^-{ok}.  Theory: min(4 beta - 1/2, 2).\n\n")
    f.write("| beta | " + " | ".join(f"h=2^-{j}" for j in levels) + " | rate | theory | GPU s |\n")
    f.write("|---|" + "---|" * len(levels) + "---|---|---|\n")
    for b, r in rows:
        f.write(f"| {b} | " + " | ".join(f"{e:.4g}" for e in r["cov_err"]) +
                f" | {r['rate']:.3f} | {r['theory_rate']:.2f} | {r['seconds']:.1f} |\n")
print("written")
