"""Config 5 as a convergence study: star of 8 unit 16x16 lattices, kappa = 8,
k = 0.2, beta in {0.3, 0.5, 0.75, 0.9}, overkill h = 2^-12, coarse h = 2^-4 .. 2^-9, 64 noise
realizations on the overkill mesh.  Writes profiles/<round>_strong_error.{json,md}.

    python tools/strong_error_study.py r01 [--samples 64] [--levels 4 5 6 7 8 9]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("round")
ap.add_argument("--samples", type=int, default=64)
ap.add_argument("--levels", type=int, nargs="+", default=[4, 5, 6, 7, 8, 9])
ap.add_argument("--ok", type=int, default=12)
ap.add_argument("--betas", type=float, nargs="+", default=[0.3, 0.5, 0.75, 0.9])
a = ap.parse_args()

import torch  # noqa: E402

from paper_2605_02670_b200.study import strong_error  # noqa: E402
from synth import star_of_lattices  # noqa: E402

torch.cuda.set_device(0)
g = star_of_lattices(8, 16)
out = {"graph": g.name, "kappa": 8.0, "k": 0.2, "ok_level": a.ok, "levels": a.levels, "n_samples": a.samples,
       "results": {}}
rows = []
for beta in a.betas:
    t0 = time.perf_counter()
    r = strong_error(g, a.levels, a.ok, 8.0, beta, 0.2, seed=0, n_samples=a.samples, batch=32)
    dt = time.perf_counter() - t0
    r.pop("per_sample_sq")
    r["seconds"] = dt
    out["results"][str(beta)] = r
    rows.append((beta, r))
    print(beta, r["rate_rms"], r["theory_rate_rms"], r["rms_err"], f"{dt:.1f}s", flush=True)
with open(os.path.join(ROOT, "profiles", f"{a.round}_strong_error.json"), "w") as f:
    json.dump(out, f, indent=1)
with open(os.path.join(ROOT, "profiles", f"{a.round}_strong_error.md"), "w") as f:
    f.write(f"# {a.round} strong-error study on B200 (config 5 as a convergence study, PAPER.md §4.1 P332-335)\n\n")
    f.write(f"Graph `{g.name}` (2049 vertices, 3848 unit edges), kappa = 8, k = 0.2 (fixed), overkill "
            f"h = 2^-{a.ok}, {a.samples} noise realizations drawn on the overkill mesh and projected down "
            "(grf_project_noise = P^T), coarse solutions upsampled (grf_prolong = P), error in the overkill "
            "lumped-mass norm (grf_mnorm_sq_diff); RMS = sqrt(mean squared error) (SURVEY §8c Q13). "
            "Rates: OLS of ln RMS on ln h. Theory 2 beta - 1/2 (P334).\n\n")
    f.write("| beta | " + " | ".join(f"RMS h=2^-{j}" for j in a.levels) + " | rate (RMS) | theory | GPU s |\n")
    f.write("|---|" + "---|" * len(a.levels) + "---|---|---|\n")
    for beta, r in rows:
        f.write(f"| {beta} | " + " | ".join(f"{e:.4g}" for e in r["rms_err"]) +
                f" | {r['rate_rms']:.3f} | {r['theory_rate_rms']:.2f} | {r['seconds']:.1f} |\n")
print("written")
