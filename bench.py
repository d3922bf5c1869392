#!/usr/bin/env python
"""Benchmark of the fractional-SPDE GRF sampler hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config lattice256] [--impl grf|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

A "step" is one grf_sample call over the whole workload: noise -> condense -> vertex
NN-PCG -> recovery + quadrature sum for every sample and every quadrature node
(the per-(kappa,beta,k) edge setup a3 is cached after the
first call, like model weights).  Default workload: BASELINE.json configs[2]
("lattice256": 32x32 lattice, N = 198325 DOFs, L = 212 nodes, 256 samples) -- the
throughput configuration the metric is quoted on and the one sharded over 1/2/4/8 GPUs.
Multi-GPU: one process per GPU; each rank draws its own 256 samples (seeds rank*256 + j),
no data-path collective -> "scaling": "weak".  Time = max over ranks of CUDA-event time
between barriers.  Inputs (W/u 406 MB, plan tables 333 MB, vertex buffers 445 MB) are
far larger than the 126 MB L2, so no explicit L2 flush is needed.

--impl reference times the CPU oracle (oracle/, scipy sparse LU per node) on a bounded
sample of the same workload; it is the deliberately slow definition, not a competitor.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GRF samples/s & DOF×quad-node solves/s; achieved HBM GB/s vs B200 peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="lattice256")
    ap.add_argument("--impl", default="grf", choices=["grf", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-nodes", type=int, default=12, help="oracle sample: quadrature nodes of 1 sample")
    ap.add_argument("--ref-nodes", type=int, default=12, help="--impl reference: nodes per step")
    ap.add_argument("--cpu-nodes-all", type=int, default=64, help="all-cores oracle sample: nodes of 1 sample")
    return ap.parse_args()


def peaks():
    p = {"hbm_gbs": None, "sm_max_mhz": 1965.0, "source": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p.update(hbm_gbs=m.get("hbm_gbs"), sm_max_mhz=m.get("sm_max_mhz", 1965.0), source="measured")
    if p["hbm_gbs"] is None:
        p["hbm_gbs"] = 6650.0  # B200_PROFILING.md fallback
    # fp64 vector peak derived from unit counts and clock:
    # 148 SMs x 64 FP64 FMA/clk/SM x 2 flop x sm_max_mhz
    p["fp64_tflops"] = 148 * 64 * 2 * p["sm_max_mhz"] * 1e6 / 1e12
    # measured fp64 FMA throughput of tools/fp64_peak.cu on this pool's B200 (profiles/fp64_peak.txt)
    p["fp64_measured_tflops"] = 33.56
    return p


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.index), "-lms", "50"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out, _ = self.p.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload(name):
    from synth import CONFIGS, config_graph
    cfg = dict(CONFIGS[name])
    return cfg, config_graph(name)


def oracle_time(g, cfg, n_nodes, sample_index=0):
    """Time the oracle (as it stands) on 1 sample x n_nodes quadrature nodes spread over the rule."""
    import numpy as np
    from oracle import noise, solve
    prob = solve.setup(g, cfg["h"], cfg["kappa"], cfg["beta"], cfg["k"])
    L = prob.plan.n_nodes
    picks = np.unique(np.linspace(0, L - 1, min(n_nodes, L)).round().astype(int))
    t0 = time.perf_counter()
    W = noise.white_noise(prob.ML, cfg["seed"], cfg["n_samples"], samples=[sample_index])
    for li in picks:
        solve.node_solve(prob, int(li), W)
    dt = time.perf_counter() - t0
    N = prob.mesh.n_dofs
    return dict(seconds=dt, nodes=len(picks), L=L, N=N,
                samples_per_s=(len(picks) / L) / dt, dof_node_per_s=N * len(picks) / dt)


def _oracle_nodes(payload):
    """Worker: the oracle (as it stands) on a subset of quadrature nodes of one sample."""
    name, nodes = payload
    from oracle import noise, solve
    cfg, g = workload(name)
    prob = solve.setup(g, cfg["h"], cfg["kappa"], cfg["beta"], cfg["k"])
    W = noise.white_noise(prob.ML, cfg["seed"], cfg["n_samples"], samples=[0])
    for li in nodes:
        solve.node_solve(prob, int(li), W)
    return len(nodes)


def oracle_time_all_cores(name, n_nodes):
    """The same oracle over n_nodes quadrature nodes of one sample, spread over every host core
    (one process per core, each with its own setup -- the paper's OpenMP-over-l layout, P164)."""
    import concurrent.futures as cf
    import numpy as np
    from oracle.quadrature import limits
    cfg, _ = workload(name)
    km, kp = limits(cfg["beta"], cfg["k"])
    L = km + kp + 1
    cores = os.cpu_count() or 1
    picks = np.unique(np.linspace(0, L - 1, min(n_nodes, L)).round().astype(int))
    chunks = [picks[i::cores] for i in range(cores) if len(picks[i::cores])]
    t0 = time.perf_counter()
    with cf.ProcessPoolExecutor(max_workers=len(chunks)) as ex:
        done = sum(ex.map(_oracle_nodes, [(name, c) for c in chunks]))
    dt = time.perf_counter() - t0
    return dict(seconds=dt, nodes=done, L=L, cores=len(chunks), samples_per_s=(done / L) / dt)


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    cfg, g = workload(args.config)
    for _ in range(max(0, args.warmup)):
        oracle_time(g, cfg, args.ref_nodes)
    ts = [oracle_time(g, cfg, args.ref_nodes, sample_index=i) for i in range(args.steps)]
    tot = sum(t["seconds"] for t in ts)
    samples = sum(t["nodes"] / t["L"] for t in ts)
    value = samples / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args.config, cfg, g, None),
        "dof_node_per_s": sum(t["N"] * t["nodes"] for t in ts) / tot,
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": 1, "kind": "oracle",
                         "sample": f"per step: sample j, {ts[0]['nodes']} of {ts[0]['L']} quadrature nodes "
                                   f"(scipy SuperLU per node); value = node-fraction of a sample per second"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(name, cfg, g, G):
    from oracle.quadrature import limits
    km, kp = limits(cfg["beta"], cfg["k"])
    d = {"workload": f"{name} (BASELINE.json configs[{['tadpole', 'lattice1', 'lattice256', 'rgg', 'star'].index(name)}])",
         "graph": g.name, "n_vertices": int(g.n_vertices), "n_edges": int(g.n_edges),
         "h": cfg["h"], "kappa": cfg["kappa"], "beta": cfg["beta"], "k": cfg["k"],
         "quad_nodes": km + kp + 1, "samples_per_rank": cfg["n_samples"],
         "l2": "inputs larger than L2 (no flush)" if name in ("lattice256", "rgg", "star") else "small: L2-resident"}
    if G is not None:
        d["n_dofs"] = G.n_dofs
    return d


def algorithmic(kernel, G, L, S, iters_mean):
    """Algorithmic work per launch: (amount, unit)."""
    NI, V, E, N = G.n_interior, G.n_vertices, G.n_edges, G.n_dofs
    if kernel == "recover":
        # Thomas forward (2 flop) + back substitution (3 flop) + sum over l (1 flop) per DOF.node.sample
        return 6.0 * NI * L * S, "flop"
    if kernel == "condense":
        # two one-sided forward eliminations (2 flop each) per interior DOF.node.sample
        return 4.0 * NI * L * S, "flop"
    if kernel == "pcg":
        # per iteration: Schur SpMV 4 flop + NN precond 6 flop per incidence (2E), 6 vector ops (2 flop) per vertex
        return (iters_mean * (20.0 * E + 12.0 * V) + 12.0 * V) * L * S, "flop"
    if kernel == "noise":
        return 8.0 * N * S, "bytes"  # one fp64 write per DOF.sample
    return 0.0, "flop"


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2605_02670_b200 import Graph

    cfg, g = workload(args.config)
    G = Graph.from_metric_graph(g, cfg["h"])
    S = cfg["n_samples"]
    kappa, beta, k = cfg["kappa"], cfg["beta"], cfg["k"]
    seed = cfg["seed"] + rank * S
    out = torch.empty((S, G.n_dofs), dtype=torch.float64, device="cuda")
    ws = torch.empty(G.workspace_size(kappa, beta, k, S), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    # cold-plan call: the first call for (kappa, beta, k) also builds the per-plan tables (K2)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    _, st = G.sample(kappa, beta, k, seed=seed, n_samples=S, out=out, workspace=ws, return_stats=True)
    c1.record(stream)
    torch.cuda.synchronize()
    cold_ms = c0.elapsed_time(c1)
    L = st["n_nodes"]
    for _ in range(args.warmup):
        G.sample(kappa, beta, k, seed=seed, n_samples=S, out=out, workspace=ws)
    torch.cuda.synchronize()
    G.profile(True)
    G.profile_read()

    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.15)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record(stream)
    marks[0].record(stream)
    for i in range(args.steps):
        G.sample(kappa, beta, k, seed=seed, n_samples=S, out=out, workspace=ws)
        marks[i + 1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    per_step = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    prof = G.profile_read()
    G.profile(False)
    if world > 1:
        t = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    # kernels launched inside the timed region: the library's own per-call count (stats) x steps
    launches = int(st["gpu_launches"]) * args.steps

    # end to end: the same call with a pinned HOST output (D2H + sync inside the timed region)
    e2e = None
    if not args.no_e2e:
        host = torch.empty((S, G.n_dofs), dtype=torch.float64, pin_memory=True)
        G.sample_into_host(kappa, beta, k, seed, S, host)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            G.sample_into_host(kappa, beta, k, seed, S, host)
        te = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": world * S * args.e2e_steps / te, "unit": "samples/s", "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": int(S * G.n_dofs * 8), "ms_per_step": 1e3 * te / args.e2e_steps,
               "note": "grf_sample_host into pinned host memory; per-step inputs are the scalars "
                       "(kappa, beta, k, seed) -- the noise is generated on the device from the seed"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    pk = peaks()
    step_s = t_ms / 1e3 / args.steps
    value = world * S / step_s
    dof_node = world * G.n_dofs * L * S / step_s
    kernels = {}
    for name, (ms, n) in prof.items():
        if n == 0:
            continue
        amt, unit = algorithmic(name, G, L, S, st["iter_mean"])
        per = ms / n
        kernels[name] = {"ms_per_launch": per, "launches": n, "share": ms / t_ms,
                         ("tflops" if unit == "flop" else "gbs"): (amt / (per / 1e3)) / (1e12 if unit == "flop" else 1e9)}
    dom = max((k_ for k_ in kernels if k_ != "noise"), key=lambda k_: kernels[k_]["share"])
    amt, unit = algorithmic(dom, G, L, S, st["iter_mean"])
    ach = amt / (kernels[dom]["ms_per_launch"] / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        if tj.get("config") == args.config and dom in tj.get("kernels", {}):
            traffic = tj["kernels"][dom].get("dram_bytes_per_launch")
    roofline = {"bound": "alu", "achieved": ach, "peak": pk["fp64_tflops"], "unit": "TFLOP/s",
                "frac": ach / pk["fp64_tflops"], "traffic": traffic, "kernel": dom,
                "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x sm_max_mhz (B200_PROFILING.md clocks)"}
    # north_star's design-independent number: the per-(l,s) streaming formulation moves
    # 32 B per DOF.node; what bandwidth would it need to match this run?
    eff_hbm = 32.0 * dof_node / world / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(args.config, cfg, g, G),
        "dof_node_per_s": dof_node,
        "effective_streaming_hbm": {"gbs_per_gpu": eff_hbm, "frac_of_hbm_peak": eff_hbm / pk["hbm_gbs"],
                                    "note": "32 B/DOF.node of the per-(l,s) streaming form / measured time; "
                                            ">1 is possible because the fused kernels keep W and the sum on chip"},
        "roofline": roofline, "kernels": kernels,
        "pcg": {"iter_min": st["iter_min"], "iter_max": st["iter_max"], "iter_mean": st["iter_mean"],
                "worst_rel_residual": st["worst_rel_residual"]},
        "step_ms": {"median": statistics.median(per_step), "best": min(per_step), "worst": max(per_step),
                    "cold_plan_first_call": cold_ms},
        "gpu_launches": launches, "clocks": clk,
        "peaks": {"hbm_gbs": pk["hbm_gbs"], "fp64_tflops": pk["fp64_tflops"], "source": pk["source"],
                  "fp64_measured_tflops": pk["fp64_measured_tflops"],
                  "frac_of_measured_fp64": ach / pk["fp64_measured_tflops"]},
    }
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        ob = oracle_time(g, cfg, args.cpu_nodes)
        line["cpu_baseline"] = {"value": ob["samples_per_s"], "unit": "samples/s", "cores": 1, "kind": "oracle",
                                "sample": f"sample 0, {ob['nodes']} of {ob['L']} quadrature nodes, "
                                          f"{ob['seconds']:.1f} s (scipy SuperLU per node, 1 thread)",
                                "dof_node_per_s": ob["dof_node_per_s"]}
        try:
            oa = oracle_time_all_cores(args.config, args.cpu_nodes_all)
            line["cpu_baseline"]["all_cores"] = {
                "value": oa["samples_per_s"], "cores": oa["cores"],
                "sample": f"sample 0, {oa['nodes']} of {oa['L']} nodes over {oa['cores']} processes "
                          f"(one per core, each with its own setup), {oa['seconds']:.1f} s"}
        except Exception as e:  # the single-thread figure above is the reported baseline
            line["cpu_baseline"]["all_cores"] = {"error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
