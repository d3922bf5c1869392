#!/usr/bin/env python
"""Benchmark of the fractional-SPDE GRF sampler hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config lattice256] [--edgepart] [--impl grf|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

A "step" is one sampling call over the whole workload of a BASELINE.json config: noise ->
condense -> vertex NN-PCG -> recovery + quadrature sum for every sample and every quadrature
node (the per-(kappa, beta, k) edge setup a3 is cached after the first
call, like model weights).  Default workload: configs[2] ("lattice256": 32x32 lattice,
N = 198 325 DOFs, L = 212 nodes, 256 samples) -- the throughput configuration the metric is
quoted on.  --config tadpole | lattice1 | lattice256 | rgg | star selects configs[0..4].

Multi-GPU (one process per GPU, policy BY_SAMPLE_THEN_NODE through the library's
grf_sample_dist): the config's samples are split over the ranks (P_s = min(N, S) contiguous
ranges) and the ranks sharing a sample range split the quadrature nodes round-robin, their
partial sums meeting on the range's root through NCCL -- the total work is fixed, so
"scaling": "strong".  --edgepart (config 4): every rank holds one edge part (recursive
coordinate bisection, grf_partition_edges / grf_graph_create_part) and the vertex NN-PCG runs
distributed (grf_sample_edgepart: neighbour halo send/recv + dot-product allreduce over NCCL).
Time = max over ranks of the CUDA-event time between barriers.  Latency-bound single-GPU
configs (tadpole, lattice1) replay the step as a captured CUDA graph (same seed each replay:
every replay recomputes everything).  Inputs far exceed the 126 MB L2 for lattice256 / rgg /
star (no flush needed); tadpole and lattice1 are L2-resident by nature.

--impl reference times the CPU oracle (oracle/, sparse LDL^T per node) on a bounded sample of
the same workload; it is the deliberately slow definition, not a competitor.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GRF samples/s & DOF×quad-node solves/s; achieved HBM GB/s vs B200 peak"
CONFIG_INDEX = {"tadpole": 0, "lattice1": 1, "lattice256": 2, "rgg": 3, "star": 4}
SMALL = ("tadpole", "lattice1")  # latency-bound: CUDA-graph replay, L2-resident


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="lattice256", choices=list(CONFIG_INDEX))
    ap.add_argument("--edgepart", action="store_true", help="config 4: edge-partitioned over the ranks")
    ap.add_argument("--no-graph", action="store_true", help="do not replay small configs as a CUDA graph")
    ap.add_argument("--impl", default="grf", choices=["grf", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
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


def config_dict(name, cfg, g, n_nodes, n_dofs, world, mode):
    """The same dict for both arms (the GPU arm takes L from grf_plan_info and N from the graph
    handle, the reference arm from the oracle: the numbers agree)."""
    return {"workload": f"{name} (BASELINE.json configs[{CONFIG_INDEX[name]}])", "graph": g.name,
            "n_vertices": int(g.n_vertices), "n_edges": int(g.n_edges), "n_dofs": int(n_dofs), "h": cfg["h"],
            "kappa": cfg["kappa"], "beta": cfg["beta"], "k": cfg["k"], "quad_nodes": int(n_nodes),
            "samples": cfg["n_samples"], "seed": cfg["seed"], "mode": mode,
            "l2": "small: L2-resident" if name in SMALL else "inputs larger than L2 (no flush)"}


# ------------------------------------------------------------------------------------ reference arm
def oracle_time(g, cfg, n_nodes, sample_index=0, prob=None):
    """The oracle (as it stands) on 1 sample x n_nodes quadrature nodes spread over the rule."""
    import numpy as np
    from oracle import noise, solve
    if prob is None:
        prob = solve.setup(g, cfg["h"], cfg["kappa"], cfg["beta"], cfg["k"])
    L = prob.plan.n_nodes
    picks = np.unique(np.linspace(0, L - 1, min(n_nodes, L)).round().astype(int))
    t0 = time.perf_counter()
    W = noise.white_noise(prob.ML, cfg["seed"], cfg["n_samples"], samples=[sample_index])
    for li in picks:
        solve.node_solve(prob, int(li), W)
    dt = time.perf_counter() - t0
    N = prob.mesh.n_dofs
    return dict(seconds=dt, nodes=len(picks), L=L, N=N, prob=prob,
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


def oracle_time_all_cores(name, n_nodes, L):
    """The same oracle over n_nodes quadrature nodes of one sample, spread over every host core
    (one process per core, each with its own setup -- the paper's OpenMP-over-l layout, P164)."""
    import concurrent.futures as cf
    import numpy as np
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
    prob = None
    for _ in range(max(0, args.warmup)):
        prob = oracle_time(g, cfg, args.ref_nodes, prob=prob)["prob"]
    ts = [oracle_time(g, cfg, args.ref_nodes, sample_index=i, prob=prob) for i in range(args.steps)]
    prob = ts[0]["prob"]
    tot = sum(t["seconds"] for t in ts)
    samples = sum(t["nodes"] / t["L"] for t in ts)
    value = samples / tot
    mode = "edgepart" if args.edgepart else "dist"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args.config, cfg, g, prob.plan.n_nodes, prob.mesh.n_dofs,
                                                   args.gpus, mode),
        "dof_node_per_s": sum(t["N"] * t["nodes"] for t in ts) / tot,
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": 1, "kind": "oracle",
                         "sample": f"per step: sample j, {ts[0]['nodes']} of {ts[0]['L']} quadrature nodes "
                                   f"(C sparse LDL^T per node, 1 thread); value = node-fraction of a sample per "
                                   f"second"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------ GPU arm
def algorithmic(kernel, n_interior, V, E, N, L, S, iters_mean):
    """Algorithmic work per launch: (amount, unit)."""
    if kernel == "recover":
        # Thomas forward (2 flop) + back substitution (3 flop) + sum over l (1 flop) per DOF.node.sample
        return 6.0 * n_interior * L * S, "flop"
    if kernel == "condense":
        # two one-sided forward eliminations (2 flop each) per interior DOF.node.sample
        return 4.0 * n_interior * L * S, "flop"
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
    from paper_2605_02670_b200 import Comm, Graph, plan_info, sample_edgepart
    from paper_2605_02670_b200.grf import dist_shard, make_options, sample_dist

    cfg, g = workload(args.config)
    S = cfg["n_samples"]
    kappa, beta, k, seed = cfg["kappa"], cfg["beta"], cfg["k"], cfg["seed"]
    km, kp, _, _ = plan_info(beta, k)
    L = km + kp + 1
    G = Graph.from_metric_graph(g, cfg["h"])
    n_dofs = G.n_dofs
    mode = "edgepart" if args.edgepart else "dist"
    comm = Comm() if world > 1 else None
    stream = torch.cuda.current_stream()
    graph_replay = None
    info = {}

    if mode == "edgepart":
        ep, pinfo = G.partition(world, xy=g.coords)
        info["partition"] = dict(pinfo, parts=world, method="RCB" if g.coords is not None else "BFS runs")
        part = Graph.part_of(G, ep, world, rank)
        work_graph = part
        n_local, sample_lo = S, 0
        outs = [torch.empty((S, part.n_dofs), dtype=torch.float64, device="cuda")]

        def step(stats=False):
            return sample_edgepart([part], kappa, beta, k, seed=seed, n_samples=S, comm=comm, return_stats=stats)
    else:
        (s0, s1), (l0, l1), root, active, is_root, pl = dist_shard(world, rank, S, L)
        info["shard"] = {"sample_range": [s0, s1], "node_begin": l0, "node_stride": pl, "ranks_per_range": pl}
        work_graph = G
        n_local, sample_lo = s1 - s0, s0
        out = torch.empty((max(n_local, 1), n_dofs), dtype=torch.float64, device="cuda")
        ws = torch.empty(G.workspace_size(kappa, beta, k, max(n_local, 1)), dtype=torch.uint8, device="cuda")

        def step(stats=False):
            if world == 1:
                return G.sample(kappa, beta, k, seed=seed, n_samples=S, out=out, workspace=ws, return_stats=stats)
            return sample_dist(G, comm, kappa, beta, k, seed=seed, n_samples=S, out=out, return_stats=stats)

    # cold-plan call: the first call for (kappa, beta, k) also builds the per-plan tables (K2)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    res = step(stats=True)
    c1.record(stream)
    torch.cuda.synchronize()
    cold_ms = c0.elapsed_time(c1)
    st = res[1] if isinstance(res, tuple) else {}
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if mode == "dist" and world == 1 and args.config in SMALL and not args.no_graph:
        graph_replay = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_replay):
            step()
        for _ in range(3):
            graph_replay.replay()
        torch.cuda.synchronize()
    work_graph.profile(True)
    work_graph.profile_read()

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
        if graph_replay is not None:
            graph_replay.replay()
        else:
            step()
        marks[i + 1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    per_step = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    prof = work_graph.profile_read()
    if graph_replay is not None:
        # the replays carry no profiling brackets (not captured): the per-kernel times for
        # `kernels` / `roofline` come from as many eager calls after the timed region
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        prof = work_graph.profile_read()
    work_graph.profile(False)
    if world > 1:
        t = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    launches_per_step = int(st.get("gpu_launches", 0))
    launches = launches_per_step * args.steps  # a replay launches the kernels of one call

    # end to end: the public API with the step's result read back to pinned host memory each step
    e2e = None
    if not args.no_e2e:
        host = None
        if mode == "edgepart":
            host = torch.empty((S, work_graph.n_dofs), dtype=torch.float64, pin_memory=True)

            def e2e_step():
                us = sample_edgepart([work_graph], kappa, beta, k, seed=seed, n_samples=S, comm=comm)
                host.copy_(us[0])
            d2h = S * work_graph.n_dofs * 8
        elif world == 1 or info["shard"]["ranks_per_range"] == 1:
            host = torch.empty((max(n_local, 1), n_dofs), dtype=torch.float64, pin_memory=True)

            def e2e_step():
                if n_local > 0:
                    G.sample_into_host(kappa, beta, k, seed + sample_lo, n_local, host)
            d2h = n_local * n_dofs * 8
        else:
            is_root = info["shard"]["node_begin"] == 0
            host = torch.empty((max(n_local, 1), n_dofs), dtype=torch.float64, pin_memory=True)

            def e2e_step():
                u, _, root_ = sample_dist(G, comm, kappa, beta, k, seed=seed, n_samples=S, out=out)
                if root_ and u is not None:
                    host.copy_(u)
            d2h = n_local * n_dofs * 8 if is_root else 0
        e2e_step()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        marks = []
        for _ in range(args.e2e_steps):
            e2e_step()  # returns after the result is in host memory (the call synchronises)
            marks.append(time.perf_counter())
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        per_step = [1e3 * (b - a) for a, b in zip([t0] + marks[:-1], marks)]
        if world > 1:
            t = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": S * args.e2e_steps / te, "unit": "samples/s", "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * te / args.e2e_steps,
               "step_ms": {"min": min(per_step), "median": sorted(per_step)[len(per_step) // 2],
                           "max": max(per_step)},
               "note": "the public call with the result copied to pinned host memory inside the timed region "
                       "(grf_sample_host / grf_sample_dist / grf_sample_edgepart + copy); per-step inputs are the "
                       "scalars (kappa, beta, k, seed) -- the noise is generated on the device from the seed"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    pk = peaks()
    step_s = t_ms / 1e3 / args.steps
    value = S / step_s
    dof_node = n_dofs * L * S / step_s
    wg = work_graph
    kernels = {}
    for name, (ms, n) in prof.items():
        if n == 0:
            continue
        amt, unit = algorithmic(name, wg.n_interior, wg.n_vertices, wg.n_edges, wg.n_dofs, L, n_local,
                                st.get("iter_mean", 0.0))
        per = ms / n
        kernels[name] = {"ms_per_launch": per, "launches": n, "share": ms / t_ms,
                         ("tflops" if unit == "flop" else "gbs"): (amt / (per / 1e3)) / (1e12 if unit == "flop" else 1e9)}
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config, cfg, g, L, n_dofs, world, mode),
        "dof_node_per_s": dof_node,
    }
    # how the step ran (kept out of `config`, which names the workload only and is the same dict
    # in the reference arm's line)
    line["run"] = {"cuda_graph": graph_replay is not None}
    if graph_replay is not None:
        line["kernels_timed"] = ("per-kernel times (kernels, roofline) from as many eager calls right after the "
                                 "timed graph replays; share = their time / the replays' time")
    line["run"].update(info)
    if kernels:
        dom = max((k_ for k_ in kernels if k_ != "noise"), key=lambda k_: kernels[k_]["share"], default=None)
        if dom is not None:
            amt, unit = algorithmic(dom, wg.n_interior, wg.n_vertices, wg.n_edges, wg.n_dofs, L, n_local,
                                    st.get("iter_mean", 0.0))
            ach = amt / (kernels[dom]["ms_per_launch"] / 1e3) / 1e12
            traffic = None
            tpath = os.path.join(ROOT, "profiles", "traffic.json")
            if os.path.exists(tpath):
                with open(tpath) as f:
                    tj = json.load(f)
                if tj.get("config") == args.config and dom in tj.get("kernels", {}):
                    traffic = tj["kernels"][dom].get("dram_bytes_per_launch")
            line["roofline"] = {"bound": "alu", "achieved": ach, "peak": pk["fp64_tflops"], "unit": "TFLOP/s",
                                "frac": ach / pk["fp64_tflops"], "traffic": traffic, "kernel": dom,
                                "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x sm_max_mhz "
                                               "(B200_PROFILING.md clocks)"}
            if dom in ("recover", "condense"):
                # what the fp64 pipe actually executes: 4 (K5) / 2 (K3) FMA per interior DOF, node slot
                # and sample over the padded node rows Lp (the correction node and the padding slots
                # included) -- the pipe efficiency, beside the algorithmic-work fraction above
                q0 = (L + 1 + 31) // 32
                r_ = (q0 + 6) // 7
                Lp = 32 * ((q0 + r_ - 1) // r_) * r_
                fma_per = 4.0 if dom == "recover" else 2.0
                ex = 2.0 * fma_per * wg.n_interior * Lp * n_local / (kernels[dom]["ms_per_launch"] / 1e3) / 1e12
                line["roofline"]["executed"] = {"tflops": ex, "frac": ex / pk["fp64_tflops"], "node_rows": Lp,
                                                "flop_per_dof_node_sample": 2.0 * fma_per}
            line["peaks"] = {"hbm_gbs": pk["hbm_gbs"], "fp64_tflops": pk["fp64_tflops"], "source": pk["source"],
                             "fp64_measured_tflops": pk["fp64_measured_tflops"],
                             "frac_of_measured_fp64": ach / pk["fp64_measured_tflops"]}
            if n_local <= 8 and dom in ("recover", "condense"):
                # 1-sample items: each item streams its edge's Thomas tables for all
                # Lp nodes (mu for K3, mu and g for K5) and no other item shares them -- the sweep is
                # bound by that HBM traffic, not by fp64
                q0 = (L + 1 + 31) // 32
                r_ = (q0 + 6) // 7
                Lp = 32 * ((q0 + r_ - 1) // r_) * r_
                ntab = 2 if dom == "recover" else 1
                byts = (ntab * 8.0 * Lp * wg.n_interior + 16.0 * wg.n_dofs) * n_local
                gbs = byts / (kernels[dom]["ms_per_launch"] / 1e3) / 1e9
                line["roofline_alu"] = line["roofline"]
                line["roofline"] = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                                    "frac": gbs / pk["hbm_gbs"], "traffic": traffic, "kernel": dom,
                                    "algorithmic_bytes": byts,
                                    "note": "Thomas-table rows (8 B x Lp per interior DOF and table) + W read + u "
                                            "write per sample; peak = MEASURED_PEAKS.json copy bandwidth"}
    # north_star's design-independent number: the per-(l,s) streaming formulation moves 32 B per
    # DOF.node; what bandwidth would it need to match this run?
    eff_hbm = 32.0 * dof_node / world / 1e9
    line["effective_streaming_hbm"] = {"gbs_per_gpu": eff_hbm, "frac_of_hbm_peak": eff_hbm / pk["hbm_gbs"],
                                       "note": "32 B/DOF.node of the per-(l,s) streaming form / measured time; "
                                               ">1 is possible because the fused kernels keep W and the sum on chip"}
    line["kernels"] = kernels
    line["pcg"] = {k_: st.get(k_) for k_ in ("iter_min", "iter_max", "iter_mean", "worst_rel_residual",
                                             "worst_true_rel_residual") if k_ in st}
    line["step_ms"] = {"median": statistics.median(per_step), "best": min(per_step), "worst": max(per_step),
                       "cold_plan_first_call": cold_ms}
    line["gpu_launches"] = launches
    line["clocks"] = clk
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        ob = oracle_time(g, cfg, args.cpu_nodes)
        line["cpu_baseline"] = {"value": ob["samples_per_s"], "unit": "samples/s", "cores": 1, "kind": "oracle",
                                "sample": f"sample 0, {ob['nodes']} of {ob['L']} quadrature nodes, "
                                          f"{ob['seconds']:.1f} s (C sparse LDL^T per node, 1 thread)",
                                "dof_node_per_s": ob["dof_node_per_s"]}
        try:
            oa = oracle_time_all_cores(args.config, args.cpu_nodes_all, L)
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
