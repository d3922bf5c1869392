"""Design study: device time of grf_sample on config 3 for chunk sizes (the grf_sample_host
pipeline's building block) and of the public host call.  usage: python tools/chunk_study.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import CONFIGS, config_graph
from paper_2605_02670_b200.grf import Graph

cfg = CONFIGS["lattice256"]
g = config_graph("lattice256")
G = Graph.from_metric_graph(g, cfg["h"])
kap, beta, k = cfg["kappa"], cfg["beta"], cfg["k"]
outs = {n: torch.empty((n, G.n_dofs), dtype=torch.float64, device="cuda") for n in (16, 32, 48, 64, 96, 128, 256)}
for n, o in outs.items():
    G.sample(kap, beta, k, seed=0, n_samples=n, out=o)
torch.cuda.synchronize()
for n, o in outs.items():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        G.sample(kap, beta, k, seed=0, n_samples=n, out=o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"chunk {n:4d}: {ms:7.3f} ms  {1e3 * ms / n:6.2f} us/sample")
host = torch.empty((256, G.n_dofs), dtype=torch.float64, pin_memory=True)
G.sample_into_host(kap, beta, k, 0, 256, host)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    G.sample_into_host(kap, beta, k, 0, 256, host)
torch.cuda.synchronize()
print(f"sample_into_host 256: {1e3 * (time.perf_counter() - t) / 5:.3f} ms")

# the same pipeline written out with the public device call: chunks on the compute stream, each
# chunk's copy on a side stream (two staging buffers), to see what the host call could reach
sizes = [64, 64, 64, 32, 32]
bufs = [torch.empty((64, G.n_dofs), dtype=torch.float64, device="cuda") for _ in range(2)]
cs = torch.cuda.Stream()
main = torch.cuda.current_stream()
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ev = []
    c0 = 0
    copied = [None, None]
    marks = []
    for c, n in enumerate(sizes):
        b = c & 1
        if copied[b] is not None:
            main.wait_event(copied[b])
        G.sample(kap, beta, k, seed=c0, n_samples=n, out=bufs[b][:n])
        e = torch.cuda.Event(enable_timing=True)
        e.record(main)
        marks.append(e)
        cs.wait_event(e)
        with torch.cuda.stream(cs):
            host[c0:c0 + n].copy_(bufs[b][:n], non_blocking=True)
            ce = torch.cuda.Event(enable_timing=True)
            ce.record(cs)
        copied[b] = ce
        c0 += n
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"python pipeline {sizes}: {1e3 * dt:.3f} ms; compute marks (ms from first):",
      [round(marks[0].elapsed_time(m), 2) for m in marks], "last copy end:", round(marks[0].elapsed_time(copied[(len(sizes) - 1) & 1]), 2))
