"""Write the round's ncu evidence into profiles/ (summaries only; the .ncu-rep stays in gpurun_out/).

    python tools/summarize_profiles.py r01 [config]
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

R = sys.argv[1]
CONFIG = sys.argv[2] if len(sys.argv) > 2 else "lattice256"
G = "gpurun_out"
P = "profiles"
os.makedirs(P, exist_ok=True)
import re

# kernel -> bench.py bracket name (bench times brackets: pcg = assemble + K4, recover = K5 + vertex sum)
def short(name):
    m = re.search(r"sweep_kernel<\s*\d+,\s*\d+,\s*\d+,\s*\d+,\s*(\d)", name)  # the REC argument
    if m:
        return "condense" if m.group(1) == "0" else "recover"
    m = re.search(r"sweep2_kernel<([^>]*)>", name)  # warp-specialised sweep: <TL, TS, REC>
    if m:
        rec = m.group(1).split(",")[-1].strip().replace("(bool)", "")
        return "condense" if rec in ("0", "false") else "recover"
    if "sweep3c_kernel" in name:  # warp-specialised condense (sweep3_impl.cuh)
        return "condense"
    if "sweep3_kernel" in name:  # warp-specialised recover (sweep3_impl.cuh)
        return "recover"
    for k, v in (("noise_kernel", "noise"), ("edge_setup_kernel", "edge_setup"), ("pcg_tables_pos_kernel", "pcg_tables_pos"),
                 ("pcg_tables_kernel", "pcg_tables"),
                 ("assemble_rhs_kernel", "assemble"), ("vertex_sum_kernel", "vertex_sum"),
                 ("pcg_warp_kernel", "pcg"), ("pcg_global_kernel", "pcg"), ("pcg_kernel", "pcg")):
        if k in name:
            return v
    return name[:40]


BRACKET = {"assemble": "pcg", "vertex_sum": "recover"}


for f in (f"{R}_bench.json", f"{R}_bench_ref.json", f"{R}_gpu.txt", f"{R}_host.txt"):
    if os.path.exists(os.path.join(G, f)):
        shutil.copy(os.path.join(G, f), os.path.join(P, f))

# ---- launch list: per-kernel totals (cold-cache, serialised: compare shares)
rows = []
with open(os.path.join(G, f"{R}_launches.csv")) as fh:
    lines = [l for l in fh if l.startswith('"')]
for rec in csv.DictReader(lines):
    if rec["Metric Name"] == "gpu__time_duration.sum":
        rows.append((short(rec["Kernel Name"]), float(rec["Metric Value"]) * (1e-3 if rec["Metric Unit"] == "ns" else 1)))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for k, us in rows:
    tot[k] += us
    cnt[k] += 1
step = [k for k in tot if k in ("noise", "condense", "assemble", "pcg", "recover", "vertex_sum")]
stot = sum(tot[k] for k in step)
bench = json.load(open(os.path.join(G, f"{R}_bench.json")))
with open(os.path.join(P, f"{R}_launches.md"), "w") as fh:
    fh.write(f"# {R} ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
    fh.write("Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py "
             "--steps 2 --warmup 1 --no-e2e --no-cpu-baseline` (config lattice256).  ncu times are cold-cache "
             "and serialised; the per-step SHARE is what must agree with bench.py's live CUDA-event timing.\n\n")
    fh.write("| kernel | launches | mean us (ncu) | share of step (ncu) | share of step (bench.py events) |\n|---|---|---|---|---|\n")
    for k in sorted(tot, key=lambda x: -tot[x]):
        sh = f"{tot[k] / stot:.3f}" if k in step else "setup (once per plan)"
        br = BRACKET.get(k, k)
        bsh = bench["kernels"].get(br, {}).get("share")
        note = "" if bsh is None else (f"{bsh:.3f}" if br == k else f"({br} bracket {bsh:.3f})")
        fh.write(f"| {k} | {cnt[k]} | {tot[k] / cnt[k]:.1f} | {sh} | {note} |\n")

# ---- full capture summary
raw = subprocess.run(["ncu", "-i", os.path.join(G, f"{R}_full.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(raw))
hdr = r[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size", "smsp__inst_executed.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]
units = r[1]
traffic = {}
with open(os.path.join(P, f"{R}_ncu_full.md"), "w") as fh:
    fh.write(f"# {R} ncu --set full summary (--clock-control none, one launch each)\n\n")
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        k = short(d["Kernel Name"])
        fh.write(f"## {k}\n\n`{d['Kernel Name'][:120]}`\n\n| metric | value | unit |\n|---|---|---|\n")
        for key in keys:
            if key in d:
                fh.write(f"| {key} | {d[key]} | {u.get(key, '')} |\n")
        st = [(float(d[x]), x) for x in hdr if x.startswith("smsp__pcsamp_warps_issue_stalled")
              and not x.endswith("not_issued") and d[x] not in ("", "n/a")]
        s_tot = sum(v for v, _ in st) or 1
        fh.write("\nTop stall reasons (PC sampling): " + ", ".join(
            f"{x.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / s_tot:.0f}%"
            for v, x in sorted(st, reverse=True)[:6]) + "\n\n")
        def tobytes(key):
            v = float(d[key].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(key, "byte"), 1)
            return v * scale
        traffic[k] = {"dram_bytes_per_launch": tobytes("dram__bytes_read.sum") + tobytes("dram__bytes_write.sum"),
                      "duration_ms": float(d["gpu__time_duration.sum"]) * (1e-6 if u["gpu__time_duration.sum"] == "ns" else 1e-3 if u["gpu__time_duration.sum"] == "us" else 1)}
# ---- config 4's global PCG (one launch), if captured
rgg = os.path.join(G, f"{R}_rgg_pcg.ncu-rep")
if os.path.exists(rgg):
    raw = subprocess.run(["ncu", "-i", rgg, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
    rr = list(csv.reader(raw))
    if len(rr) > 2:
        d = dict(zip(rr[0], rr[2]))
        u = dict(zip(rr[0], rr[1]))
        with open(os.path.join(P, f"{R}_ncu_rgg_pcg.md"), "w") as fh:
            fh.write(f"# {R} ncu --set full of config 4's global PCG (rgg, one launch, --clock-control none)\n\n"
                     f"`{d['Kernel Name'][:120]}`\n\n| metric | value | unit |\n|---|---|---|\n")
            for key in keys + ["lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sector_hit_rate.pct"]:
                if key in d:
                    fh.write(f"| {key} | {d[key]} | {u.get(key, '')} |\n")
            st = [(float(d[x]), x) for x in rr[0] if x.startswith("smsp__pcsamp_warps_issue_stalled")
                  and not x.endswith("not_issued") and d[x] not in ("", "n/a")]
            s_tot = sum(v for v, _ in st) or 1
            fh.write("\nTop stall reasons (PC sampling): " + ", ".join(
                f"{x.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / s_tot:.0f}%"
                for v, x in sorted(st, reverse=True)[:6]) + "\n")
json.dump({"round": R, "config": CONFIG, "kernels": traffic}, open(os.path.join(P, "traffic.json"), "w"), indent=1)
print(open(os.path.join(P, f"{R}_launches.md")).read())
print(json.dumps(traffic, indent=1))
