import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr = r[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__block_size",
        "launch__grid_size", "l1tex__t_bytes.sum"]
for row in r[2:]:
    d = dict(zip(hdr, row))
    print(d["Kernel Name"][:60])
    for k in keys:
        if k in d:
            print("   ", k, d[k])
    st = [(float(d[k]), k) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and d[k] not in ("", "n/a")]
    tot = sum(v for v, _ in st) or 1
    for v, k in sorted(st, reverse=True)[:7]:
        print("      stall", k.replace("smsp__pcsamp_warps_issue_stalled_", ""), f"{100*v/tot:.1f}%")
