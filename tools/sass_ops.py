"""Per-kernel SASS opcode mix and (opcode, stall reason) shares from an ncu report's source page.

    python tools/sass_ops.py gpurun_out/x.ncu-rep [kernel-substring]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows, kern, hdr = {}, None, None
for rec in csv.reader(out):
    if rec and rec[0] == "Kernel Name":
        kern = rec[1]; rows[kern] = []; hdr = None; continue
    if rec and rec[0] == "Address":
        hdr = rec; continue
    if kern and hdr:
        rows[kern].append(dict(zip(hdr, rec)))
for k, rs in rows.items():
    if pat not in k:
        continue
    print("==", k[:110])
    byop, stalls, tot = collections.Counter(), collections.Counter(), 0
    for r in rs:
        ex = int(r["Instructions Executed"] or 0)
        src = r["Source"].split()
        if not src:
            continue
        op = (src[1] if src[0].startswith("@") else src[0]).split(".")[0]
        byop[op] += ex
        tot += ex
        for c in hdr:
            if c.startswith("stall_") and "Not Issued" not in c:
                stalls[(op, c[6:])] += int(r[c] or 0)
    print("  warp-instr", tot)
    print("  ops:", ", ".join(f"{op} {100*n/tot:.1f}%" for op, n in byop.most_common(12)))
    st = sum(stalls.values()) or 1
    print("  stalls:", ", ".join(f"{op}/{c} {100*n/st:.1f}%" for (op, c), n in stalls.most_common(12)))
