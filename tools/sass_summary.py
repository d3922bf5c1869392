"""Static SASS summary of the hot kernels in the built libgrf.so objects: instruction counts of
the opcodes that prove the design (DFMA, bulk copies UBLKCP, mbarrier SYNCS, LDS/STS, shuffles,
local-memory spills LDL/STL) and ptxas register counts.  Writes profiles/<tag>_sass.md.
usage: python tools/sass_summary.py TAG"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2605_02670_b200", "lib", "obj")
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
KERNELS = [  # (object, mangled-name regex, label)
    ("sweep3_r32.cu.o", r"sweep3_kernelILi7ELi3ELi2E", "K5 recover sweep3_kernel<TL=7, NST=3, CL=2> (config 3)"),
    ("sweep3_c32.cu.o", r"sweep3c_kernelILi7ELi28ELi3E", "K3 condense sweep3c_kernel<TL=7, IBK=28, NST=3> (config 3)"),
    ("pcg_warp.cu.o", r"pcg_warp_kernelILi16ELi4ELb1ELi2E", "K4 pcg_warp_kernel<VPL=16, W=4, staged, WPS=2> (config 3)"),
    ("pcg_global.cu.o", r"pcg_global_kernelILi16E", "K4 pcg_global_kernel<CS=16> (config 4)"),
    ("noise.cu.o", r"noise_kernel", "K1 noise_kernel"),
]
OPS = ["DFMA", "DMUL", "DADD", "UBLKCP", "SYNCS", "LDS", "STS", "LDG", "STG", "SHFL", "LDL", "STL", "BAR"]
out = [f"# {tag} static SASS summary (cuobjdump -sass of the built objects, sm_100a)\n",
       "Counts are static instructions in the kernel body (not executed counts); UBLKCP = bulk copy "
       "(cp.async.bulk), SYNCS = mbarrier operations, LDL/STL = local-memory spills.\n",
       "| kernel | " + " | ".join(OPS) + " | total |", "|---|" + "---|" * (len(OPS) + 1)]
for obj, rx, label in KERNELS:
    path = os.path.join(OBJ, obj)
    if not os.path.exists(path):
        continue
    names = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    fn = None
    for m in re.finditer(r"Function : (\S+)", names):
        if re.search(rx, m.group(1)):
            fn = m.group(1)
            break
    if fn is None:
        continue
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, path], capture_output=True, text=True).stdout
    cnt, tot = collections.Counter(), 0
    for line in sass.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if not m:
            continue
        tot += 1
        op = m.group(1)
        for k in OPS:
            if op.startswith(k):
                cnt[k] += 1
    out.append(f"| {label} | " + " | ".join(str(cnt[k]) for k in OPS) + f" | {tot} |")
open(os.path.join(ROOT, "profiles", f"{tag}_sass.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
