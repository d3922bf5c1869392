"""Summarise an ncu report's SASS source page: stall and instruction shares by opcode + top stall sites.
usage: python tools/ncu_ops.py REPORT.ncu-rep [kernel-substring] [ntop]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
for b in blocks:
    if sub not in b["name"]:
        continue
    print("==", b["name"][:100])
    hdr = b["rows"][0]
    data = [r for r in b["rows"][1:] if len(r) == len(hdr)]
    ia, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    tot = sum(float(r[ia] or 0) for r in data)
    ti = sum(float(r[ie] or 0) for r in data)
    byop, byopi = collections.Counter(), collections.Counter()
    for r in data:
        toks = r[1].split()
        op = toks[0] if toks else "?"
        if op.startswith("@"):
            op = toks[1]
        op = op.split(".")[0]
        byop[op] += float(r[ia] or 0)
        byopi[op] += float(r[ie] or 0)
    print(" instructions executed:", int(ti))
    print(" stall% by op:", [(k, round(100 * v / tot, 1)) for k, v in byop.most_common(14)])
    print(" inst% by op:", [(k, round(100 * v / ti, 1)) for k, v in byopi.most_common(14)])
    for r in sorted(data, key=lambda r: -float(r[ia] or 0))[:ntop]:
        print("   ", round(100 * float(r[ia]) / tot, 1), r[0][-5:], r[1][:90])
