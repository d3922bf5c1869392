"""Hot SASS instructions of an ncu source page exported with --print-source sass: the top
instructions by warp-stall samples with their dominant reasons, and the samples per region
(runs of consecutive instructions split at large sample gaps are not attempted: regions are
address ranges given on the command line as lo:hi hex offsets from the kernel start).
usage: python tools/ncu_sass_hot.py SRC.csv [ntop] [lo:hi ...]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ranges = [tuple(int(x, 16) for x in a.split(":")) for a in sys.argv[3:]]
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
ci = {c: hdr.index(c) for c in cols}
ins = []
base = None
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    a = int(r[0], 16)
    base = a if base is None else base
    s = int(r[2] or 0)
    st = {c: int(r[ci[c]] or 0) for c in cols}
    ins.append((a - base, r[1].strip(), s, st, int(r[5] or 0)))
tot = sum(x[2] for x in ins)
print(f"total samples {tot}, instructions {len(ins)}")
agg = {c: sum(x[3][c] for x in ins) for c in cols}
print("all:", ", ".join(f"{c[6:]} {100*v/tot:.1f}%" for c, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
for lo, hi in ranges:
    sub = [x for x in ins if lo <= x[0] < hi]
    t = sum(x[2] for x in sub)
    ag = {c: sum(x[3][c] for x in sub) for c in cols}
    print(f"[{lo:#x},{hi:#x}) {100*t/tot:.1f}% of samples:", ", ".join(f"{c[6:]} {100*v/max(t,1):.1f}%" for c, v in sorted(ag.items(), key=lambda q: -q[1])[:6]))
for off, txt, s, st, ex in sorted(ins, key=lambda x: -x[2])[:ntop]:
    top = sorted(st.items(), key=lambda t: -t[1])[:3]
    print(f"{100*s/tot:5.2f}% {off:#7x} {txt[:58]:58s} " + " ".join(f"{c[6:]}:{v}" for c, v in top if v))
