"""Top SASS sites of one stall reason from an ncu source-page CSV (--print-source cuda,sass), with the
CUDA source line each falls under.  usage: python tools/ncu_stall.py SRC.csv REASON [ntop]
(REASON: a column name such as stall_long_sb, stall_wait, stall_barrier)"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
reason = sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 15
hdr = next(r for r in rows if r and r[0] == "Line No")
ci = hdr.index(reason)
cur, sites, tot = None, [], 0.0
for r in rows:
    if len(r) != len(hdr) or r[0] == "Line No":
        continue
    if r[0]:
        cur = (r[0], r[1].strip()[:90])
        continue
    try:
        v = float(r[ci] or 0)
    except ValueError:
        continue
    tot += v
    sites.append((v, r[2], r[3].strip()[:60], cur))
sites.sort(reverse=True)
print(f"{reason}: {tot:.0f} samples")
for v, a, s, c in sites[:ntop]:
    print(f"{100 * v / max(tot, 1):5.1f}% {a[-5:]} {s:60s} <- {c}")
