"""Stall samples aggregated by CUDA source line (and by reason) from an ncu source-page CSV
(--print-source cuda,sass).  usage: python tools/ncu_lines.py SRC.csv [ntop] [lo-hi line range]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
lo, hi = (map(int, sys.argv[3].split("-")) if len(sys.argv) > 3 else (0, 10 ** 9))
hdr = next(r for r in rows if r and r[0] == "Line No")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = {h: hdr.index(h) for h in reasons}
ia = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
cur = None
by_line = collections.defaultdict(lambda: collections.Counter())
src = {}
tot = collections.Counter()
for r in rows:
    if len(r) != len(hdr) or r[0] == "Line No":
        continue
    if r[0]:
        cur = (r[0], r[1].strip()[:80])
        continue
    if cur is None:
        continue
    ln = int(cur[0]) if cur[0].isdigit() else -1
    def f(x):
        try:
            return float(x or 0)
        except ValueError:
            return 0.0
    c = by_line[cur]
    c["all"] += f(r[ia])
    c["inst"] += f(r[ie])
    for h, i in ri.items():
        c[h] += f(r[i])
    if lo <= ln <= hi:
        tot["all"] += f(r[ia])
        for h, i in ri.items():
            tot[h] += f(r[i])
sel = [(c["all"], k, c) for k, c in by_line.items() if k[0].isdigit() and lo <= int(k[0]) <= hi]
sel.sort(reverse=True)
T = max(tot["all"], 1)
print("range total samples", int(T), " by reason:",
      ", ".join(f"{h[6:]} {100 * tot[h] / T:.0f}%" for h in sorted(reasons, key=lambda h: -tot[h])[:8]))
for a, k, c in sel[:ntop]:
    top = ", ".join(f"{h[6:]} {100 * c[h] / max(a, 1):.0f}%" for h in sorted(reasons, key=lambda h: -c[h])[:3])
    print(f"{100 * a / T:5.1f}% L{k[0]:>4} inst {c['inst']:.2e} {k[1]:80s} [{top}]")
