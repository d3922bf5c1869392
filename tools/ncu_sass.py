"""Aggregate ncu --page source (SASS) per kernel: executed instructions by opcode, top stall PCs."""
import collections, csv, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
kern, rows, hdr = None, {}, None
for line in out:
    if line.startswith('"Kernel Name"'):
        kern = next(csv.reader([line]))[1]; rows[kern] = []; hdr = None; continue
    rec = next(csv.reader([line]))
    if rec and rec[0] == "Address":
        hdr = rec; continue
    if kern and hdr:
        rows[kern].append(dict(zip(hdr, rec)))
for k, rs in rows.items():
    if pat not in k:
        continue
    print("==", k)
    byop = collections.Counter(); stall = []
    tot = 0
    for r in rs:
        ex = int(r.get("Instructions Executed", "0") or 0)
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        byop[op.split(".")[0]] += ex; tot += ex
        stall.append((int(r.get("Warp Stall Sampling (All Samples)", "0") or 0), r["Address"][-5:], r["Source"].strip()[:70], ex))
    print("total warp-instr", tot)
    for op, n in byop.most_common(18):
        print(f"   {op:10s} {n:14d} {100*n/tot:5.1f}%")
    print(" top stall PCs:")
    st = sum(s for s, *_ in stall) or 1
    for s, a, src, ex in sorted(stall, reverse=True)[:25]:
        print(f"   {100*s/st:5.1f}% {a} {src:70s} ex={ex}")


def per_pc_reasons(rep, pat, top=30):
    """Print the top-stall PCs with their dominant stall reasons."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    kern, hdr, rows = None, None, []
    for line in out:
        if line.startswith('"Kernel Name"'):
            kern = next(csv.reader([line]))[1]; hdr = None; continue
        rec = next(csv.reader([line]))
        if rec and rec[0] == "Address":
            hdr = rec; continue
        if kern and hdr and pat in kern:
            rows.append(dict(zip(hdr, rec)))
    reasons = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows) or 1
    agg = collections.Counter()
    for r in rows:
        for h in reasons:
            agg[h] += int(r.get(h) or 0)
    print("stall reasons:", ", ".join(f"{h[6:]} {100*v/tot:.1f}%" for h, v in agg.most_common(8)))
    rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in rows[:top]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        rs = sorted(((int(r.get(h) or 0), h[6:]) for h in reasons), reverse=True)[:3]
        print(f"  {100*s/tot:5.1f}% {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in rs if v))


if len(sys.argv) > 3 and sys.argv[3] == "pc":
    per_pc_reasons(rep, pat)
