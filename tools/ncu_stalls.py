"""Summarise an ncu source page (SASS): stall reasons overall and the top instructions.
usage: ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv; python tools/ncu_stalls.py src.csv [lo hi]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
ia, isrc, iss, iex = h.index('Address'), h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
st = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
f = lambda x: float(x or 0)
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, len(data))
sel = data[lo:hi]
tot = sum(f(r[iss]) for r in sel)
print(f"samples {tot:.0f} over instructions {lo}..{hi}")
agg = {h[i]: sum(f(r[i]) for r in sel) for i in st}
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {k:24s} {v / max(tot, 1) * 100:5.1f}%")
print("top instructions:")
for r in sorted(sel, key=lambda r: -f(r[iss]))[:int(sys.argv[4]) if len(sys.argv) > 4 else 30]:
    i = data.index(r)
    why = sorted(((h[j], f(r[j])) for j in st), key=lambda kv: -kv[1])[:2]
    print(f"{i:5d} {f(r[iss]) / max(tot, 1) * 100:5.1f}% ex={r[iex]:>8} {r[isrc].strip()[:60]:60s} {why[0][0]}:{why[0][1]:.0f} {why[1][0]}:{why[1][1]:.0f}")
