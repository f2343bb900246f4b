"""Top stall-sampled SASS instructions of one kernel (ncu source page CSV with --print-source sass):
python tools/ncu_top_stalls.py <csv> [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = next(i for i, r in enumerate(rows) if 'Address' in r and 'Source' in r)
hdr, body = rows[hi], rows[hi + 1:]
ia, isrc, iex, ist = (hdr.index(k) for k in ("Address", "Source", "Instructions Executed", "Warp Stall Sampling (All Samples)"))
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
body = [r for r in body if len(r) > iex and r[iex].replace('.', '').isdigit()]
first = body[0][ia]
dup = [i for i, r in enumerate(body) if r[ia] == first]
b = body[:dup[1]] if len(dup) > 1 else body
tot = sum(float(r[ist] or 0) for r in b)
agg = {}
for r in b:
    for j, h in stall_cols:
        agg[h] = agg.get(h, 0) + float(r[j] or 0)
print("stall samples by reason:", ", ".join(f"{k[6:]}={100 * v / tot:.1f}%" for v, k in sorted(((v, k) for k, v in agg.items()), reverse=True)[:8]))
for i in sorted(range(len(b)), key=lambda i: -float(b[i][ist] or 0))[:top_n]:
    r = b[i]
    st = float(r[ist] or 0)
    t = max(((float(r[j] or 0), h) for j, h in stall_cols))
    print(f"{i:5d} {100 * st / tot:5.1f}%  x{float(r[iex]) / 1e3:8.1f}k  {r[isrc].strip()[:60]:60s} {t[1][6:]}")
