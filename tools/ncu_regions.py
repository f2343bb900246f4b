"""Regions of one kernel's SASS by execution count (ncu source page CSV with --print-source sass):
python tools/ncu_regions.py <csv> [min share %]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
minshare = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = next(i for i, r in enumerate(rows) if 'Address' in r and 'Source' in r)
hdr, body = rows[hi], rows[hi + 1:]
ia, isrc, iex, ist = (hdr.index(k) for k in ("Address", "Source", "Instructions Executed", "Warp Stall Sampling (All Samples)"))
body = [r for r in body if len(r) > iex and r[iex].replace('.', '').isdigit()]
first = body[0][ia]
dup = [i for i, r in enumerate(body) if r[ia] == first]
b = body[:dup[1]] if len(dup) > 1 else body
tot = sum(float(r[iex]) for r in b)
stot = sum(float(r[ist] or 0) for r in b)
print(f"{len(b)} SASS instructions, {tot / 1e6:.1f} M warp instructions executed, {stot:.0f} stall samples")
segs, prev, start = [], None, 0
for i, r in enumerate(b):
    c = float(r[iex])
    if prev is None or abs(c - prev) > 0.02 * max(c, prev, 1):
        if prev is not None:
            segs.append((start, i - 1, prev))
        start, prev = i, c
segs.append((start, len(b) - 1, prev))
for s, e, c in segs:
    w = (e - s + 1) * c
    samp = sum(float(r[ist] or 0) for r in b[s:e + 1])
    if w > minshare / 100 * tot or samp > minshare / 100 * stot:
        ops = {}
        for r in b[s:e + 1]:
            op = r[isrc].split()
            op = op[1] if op and op[0].startswith('@') and len(op) > 1 else (op[0] if op else '?')
            ops[op.split('.')[0]] = ops.get(op.split('.')[0], 0) + 1
        top = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
        print(f"  [{s:5d}-{e:5d}] n={e - s + 1:4d} x {c / 1e3:8.1f}k = {100 * w / tot:5.1f}% inst, {100 * samp / max(stot, 1):5.1f}% stalls | {top}")
