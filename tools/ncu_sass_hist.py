"""Histogram of executed SASS opcodes and the top stall-sampled instructions of
one kernel in an ncu report:  python tools/ncu_sass_hist.py rep.ncu-rep <kernel regex> [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1:3]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iex, ist = (hdr.index(k) for k in ("Address", "Source", "Instructions Executed",
                                             "Warp Stall Sampling (All Samples)"))
body = [r for r in rows[2:] if len(r) > iex and r[iex].isdigit()]
tot = sum(int(r[iex]) for r in body)
samples = sum(int(r[ist] or 0) for r in body)
ops = Counter()
for r in body:
    op = r[isrc].split()
    op = op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "?")
    ops[op.split(".")[0]] += int(r[iex])
print(f"{kern}: {tot} warp instructions, {samples} stall samples")
for k, v in ops.most_common(top):
    print(f"  {k:10s} {v:12d} {100 * v / tot:5.1f}%")
print("top stall-sampled instructions:")
for r in sorted(body, key=lambda r: -int(r[ist] or 0))[:top]:
    print(f"  {r[ia][-5:]} {int(r[ist] or 0):6d} {r[isrc].strip()[:70]}")
