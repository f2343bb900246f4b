"""Attribute ncu SASS-level samples/instructions to source lines.

usage: python tools/sass_lines.py <nvdisasm -g -c output> <kernel mangled name> <ncu source --print-source sass csv> [top]
"""
import csv
import re
import sys
from collections import defaultdict

dis, kern, sass_csv = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
addr_line = {}
inside = False
cur = None
for ln in open(dis):
    if ln.startswith("//----") and ".text." in ln:
        inside = ln.strip().endswith(kern + " --------------------------") or (".text." + kern + " ") in ln
        continue
    if not inside:
        continue
    m = re.search(r'## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        addr_line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ia, isamp, iinst = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
base = None
agg = defaultdict(lambda: [0, 0])
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ir = [hdr.index(h) for h in reasons]
rs = defaultdict(lambda: defaultdict(float))
rtot = defaultdict(float)
tot = [0, 0]
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    if base is None:
        base = a  # ncu reports absolute addresses; the disassembly is kernel-relative
    a -= base
    s, i = float(r[isamp] or 0), float(r[iinst] or 0)
    key = addr_line.get(a, ("?", 0))
    for h, j in zip(reasons, ir):
        v = float(r[j] or 0)
        rs[key][h[6:]] += v
        rtot[h[6:]] += v
    agg[key][0] += s
    agg[key][1] += i
    tot[0] += s
    tot[1] += i
print(f"total samples {tot[0]:.0f} instructions {tot[1]:.0f}; mapped addrs {len(addr_line)}")
def top3(d):
    t = sum(d.values()) or 1
    return " ".join(f"{k}={100 * v / t:.0f}%" for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:3])


print("stall reasons:", " ".join(f"{k}={100 * v / tot[0]:.1f}%" for k, v in sorted(rtot.items(), key=lambda kv: -kv[1])[:9]))
for key, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{key[0]}:{key[1]:<5d} samples {100 * s / tot[0]:5.1f}%  inst {100 * i / tot[1]:5.1f}%  {top3(rs[key])}")
