"""Aggregate SASS-level stall samples of a .ncu-rep by region (source page), print hottest instructions
and a per-region summary.  usage: python scripts/ncu_hot.py rep [topN]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[1]
ia, isrc, isamp, iexe = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Instructions Executed")
ish = h.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in h else None
data = []
for r in rows[2:]:
    if len(r) <= isamp:
        continue
    try:
        data.append((int(r[ia], 16), r[isrc].strip(), int(r[isamp] or 0), int(r[iexe] or 0),
                     int(r[ish] or 0) if ish is not None else 0))
    except ValueError:
        pass
tot = sum(d[2] for d in data) or 1
texe = sum(d[3] for d in data) or 1
print(f"{len(data)} SASS instrs, {tot} samples, {texe} warp-instrs executed")
ops = {}
for _, s, n, e, x in data:
    op = s.split()[0] if s else "?"
    if op.startswith("@"):
        op = s.split()[1]
    op = op.split(".")[0]
    o = ops.setdefault(op, [0, 0, 0])
    o[0] += n; o[1] += e; o[2] += x
print("by opcode (samples%, exec%, excess smem wavefronts):")
for op, (n, e, x) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:18]:
    print(f"  {op:10s} {100*n/tot:5.1f}% {100*e/texe:5.1f}% {x}")
print("hottest:")
for a, s, n, e, x in sorted(data, key=lambda d: -d[2])[:top]:
    print(f"  {a & 0xfffff:6x} {100*n/tot:5.2f}% exe={e:8d} xs={x:6d}  {s[:90]}")
