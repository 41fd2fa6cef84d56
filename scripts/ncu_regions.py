"""Bucket SASS-level stall samples of a .ncu-rep by code address (to locate hot regions of a big kernel).
usage: python scripts/ncu_regions.py rep [bucket_instrs]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[1]
isrc, isamp, iexe = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) <= isamp:
        continue
    try:
        data.append((r[isrc].strip(), int(r[isamp] or 0), int(r[iexe] or 0)))
    except ValueError:
        pass
tot = sum(d[1] for d in data) or 1
texe = sum(d[2] for d in data) or 1
for b0 in range(0, len(data), B):
    chunk = data[b0:b0 + B]
    smp = sum(c[1] for c in chunk)
    exe = sum(c[2] for c in chunk)
    if smp == 0 and exe == 0:
        continue
    ops = collections.Counter()
    for s, n, e in chunk:
        op = s.split()[0] if s else "?"
        if op.startswith("@"):
            op = s.split()[1]
        ops[op.split(".")[0]] += e
    top = ", ".join(f"{k}:{v * 100 // max(exe, 1)}%" for k, v in ops.most_common(4))
    print(f"[{b0:5d}-{b0 + len(chunk):5d}] samples {100 * smp / tot:5.1f}%  exec {100 * exe / texe:5.1f}%  {top}")
