"""Stall-reason breakdown per code region (SASS index ranges) of a .ncu-rep.
usage: python scripts/ncu_region_stalls.py rep start:end[:name] ..."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[1]
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
iexe = h.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) == len(h)]
for spec in sys.argv[2:]:
    parts = spec.split(":")
    a, b = int(parts[0]), int(parts[1])
    name = parts[2] if len(parts) > 2 else spec
    tot = {h[i]: 0 for i in cols}
    exe = 0
    for r in data[a:b]:
        for i in cols:
            tot[h[i]] += int(r[i] or 0)
        exe += int(r[iexe] or 0)
    s = sum(tot.values()) or 1
    top = sorted(tot.items(), key=lambda kv: -kv[1])[:8]
    print(f"{name:8s} samples={s:6d} exec={exe:10d}  " + ", ".join(f"{k[6:]} {100*v/s:.0f}%" for k, v in top))
