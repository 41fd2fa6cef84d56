"""Shared-memory instructions with the most excess (bank-conflict) wavefronts in a .ncu-rep.
usage: python scripts/ncu_conflicts.py rep [topN]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[1]
isrc, iex, iwf, iexe = (h.index("Source"), h.index("L1 Wavefronts Shared Excessive"), h.index("L1 Wavefronts Shared"),
                        h.index("Instructions Executed"))
data = []
for k, r in enumerate(rows[2:]):
    if len(r) != len(h):
        continue
    try:
        data.append((int(r[iex] or 0), int(r[iwf] or 0), int(r[iexe] or 0), k, r[isrc].strip()))
    except ValueError:
        pass
tot_ex = sum(d[0] for d in data) or 1
tot_wf = sum(d[1] for d in data) or 1
print(f"excess wavefronts {tot_ex} of {tot_wf} shared wavefronts ({100 * tot_ex / tot_wf:.1f}%)")
for ex, wf, exe, k, src in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"  [{k:5d}] excess {ex:9d} ({100 * ex / tot_ex:4.1f}%) wf {wf:9d} exe {exe:8d}  {src[:70]}")
