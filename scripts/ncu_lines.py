"""Per-CUDA-source-line stall samples of a .ncu-rep (all files), hottest first.
usage: python scripts/ncu_lines.py rep [topN]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
cur, hdr, out = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Name":
        cur = r[1].split("/")[-1]
        hdr = None
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        try:
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            exe = int(r[hdr.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        if smp or exe:
            out.append((smp, exe, cur, r[0], r[1].strip()[:80]))
tot = sum(o[0] for o in out) or 1
texe = sum(o[1] for o in out) or 1
byfile = {}
for o in out:
    b = byfile.setdefault(o[2], [0, 0]); b[0] += o[0]; b[1] += o[1]
print("by file:", {k: (f"{100*v[0]/tot:.1f}%", f"{100*v[1]/texe:.1f}%") for k, v in byfile.items()})
for smp, exe, f, ln, src in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{100*smp/tot:5.1f}% exe={100*exe/texe:5.1f}%  {f}:{ln}  {src}")
