"""Summarise ncu outputs from gpurun_out/ into tracked files under profiles/.

usage: python scripts/make_profiles.py <round-tag> <launches.csv> [full.ncu-rep ...]

Writes profiles/<tag>_launches.md (per-kernel device time and share of the
step from the serialized, cold-cache launch list), profiles/<tag>_<rep>.txt
(key raw metrics + stall summary of each full capture) and merges per-launch
DRAM traffic into profiles/ncu_traffic.json (read by bench.py's roofline).
"""
import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

# libdbp kernel symbol -> bench kernel-timer name
NAMES = [(r"k_fused<\d+, 3>", "fused_mmse"), (r"k_fused<\d+, 4>", "fused_zf"), (r"k_fused<\d+, 0>", "fused_cg"), (r"k_fused<\d+, 1>", "fused_ul"), (r"k_fused<\d+, 2>", "fused_dl"),
         (r"k_prefold<\d+, 0, 0", "pre_cg"), (r"k_prefold<\d+, 0, 1", "pre_ul"), (r"k_prefold<\d+, 1, 2", "pre_dl"),
         (r"k_prelr<\d+, 0, 0", "pre_cg"), (r"k_prelr<\d+, 0, 1", "pre_ul"), (r"k_prelr<\d+, 1, 2", "pre_dl"),
         (r"k_gram<\d+, 0, 1", "gram_ul"), (r"k_gram<\d+, 1,", "gram_dl"), (r"k_inv_ul", "inv_ul"),
         (r"k_inv_dl", "inv_dl"), (r"k_admm_gj", "admm_fused"), (r"k_bf_gj", "bf_fused"),
         (r"k_admm_it", "admm_step"), (r"k_bf_it<\d+, 1>", "bf_final"), (r"k_bf_it", "bf_step"), (r"k_cg_gsum", "cg_gsum"),
         (r"k_cg_it<\d+, 1", "cg_fused"), (r"k_cg_tc", "cg_tc"), (r"k_cgg_tc", "cgg_tc"), (r"k_cg_it<\d+, 0", "cg_step"), (r"k_prox_out", "prox_out"),
         (r"k_mf", "mf"), (r"k_slice", "slice")]


def short(kname: str) -> str:
    for pat, n in NAMES:
        if re.search(pat, kname):
            return n
    return kname.split("(")[0][:50]


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("nsecond", "ns") else v * 1e3 if r[ui] in ("msecond", "ms") else v
        agg.setdefault(r[ki], []).append(v)
    ours = {k: v for k, v in agg.items() if "dbp::" in k}
    # shares over the timed step's kernels; everything else bench.py runs afterwards (the split path's per-round
    # timing, the centralized baselines) is listed apart
    STEP = ("fused_ul", "fused_dl", "fused_cg", "cg_tc")
    BASE = tuple(short(k) for k in ours if short(k) not in STEP)
    tot = sum(sum(v) for k, v in ours.items() if short(k) not in BASE) or 1.0
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             "Serialised, cold-cache per-launch times of `" + os.environ.get(
                 "LAUNCH_CMD", "bench.py --steps 3 --warmup 3") + "` (all launches of the",
             "process, libdbp kernels only below).  Compare SHARES with bench.py's live event timing, not",
             "absolute times.", "", "| kernel | launches | mean us | share of the step's libdbp time |", "|---|---|---|---|"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        sh = "not in the step" if short(k) in BASE else f"{sum(v)/tot:.3f}"
        lines.append(f"| {short(k)} (`{k.split('(')[0]}`) | {len(v)} | {sum(v)/len(v):.1f} | {sh} |")
    others = {k: v for k, v in agg.items() if "dbp::" not in k}
    lines += ["", "Non-libdbp launches in the same process (torch flush / setup): " +
              ", ".join(f"{k.split('(')[0][:40]} x{len(v)}" for k, v in others.items())]
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sector_hit_rate.pct"]


def full(tag, rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    out = [f"# {tag}: ncu --set full summary of {os.path.basename(rep)}", ""]
    traffic = {}
    tp = os.path.join(PROF, "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        out.append(f"## {short(name)}  ({name[:100]})")
        vals = {}
        for k in KEYS:
            if k in h:
                out.append(f"- {k} = {r[h.index(k)]} {units[h.index(k)]}")
                vals[k] = (r[h.index(k)], units[h.index(k)])
        st = [(h[i], float(r[i] or 0)) for i in range(len(h))
              if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued") and r[i]]
        tot = sum(v for _, v in st) or 1
        out.append("- stalls: " + ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100*v/tot:.0f}%"
                                           for n, v in sorted(st, key=lambda t: -t[1])[:8]))
        out.append("")

        def mb(k):
            v, u = vals[k]
            f = float(v.replace(",", ""))
            return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        if "dram__bytes_read.sum" in vals:
            traffic[short(name)] = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
    base = os.path.splitext(os.path.basename(rep))[0]
    open(os.path.join(PROF, f"{tag}_{base}.txt"), "w").write("\n".join(out) + "\n")
    json.dump(traffic, open(tp, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    os.makedirs(PROF, exist_ok=True)
    tag, lcsv = sys.argv[1], sys.argv[2]
    launches(tag, lcsv)
    for rep in sys.argv[3:]:
        full(tag, rep)
    print("wrote", sorted(os.listdir(PROF)))
