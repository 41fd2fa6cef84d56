"""Summarise an ncu report: key raw metrics + top SASS lines by stall samples."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]


def stalls(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    for r in rows[2:]:
        items = [(h[i], float(r[i] or 0)) for i in range(len(h))
                 if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued") and r[i]]
        tot = sum(v for _, v in items) or 1
        top = sorted(items, key=lambda t: -t[1])[:8]
        print("  stalls:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100*v/tot:.0f}%"
                                     for n, v in top))


def run(rep, top=25):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("kernel:", r[h.index("Kernel Name")][:90])
        for k in KEYS:
            if k in h:
                print(f"  {k} = {r[h.index(k)]} {units[h.index(k)]}")
    stalls(rep)
    n_kernels = len(rows) - 2
    for kid in range(max(n_kernels, 1)):
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                              "--launch-skip", str(kid), "--launch-count", "1"],
                             capture_output=True, text=True).stdout
        srows = list(csv.reader(src.splitlines()))
        his = [i for i, r in enumerate(srows) if "Address" in r]
        if not his:
            continue
        hi = his[0]
        h = srows[hi]
        si = h.index("Warp Stall Sampling (All Samples)")
        data = [r for r in srows[hi + 1:] if len(r) == len(h) and r[si].replace(".", "").isdigit()]
        tot = sum(float(r[si] or 0) for r in data) or 1
        data.sort(key=lambda r: -float(r[si] or 0))
        print(f"[launch {kid}] top SASS by stall samples (total {tot:.0f}):")
        for r in data[:top]:
            print(f"  {100*float(r[si])/tot:5.1f}%  {r[h.index('Source')][:70]}")


if __name__ == "__main__":
    run(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
