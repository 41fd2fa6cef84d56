"""Print key metrics + stall breakdown of every kernel in .ncu-rep files (reads here, no GPU)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print("==", rep, v[h.index("Kernel Name")][:90])
        for k in KEYS:
            if k in h:
                print(f"  {k} = {v[h.index(k)]} {u[h.index(k)]}")
        st = [(h[i], float(v[i] or 0)) for i in range(len(h))
              if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued") and v[i]]
        t = sum(x for _, x in st) or 1
        print("  stalls:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * x / t:.0f}%"
                                     for n, x in sorted(st, key=lambda a: -a[1])[:9]))
