#!/usr/bin/env python
"""bench.py -- detected Gbit/s per frame (and per-iteration latency) of libdbp.

Workload: one TDD slot on the B = 1024-antenna array of
BASELINE configs C and D -- C = 32 clusters of S = 32 antennas, U = 16 users,
N = 1200 subcarriers, N_sym = 1, T = 5 iterations, rho = 1.  A step runs the
whole hot path (every SURVEY 8(a) row) on one synthetic frame:
  * uplink 64-QAM frame (SNR 25 dB) detected by ADMM (Alg. 1) and by
    decentralized CG (Alg. 2);
  * downlink 16-QAM frame precoded by ADMM beamforming (Alg. 3).
value = (bits detected by ADMM + bits detected by CG + bits precoded) / step
time, bits = U * N * N_sym * log2|O| per solver (P753, P800).  Clusters are
split over the ranks (strong scaling) with one NCCL allreduce per consensus
round -- the only communication (P744-746).

Timing: W untimed warm-up steps; then exactly K steps, each bracketed by CUDA
events on the launch stream, with an untimed 256 MiB L2-flush write between
steps; barrier + synchronize on both sides; max over ranks.  At world = 1
the step runs the uplink pair (ADMM-UL then CG-UL, one stream) concurrently
with ADMM-DL (second stream, forked from and joined to the launch stream
inside the event bracket); a separate sequential region (all three back to
back on one stream) gives the per-solver times, per-iteration latencies and
the kernel-timer shares the roofline uses.  At world > 1 the step is the
sequential schedule (one communicator, one collective order).  The end-to-end
figure (e2e) calls the same C ABI with pinned HOST buffers, so every step
includes the host->device copy of its inputs and the device->host copy of
its outputs.  `--impl reference` times the fp64 oracle (oracle/) on the
host cores instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1702_04458_b200 import synth  # noqa: E402

METRIC = "detected Gbit/s per frame (and per-iteration latency) at 1/2/4/8 B200"
UL = synth.CONFIGS["C"]
DL = synth.CONFIGS["D"]
BITS = {"admm_ul": UL.bits_per_frame, "cg_ul": UL.bits_per_frame, "admm_dl": DL.bits_per_frame}
BITS_PER_STEP = sum(BITS.values())


def workload_config(world: int) -> dict:
    return {"workload": "TDD slot on configs C+D: B=1024 (C=32 x S=32), U=16, N=1200, N_sym=1, T=5; "
                        "ADMM-UL + CG-UL on a 64-QAM uplink frame (SNR 25 dB), ADMM-DL on a 16-QAM "
                        "downlink frame",
            "B": UL.B, "C": UL.C, "S": UL.S, "U": UL.U, "N": UL.N, "N_sym": UL.N_sym, "T": UL.T,
            "rho": UL.rho, "mod_ul": UL.mod, "mod_dl": DL.mod, "snr_db": UL.snr_db,
            "bits_per_step": BITS_PER_STEP, "parallelism": f"clusters split over {world} GPU(s), "
                                                             f"{UL.C // world} per GPU",
            "l2": "L2 flushed between timed steps (untimed 256 MiB write + read-back, so no dirty lines "
                  "are written back inside the timed step); each 157 MB channel input exceeds the 126 MB L2"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        self.proc.wait()
        self.th.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 9]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ oracle legs
_SAMPLES = {}


def _oracle_sample(n_sub: int):
    """Oracle on subcarriers [0, n_sub) of the same workload; returns (seconds, bits).
    The synthetic inputs are generated once per size (not timed)."""
    import oracle
    ul, dl = UL.scaled(N=n_sub), DL.scaled(N=n_sub)
    if n_sub not in _SAMPLES:
        H, y, _ = synth.uplink_frame(UL, n0=0, n1=n_sub)
        Hd, s = synth.downlink_frame(DL, n0=0, n1=n_sub)
        _SAMPLES[n_sub] = (H, y, Hd, s)
    H, y, Hd, s = _SAMPLES[n_sub]
    t0 = time.perf_counter()
    oracle.detect_admm(H, y, rho=ul.rho, N0=ul.N0, mod=ul.mod, T=ul.T)
    oracle.beamform_admm(Hd, s, rho=dl.rho, T=dl.T)
    oracle.detect_cg(H, y, rho=ul.N0, mod=ul.mod, T=ul.T)
    dt = time.perf_counter() - t0
    bits = 2 * ul.bits_per_frame + dl.bits_per_frame
    return dt, bits


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(budget_s: float = 10.0, n_sub: int = 240) -> dict:
    import oracle
    oracle.build()
    tot_t, tot_b, reps = 0.0, 0, 0
    while tot_t < budget_s and reps < 1000:
        dt, b = _oracle_sample(n_sub)
        tot_t += dt
        tot_b += b
        reps += 1
    return {"value": tot_b / tot_t / 1e9, "unit": "Gbit/s", "cores": host_cores(), "kind": "oracle",
            "sample": f"{n_sub} of {UL.N} subcarriers x all 3 solvers (all 32 clusters), {reps} repetition(s), "
                      f"{tot_t:.1f} s of fp64 C oracle with OpenMP over subcarriers"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    import oracle
    oracle.build()
    n_sub = args.ref_subcarriers
    for _ in range(args.warmup):
        _oracle_sample(n_sub)
    times, bits = [], 0
    for _ in range(args.steps):
        dt, b = _oracle_sample(n_sub)
        times.append(dt)
        bits = b
    tot = sum(times)
    value = bits * len(times) / tot / 1e9
    sample = (f"{n_sub} of {UL.N} subcarriers x all 3 solvers per step (all 32 clusters); fp64 C oracle, "
              f"OpenMP over subcarriers")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(world),
            "cpu_baseline": {"value": value, "unit": "Gbit/s", "cores": host_cores(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ roofline model
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # SMs x FP32 lanes x 2 flop/FMA x max SM clock


def algorithmic(kernel: str, C_loc: int):
    """(bound, amount) per launch of a libdbp kernel (DESIGN.md section 5 table).

    HBM-bound kernels: algorithmic bytes (each operand read once, each result
    written once).  FP32-bound preprocessing: algorithmic flops, 8 per complex
    MAC, counting the Hermitian Gram (S*tri(U) MACs), the matched filter
    (S*U*J), the Hermitian inverse (U*tri(U): one rank-1 update of the lower
    triangle per pivot) and y^reg (U*U*J).
    """
    S, U, N, J = UL.S, UL.U, UL.N, UL.N_sym
    tri = U * (U + 1) // 2
    P = C_loc * N
    c8 = 8
    gram, mf, inv, yreg = S * tri, S * U * J, U * tri, U * U * J
    T = UL.T
    mv = U * U                                   # one Hermitian mat-vec per pair and round
    flops = {
        "pre_cg": P * (gram + mf) * 8,
        "pre_ul": P * (gram + mf + inv + yreg) * 8,
        "pre_dl": P * (gram + inv) * 8,
        # single-kernel solvers: local preprocessing + the per-round local updates
        "fused_cg": (P * (gram + mf) + N * T * mv) * 8,
        "fused_ul": P * (gram + mf + inv + yreg + (T - 1) * mv) * 8,
        "fused_dl": P * (gram + inv + T * mv + S * U * J) * 8,
    }
    if kernel in flops:
        return "alu", float(flops[kernel])
    table = {
        # fused iterations: read G^{-1} (+ y^reg / s, H_c for the DL output), write outputs
        "admm_fused": P * (tri + J * U) * c8 + N * J * U * (c8 + 1),
        "bf_fused": P * (tri + S * U + J * S) * c8 + N * J * U * c8,
        "cg_gsum": P * (tri + J * U) * c8 + N * (tri + J * U) * c8,
        "cg_fused": N * (tri + J * U) * c8 + N * J * U * (c8 + 1),
    }
    return "hbm", float(table.get(kernel, 0.0))


def load_traffic() -> dict:
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


# ------------------------------------------------------------------ main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="dbp", choices=["dbp", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-table2", action="store_true")
    ap.add_argument("--sequential", action="store_true",
                    help="world = 1: time the step with the three solvers back to back on one stream")
    ap.add_argument("--device-consensus", action="store_true",
                    help="world > 1: consensus inside the fused kernels over NVLink (DBP_OPT_DEVICE_CONSENSUS)")
    ap.add_argument("--streams", type=int, default=2, choices=[2, 3],
                    help="world-1 concurrent schedule: 2 = ADMM-UL then ADMM-DL on one stream, CG-UL on another; "
                         "3 = every solver on its own stream")
    ap.add_argument("--plan", default=None,
                    help="world-1 concurrent schedule as solver lists per stream, e.g. "
                         "'admm_ul,cg_ul|admm_dl' (overrides --streams)")
    ap.add_argument("--ref-subcarriers", type=int, default=60)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "RANK" not in os.environ:
        world = 1
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1702_04458_b200 import dbp

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [dbp.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = dbp.Context(device=local, rank=rank, world=world, unique_id=uid)
    if args.device_consensus:
        ctx.set_option(dbp.OPT_DEVICE_CONSENSUS, 1)

    c0, c1 = synth.cluster_range(UL.C, rank, world)
    H, y, _ = synth.uplink_frame(UL, c0, c1)
    Hd, s = synth.downlink_frame(DL, c0, c1)
    C_loc = c1 - c0
    Hg, yg = torch.from_numpy(H).to(dev), torch.from_numpy(y).to(dev)
    Hdg, sg = torch.from_numpy(Hd).to(dev), torch.from_numpy(s).to(dev)
    s_hat = torch.empty((UL.N, UL.N_sym, UL.U), dtype=torch.complex64, device=dev)
    hard = torch.empty((UL.N, UL.N_sym, UL.U), dtype=torch.uint8, device=dev)
    x_hat = torch.empty_like(s_hat)
    hard2 = torch.empty_like(hard)
    xbf = torch.empty((C_loc, DL.N, DL.N_sym, DL.S), dtype=torch.complex64, device=dev)
    ws = {a: torch.empty(max(1, ctx.workspace_bytes(UL.C, UL.S, UL.U, UL.N, UL.N_sym, a)), dtype=torch.uint8,
                         device=dev) for a in ("admm_ul", "cg_ul", "admm_dl")}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_sink = torch.empty((), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def flush_l2(k):
        # evict L2 (untimed): write 256 MiB, then read it back so no dirty lines are
        # left to be written back inside the next timed step
        flush.fill_(k & 0xFF)
        torch.sum(flush.view(torch.int64), dim=0, out=flush_sink)

    def solver(name, T, st=None):
        sp = None if st is None else st.cuda_stream
        if name == "admm_ul":
            dbp.detect_admm(ctx, Hg, yg, rho=UL.rho, N0=UL.N0, mod=UL.mod, T=T, s_hat=s_hat, hard=hard,
                            ws=ws["admm_ul"], stream=sp)
        elif name == "admm_dl":
            dbp.beamform_admm(ctx, Hdg, sg, rho=DL.rho, T=T, x=xbf, ws=ws["admm_dl"], stream=sp)
        else:
            dbp.detect_cg(ctx, Hg, yg, rho=UL.N0, mod=UL.mod, T=T, x_hat=x_hat, hard=hard2, ws=ws["cg_ul"],
                          stream=sp)

    # Step schedule.  world == 1: ADMM-UL then ADMM-DL on one stream, CG-UL on a second, so each
    # kernel's CTAs fill the other's wave tail (the fastest of the six two-lane orders measured,
    # DESIGN.md section 6).  world > 1: sequential on one stream (every solver issues one NCCL allreduce per round
    # on the same communicator; two streams could order them differently across ranks).
    concurrent = world == 1 and not args.sequential
    plan = args.plan or ("admm_ul|admm_dl|cg_ul" if args.streams == 3 else "admm_ul,admm_dl|cg_ul")
    plan = [lane.split(",") for lane in plan.split("|")]
    assert sorted(sum(plan, [])) == ["admm_dl", "admm_ul", "cg_ul"], "--plan must name each solver once"
    side = tuple(torch.cuda.Stream(dev) for _ in plan) if concurrent else None
    join = (torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event())

    def step_concurrent(T, e_start):
        for sx in side:
            sx.wait_event(e_start)
        for sx, lane in zip(side, plan):
            for nm in lane:
                solver(nm, T, sx)
        for i, sx in enumerate(side):
            join[i].record(sx)
            stream.wait_event(join[i])

    def timed_concurrent(K, T):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        barrier()
        torch.cuda.synchronize()
        for k in range(K):
            flush_l2(k)
            ev[k][0].record(stream)
            step_concurrent(T, ev[k][0])
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        barrier()
        return sum(e0.elapsed_time(e1) for e0, e1 in ev)   # ms over K steps

    order = ["admm_ul", "admm_dl", "cg_ul"]   # BF between the two uplink passes: no L2 reuse of H

    def barrier():
        if world > 1:
            dist.barrier()

    def timed_region(K, T, names):
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)] for _ in range(K)]
        barrier()
        torch.cuda.synchronize()
        for k in range(K):
            flush_l2(k)
            ev[k][0].record(stream)
            for i, nm in enumerate(names):
                solver(nm, T)
                ev[k][i + 1].record(stream)
        torch.cuda.synchronize()
        barrier()
        per = np.zeros(len(names))
        for k in range(K):
            for i in range(len(names)):
                per[i] += ev[k][i].elapsed_time(ev[k][i + 1])
        return per  # ms summed over K steps, per solver

    for _ in range(args.warmup):
        for nm in order:
            solver(nm, UL.T)
        if concurrent:
            join[3].record(stream)
            step_concurrent(UL.T, join[3])
    ctx.sync()

    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.15)
    ctx.set_option(dbp.OPT_KERNEL_TIMING, 1)
    ctx.kernel_times(reset=True)
    st0 = ctx.stats()
    per = timed_region(args.steps, UL.T, order)        # sequential: per-solver times + kernel timer
    st1 = ctx.stats()
    ktimes = ctx.kernel_times(reset=True)
    ctx.set_option(dbp.OPT_KERNEL_TIMING, 0)
    conc_ms = None
    if concurrent:                                     # the step as scheduled (headline)
        st0 = ctx.stats()
        conc_ms = timed_concurrent(args.steps, UL.T)
        st1 = ctx.stats()
    clocks = clk.stop()
    ctx.sync()

    # per-iteration latency: (L(T) - L(1)) / (T - 1), per solver
    K1 = min(args.steps, 200)
    per1 = timed_region(K1, 1, order)


    def mx(v):
        if world == 1:
            return np.asarray(v, dtype=np.float64)
        t = torch.tensor(np.asarray(v, dtype=np.float64), device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().numpy()

    per = mx(per)
    per1 = mx(per1)

    # centralized baselines (Table I rows MMSE-UL / ZF-DL, the paper's comparison P789-792,
    # P810): same frames, timed alone; context only, not part of the step
    xb = torch.empty_like(s_hat)
    hb = torch.empty_like(hard)
    xz = torch.empty_like(xbf)
    wsb = {a: torch.empty(max(1, ctx.workspace_bytes(UL.C, UL.S, UL.U, UL.N, UL.N_sym, a)), dtype=torch.uint8,
                          device=dev) for a in ("mmse_ul", "zf_dl")}
    base_fns = {"mmse_ul": lambda: dbp.detect_mmse(ctx, Hg, yg, N0=UL.N0, mod=UL.mod, x_hat=xb, hard=hb,
                                                   ws=wsb["mmse_ul"]),
                "zf_dl": lambda: dbp.precode_zf(ctx, Hdg, sg, x=xz, ws=wsb["zf_dl"])}
    baselines = {}
    for nm, fn in base_fns.items():
        for _ in range(3):
            fn()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K1)]
        barrier()
        torch.cuda.synchronize()
        for e0, e1 in evs:
            flush_l2(0)
            e0.record(stream)
            fn()
            e1.record(stream)
        torch.cuda.synchronize()
        ms = float(mx([sum(e0.elapsed_time(e1) for e0, e1 in evs) / K1])[0])
        bits = UL.bits_per_frame if nm == "mmse_ul" else DL.bits_per_frame
        baselines[nm] = {"ms": ms, "gbps": bits / (ms * 1e-3) / 1e9}

    # the paper's own Table II workload (P803-804: U=16, 64-QAM, N=1200, N_sym=7 per coherence
    # interval, T=5, B=1024 = 32 x 32) next to its printed K40-cluster cells -- context only
    table2 = None
    if not args.no_table2:
        t2 = UL.scaled(N_sym=7)
        H7, y7, _ = synth.uplink_frame(t2, c0, c1)
        Hd7, s7 = synth.downlink_frame(t2.scaled(algo="admm_dl"), c0, c1)
        H7g, y7g = torch.from_numpy(H7).to(dev), torch.from_numpy(y7).to(dev)
        Hd7g, s7g = torch.from_numpy(Hd7).to(dev), torch.from_numpy(s7).to(dev)
        bits7 = t2.U * t2.N * t2.N_sym * 6
        paper = {"admm_ul": (21.53, 39.95, "P771"), "cg_ul": (13.61, 59.25, "P779"), "admm_dl": (11.11, 77.40, "P787")}
        fns = {"admm_ul": lambda: dbp.detect_admm(ctx, H7g, y7g, rho=t2.rho, N0=t2.N0, mod="qam64", T=t2.T),
               "cg_ul": lambda: dbp.detect_cg(ctx, H7g, y7g, rho=t2.N0, mod="qam64", T=t2.T),
               "admm_dl": lambda: dbp.beamform_admm(ctx, Hd7g, s7g, rho=t2.rho, T=t2.T)}
        table2 = {"workload": "B=1024 (C=32 x S=32), U=16, 64-QAM, N=1200, N_sym=7, T=5 (PAPER.md P803-804); "
                              "two-kernel path (the fused kernel takes N_sym = 1)",
                  "paper_hw": "32 x Tesla K40 + Cray Aries MPI (P685, P799), CPU wall clock"}
        K2 = 20
        for nm, fn in fns.items():
            for _ in range(2):
                fn()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K2)]
            barrier()
            torch.cuda.synchronize()
            for e0, e1 in evs:
                flush_l2(1)
                e0.record(stream)
                fn()
                e1.record(stream)
            torch.cuda.synchronize()
            ms = float(mx([sum(e0.elapsed_time(e1) for e0, e1 in evs) / K2])[0])
            pl, pt, cite = paper[nm]
            table2[nm] = {"ms": ms, "mbps": bits7 / (ms * 1e-3) / 1e6, "paper_ms": pl, "paper_mbps": pt,
                          "paper_cite": cite}
        del H7g, y7g, Hd7g, s7g
    total_ms = float(per.sum())
    ms_seq = total_ms / args.steps
    ms_step = float(mx([conc_ms])[0]) / args.steps if concurrent else ms_seq
    value = BITS_PER_STEP / (ms_step * 1e-3) / 1e9
    solvers = {}
    for i, nm in enumerate(order):
        msT = per[i] / args.steps
        ms1 = per1[i] / K1
        solvers[nm] = {"ms": msT, "gbps": BITS[nm] / (msT * 1e-3) / 1e9, "ms_T1": ms1,
                       "per_iter_us": 1e3 * (msT - ms1) / (UL.T - 1)}

    # dominant kernel and its roofline (algorithmic bytes / average launch time)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)"
    kern = {k: {"launches": int(v[0]), "avg_us": 1e3 * v[1] / max(v[0], 1), "share": v[1] / max(total_ms, 1e-9)}
            for k, v in ktimes.items()}
    dom = max(ktimes, key=lambda k: ktimes[k][1]) if ktimes else None
    roof = None
    if dom:
        avg_s = ktimes[dom][1] / ktimes[dom][0] * 1e-3
        bound, amt = algorithmic(dom, C_loc)
        traffic = load_traffic().get(dom)
        if bound == "hbm":
            roof = {"kernel": dom, "bound": "hbm", "achieved": amt / avg_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "frac": amt / avg_s / 1e9 / hbm_peak, "traffic": traffic, "algorithmic_bytes": amt,
                    "avg_launch_us": avg_s * 1e6, "peak_source": peak_src}
        else:
            roof = {"kernel": dom, "bound": "alu", "achieved": amt / avg_s / 1e12, "peak": FP32_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": amt / avg_s / 1e12 / FP32_PEAK_TFLOPS, "traffic": traffic,
                    "algorithmic_flops": amt, "avg_launch_us": avg_s * 1e6,
                    "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x 1965 MHz (B200_PROFILING.md)"}

    # end to end through the C ABI with pinned host buffers
    e2e = None
    if args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
        Hh, yh, Hdh, sh = pin(H), pin(y), pin(Hd), pin(s)
        o1 = torch.empty(tuple(s_hat.shape), dtype=torch.complex64).pin_memory().numpy()
        o2 = torch.empty(tuple(hard.shape), dtype=torch.uint8).pin_memory().numpy()
        o3 = torch.empty(tuple(s_hat.shape), dtype=torch.complex64).pin_memory().numpy()
        o4 = torch.empty(tuple(hard.shape), dtype=torch.uint8).pin_memory().numpy()
        o5 = torch.empty(tuple(xbf.shape), dtype=torch.complex64).pin_memory().numpy()

        def e2e_step():
            dbp.detect_admm(ctx, Hh, yh, rho=UL.rho, N0=UL.N0, mod=UL.mod, T=UL.T, s_hat=o1, hard=o2)
            dbp.beamform_admm(ctx, Hdh, sh, rho=DL.rho, T=DL.T, x=o5)
            dbp.detect_cg(ctx, Hh, yh, rho=UL.N0, mod=UL.mod, T=UL.T, x_hat=o3, hard=o4)

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier()
        dt = float(mx([time.perf_counter() - t0])[0]) / args.e2e_steps
        h2d = 2 * (Hh.nbytes + yh.nbytes) + Hdh.nbytes + sh.nbytes
        d2h = o1.nbytes + o2.nbytes + o3.nbytes + o4.nbytes + o5.nbytes
        e2e = {"value": BITS_PER_STEP / dt / 1e9, "unit": "Gbit/s", "ms_per_step": dt * 1e3,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "how": "same C-ABI calls on pinned host numpy buffers; library stages H2D/D2H on the stream; "
                      "host wall clock, max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()

    if rank == 0:
        launches = st1["kernel_launches"] - st0["kernel_launches"]
        line = {"metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_sequential": ms_seq,
                "schedule": ("concurrent, one stream per lane: " + " | ".join(" then ".join(l) for l in plan)
                             if concurrent else "sequential on one stream"),
                "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Philox-4x32: i.i.d. Rayleigh "
                "CN(0,1) channels, uniform Gray QAM, AWGN)", "config": workload_config(world),
                "solvers": solvers, "centralized_baselines": baselines, "paper_table2_context": table2,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
                "consensus_rounds_per_step": (st1["consensus_rounds"] - st0["consensus_rounds"]) / args.steps,
                "allreduce_calls_per_step": (st1["allreduce_calls"] - st0["allreduce_calls"]) / args.steps,
                "kernels": kern, "clocks": clocks}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
