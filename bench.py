#!/usr/bin/env python
"""bench.py -- detected Gbit/s per frame (and per-iteration latency) of libdbp.

Workload: one TDD slot on the B = 1024-antenna array of
BASELINE configs C and D -- C = 32 clusters of S = 32 antennas, U = 16 users,
N = 1200 subcarriers, N_sym = 1, T = 5 iterations, rho = 1.  A step runs the
whole hot path (every SURVEY 8(a) row) on three synthetic frames:
  * a 64-QAM uplink frame (SNR 25 dB) detected by ADMM (Alg. 1);
  * a second, independent 64-QAM uplink frame (its own seed) detected by
    decentralized CG (Alg. 2) -- no two passes of a step share a channel, so
    no pass can be served from another's L2 lines;
  * a 16-QAM downlink frame precoded by ADMM beamforming (Alg. 3).
value = (bits detected by ADMM + bits detected by CG + bits precoded) / step
time, bits = U * N * N_sym * log2|O| per frame (P753, P800).  Clusters are
split over the ranks (strong scaling) with one NCCL allreduce per consensus
round -- the only communication (P744-746).

Launch: `--gpus N` with N > 1 and no torchrun environment re-executes itself
under `torch.distributed.run` (127.0.0.1) with N ranks, after checking that N
GPUs are visible (it fails loudly otherwise); under torchrun WORLD_SIZE must
equal --gpus.  At world > 1 the run also reports (i) the same step with the
device-side consensus (DBP_OPT_DEVICE_CONSENSUS, NEXT-1) cross-checked against
the NCCL path, (ii) a world-1 solve of the whole frame on every rank that both
must match to rel-L2 <= 1e-5 (SURVEY 8(c) "across GPU counts"), (iii) the
subcarrier-sharded control (every rank all clusters of N/G subcarriers, no
communication) and (iv) per-rank exposed-allreduce time and the
NCCL communicator size.

Timing: W untimed warm-up steps; then exactly K steps, each bracketed by CUDA
events on the launch stream, with an untimed 256 MiB L2-flush write between
steps; barrier + synchronize on both sides; max over ranks.  At world = 1
the step runs ADMM-UL, ADMM-DL and CG-UL back to back on one stream (forked
from and joined to the launch stream inside the event bracket), each solver
launched with DBP_OPT_OVERLAP_PREV so its CTAs fill its predecessor's last wave
(the three frames are independent); a separate sequential region (all three back to back) gives the
per-solver times, per-iteration latencies and the kernel-timer shares the
roofline uses.  At world > 1 the step is sequential (one communicator, one
collective order).  `e2e` calls the same C ABI with pinned HOST buffers, so
every step includes the host->device copy of its inputs and the device->host
copy of its outputs.  `--impl reference` times the fp64 oracle (oracle/) on
the host cores instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1702_04458_b200 import synth  # noqa: E402

METRIC = "detected Gbit/s per frame (and per-iteration latency) at 1/2/4/8 B200"
UL = synth.CONFIGS["C"]
CG = UL.scaled(name="C-cg", algo="cg_ul", seed=UL.seed + 1000)     # an independent uplink frame
DL = synth.CONFIGS["D"]
BITS = {"admm_ul": UL.bits_per_frame, "cg_ul": CG.bits_per_frame, "admm_dl": DL.bits_per_frame}
BITS_PER_STEP = sum(BITS.values())
ORDER = ["admm_ul", "admm_dl", "cg_ul"]


def workload_config(world: int) -> dict:
    return {"workload": "TDD slot on configs C+D: B=1024 (C=32 x S=32), U=16, N=1200, N_sym=1, T=5; "
                        "ADMM-UL on a 64-QAM uplink frame, CG-UL on a second independent 64-QAM uplink "
                        "frame (SNR 25 dB), ADMM-DL on a 16-QAM downlink frame",
            "B": UL.B, "C": UL.C, "S": UL.S, "U": UL.U, "N": UL.N, "N_sym": UL.N_sym, "T": UL.T,
            "rho": UL.rho, "mod_ul": UL.mod, "mod_dl": DL.mod, "snr_db": UL.snr_db,
            "seeds": {"admm_ul": UL.seed, "cg_ul": CG.seed, "admm_dl": DL.seed},
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


# ------------------------------------------------------------------ synthetic frames
def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _gen(args):
    kind, cfg, c0, c1, n0, n1 = args
    if kind == "ul":
        H, y, _ = synth.uplink_frame(cfg, c0, c1, n0, n1)
        return H, y
    return synth.downlink_frame(cfg, c0, c1, n0, n1)


_POOL = {}


def _pool(workers: int):
    """One process pool for all frame generation, started with 'spawn' (the bench process already
    holds CUDA / NCCL threads, which a fork would copy in an undefined state)."""
    if workers not in _POOL:
        import multiprocessing as mp
        _POOL[workers] = ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn"))
    return _POOL[workers]


def gen_frame(kind: str, cfg, c0: int, c1: int, n0: int = 0, n1: int | None = None, workers: int = 1):
    """synth frame of clusters [c0, c1), subcarriers [n0, n1), generated per cluster in parallel
    (the values do not depend on the split: counter-based Philox)."""
    n1 = cfg.N if n1 is None else n1
    jobs = [(kind, cfg, c, c + 1, n0, n1) for c in range(c0, c1)]
    if workers <= 1 or len(jobs) == 1:
        parts = [_gen(j) for j in jobs]
    else:
        parts = list(_pool(workers).map(_gen, jobs))
    if kind == "ul":
        return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])
    return np.concatenate([p[0] for p in parts]), parts[0][1]


# ------------------------------------------------------------------ oracle legs
_SAMPLES = {}


_ORACLE_OUT = {}


def _oracle_sample(n_sub: int, keep: bool = False):
    """Oracle on subcarriers [0, n_sub) of the same three frames; returns (seconds, bits).
    The synthetic inputs are generated once per size (not timed); keep: store the outputs."""
    import oracle
    ul, cg, dl = UL.scaled(N=n_sub), CG.scaled(N=n_sub), DL.scaled(N=n_sub)
    if n_sub not in _SAMPLES:
        H, y, _ = synth.uplink_frame(UL, n0=0, n1=n_sub)
        Hc, yc, _ = synth.uplink_frame(CG, n0=0, n1=n_sub)
        Hd, s = synth.downlink_frame(DL, n0=0, n1=n_sub)
        _SAMPLES[n_sub] = (H, y, Hc, yc, Hd, s)
    H, y, Hc, yc, Hd, s = _SAMPLES[n_sub]
    t0 = time.perf_counter()
    o_ul = oracle.detect_admm(H, y, rho=ul.rho, N0=ul.N0, mod=ul.mod, T=ul.T)
    o_dl = oracle.beamform_admm(Hd, s, rho=dl.rho, T=dl.T)
    o_cg = oracle.detect_cg(Hc, yc, rho=cg.N0, mod=cg.mod, T=cg.T)
    dt = time.perf_counter() - t0
    if keep:
        _ORACLE_OUT[n_sub] = (o_ul, o_cg, o_dl)
    bits = ul.bits_per_frame + cg.bits_per_frame + dl.bits_per_frame
    return dt, bits


PARITY_SUB = 240                                       # subcarriers of the cpu_baseline sample


def parity_report(gpu, n_sub: int = PARITY_SUB) -> dict:
    """The timed step's outputs on the cpu_baseline sample against the oracle's (same frames, same
    subcarriers): rel-L2 over the sample and the worst subcarrier, hard-bit mismatches."""
    (s_ref, h_ref), (x_ref, hx_ref), b_ref = _ORACLE_OUT[n_sub]
    s_g, h_g, x_g, hx_g, b_g = gpu

    def rel(a, b, ax):
        a, b = np.asarray(a), np.asarray(b)
        whole = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
        bb = np.moveaxis(b, ax, 0).reshape(b.shape[ax], -1)
        aa = np.moveaxis(a, ax, 0).reshape(a.shape[ax], -1)
        den = np.maximum(np.linalg.norm(bb, axis=1), 1e-3 * np.sqrt(np.mean(np.linalg.norm(bb, axis=1) ** 2)))
        return whole, float(np.max(np.linalg.norm(aa - bb, axis=1) / den))
    out = {"how": f"the timed step's outputs on subcarriers [0, {n_sub}) against the fp64 oracle's (cpu_baseline "
                  "sample): rel-L2 over the sample / worst subcarrier; hard-bit mismatches (ties not excused)",
           "bar": 1e-4}
    for nm, a, b, ax, hg, hr in (("admm_ul", s_g, s_ref, 0, h_g, h_ref), ("cg_ul", x_g, x_ref, 0, hx_g, hx_ref),
                                 ("admm_dl", b_g, b_ref, 1, None, None)):
        w, m = rel(a, b, ax)
        out[nm] = {"rel_l2": w, "max_subcarrier": m}
        if hg is not None:
            out[nm]["hard_mismatch"] = int(np.count_nonzero(np.asarray(hg) != np.asarray(hr)))
    return out


def cpu_baseline(budget_s: float = 10.0, n_sub: int = PARITY_SUB) -> dict:
    import oracle
    oracle.build()
    tot_t, tot_b, reps = 0.0, 0, 0
    while tot_t < budget_s and reps < 1000:
        dt, b = _oracle_sample(n_sub, keep=reps == 0)
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
        # tensor-core CG (world 1): read H_c and y_c once, write x_hat (+ hard bits)
        "cg_tc": P * (S * U + S * J) * c8 + N * J * U * (c8 + 1),
    }
    return "hbm", float(table.get(kernel, 0.0))


def peaks_hbm():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except Exception:
        return None


def load_traffic() -> dict:
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


# ------------------------------------------------------------------ launcher / rank plumbing
def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args) -> int | None:
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run with N ranks (None: no
    relaunch needed).  Refuses (exit 2) if fewer than N GPUs are visible -- a multi-GPU number is
    never silently measured on fewer GPUs."""
    if "RANK" in os.environ or args.gpus <= 1:
        return None
    if not args.plumbing_check and not args.host_comm:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible; "
                             f"refusing to report a {args.gpus}-GPU number\n")
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def rank_env(args):
    if "RANK" not in os.environ:
        return 0, 1, 0
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; launch one rank per GPU")
    return rank, world, local


def _coll_device(dist, device):
    """Collectives of the bench's own bookkeeping run on the process group's device (CPU for gloo)."""
    return device if dist.get_backend() == "nccl" else None


def max_over_ranks(vals, world, dist, device=None):
    if world == 1:
        return np.asarray(vals, dtype=np.float64)
    import torch
    t = torch.tensor(np.asarray(vals, dtype=np.float64), device=_coll_device(dist, device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


def gather_rows(row, world, dist, device=None):
    """all ranks' float rows (same length) -> [world][len] on every rank."""
    if world == 1:
        return [list(row)]
    import torch
    t = torch.tensor(np.asarray(row, dtype=np.float64), device=_coll_device(dist, device))
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [o.cpu().numpy().tolist() for o in out]


def plumbing_check(args, rank: int, world: int):
    """CPU stand-in for the multi-rank GPU run (gloo): the same launcher, rank/world checks,
    unique-id broadcast, cluster partition and max-over-ranks / gather reductions, with a
    rank-dependent fake step time -- so the N > 1 plumbing is testable without GPUs."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    uid = None
    if world > 1:
        obj = [os.urandom(128) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    c0, c1 = synth.cluster_range(UL.C, rank, world)
    fake_ms = 1.0 + rank
    mx = float(max_over_ranks([fake_ms], world, dist)[0])
    rows = gather_rows([rank, c0, c1, len(uid) if uid else 0], world, dist)
    if rank == 0:
        print(json.dumps({"plumbing": True, "n_gpus": world, "max_ms": mx,
                          "ranks": [{"rank": int(r[0]), "clusters": [int(r[1]), int(r[2])], "uid_bytes": int(r[3])}
                                    for r in rows]}), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config entries (world = 1)")
    ap.add_argument("--sequential", action="store_true",
                    help="world = 1: time the step with the three solvers back to back on one stream")
    ap.add_argument("--no-device-consensus", action="store_true",
                    help="world > 1: skip the device-side consensus leg (DBP_OPT_DEVICE_CONSENSUS)")
    ap.add_argument("--streams", type=int, default=1, choices=[1, 2, 3],
                    help="world-1 step schedule: 1 = ADMM-UL, ADMM-DL, CG-UL on one stream (overlapped launches); "
                         "2 = ADMM-UL then ADMM-DL on one stream, CG-UL on another; 3 = every solver on its own "
                         "stream")
    ap.add_argument("--plan", default=None,
                    help="world-1 concurrent schedule as solver lists per stream, e.g. "
                         "'admm_ul,cg_ul|admm_dl' (overrides --streams)")
    ap.add_argument("--no-overlap", action="store_true",
                    help="world-1 concurrent schedule without DBP_OPT_OVERLAP_PREV (a solver following another on "
                         "its stream then waits for it to drain instead of filling its last wave)")
    ap.add_argument("--ref-subcarriers", type=int, default=60)
    ap.add_argument("--plumbing-check", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--host-comm", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()

    rc = relaunch(args)
    if rc is not None:
        sys.exit(rc)
    rank, world, local = rank_env(args)
    if args.plumbing_check:
        plumbing_check(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1702_04458_b200 import dbp

    if args.host_comm:
        # test mode: ranks may share a GPU; the consensus exchange is the library's host allreduce hook
        # over gloo instead of NCCL (which refuses two ranks on one device) -- everything else is the
        # world > 1 path of this script
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    uid = None
    if world > 1 and args.host_comm:
        dist.init_process_group("gloo")
    elif world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [dbp.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = dbp.Context(device=local, rank=rank, world=world, unique_id=uid)
    if world > 1 and args.host_comm:
        def _hook(arr):
            t = torch.from_numpy(arr)
            dist.all_reduce(t)
        ctx.set_allreduce_hook(_hook)
    comm = ctx.comm_info()
    if comm["nranks"] != world or comm["rank"] != rank:
        raise SystemExit(f"bench.py: NCCL communicator {comm} does not match rank {rank} / world {world}")

    workers = max(1, host_cores() // max(world, 1))
    c0, c1 = synth.cluster_range(UL.C, rank, world)
    C_loc = c1 - c0
    if world == 1:
        H, y = gen_frame("ul", UL, 0, UL.C, workers=workers)
        Hc, yc = gen_frame("ul", CG, 0, CG.C, workers=workers)
        Hd, s = gen_frame("dl", DL, 0, DL.C, workers=workers)
        full = (H, y, Hc, yc, Hd, s)
    else:
        # every rank generates the whole frames: its cluster block runs the decentralized path, the
        # whole frame the world-1 reference solve and the subcarrier-sharded control
        full = (*gen_frame("ul", UL, 0, UL.C, workers=workers), *gen_frame("ul", CG, 0, CG.C, workers=workers),
                *gen_frame("dl", DL, 0, DL.C, workers=workers))
        H, y, Hc, yc, Hd, s = (full[0][c0:c1], full[1][c0:c1], full[2][c0:c1], full[3][c0:c1],
                               full[4][c0:c1], full[5])
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    Hg, yg, Hcg, ycg, Hdg, sg = to(H), to(y), to(Hc), to(yc), to(Hd), to(s)
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

    def barrier():
        if world > 1:
            dist.barrier()

    def mx(v):
        return max_over_ranks(v, world, dist, dev)

    def solver(name, T, st=None, c=None):
        c = ctx if c is None else c
        sp = None if st is None else st.cuda_stream
        if name == "admm_ul":
            dbp.detect_admm(c, Hg, yg, rho=UL.rho, N0=UL.N0, mod=UL.mod, T=T, s_hat=s_hat, hard=hard,
                            ws=ws["admm_ul"], stream=sp)
        elif name == "admm_dl":
            dbp.beamform_admm(c, Hdg, sg, rho=DL.rho, T=T, x=xbf, ws=ws["admm_dl"], stream=sp)
        else:
            dbp.detect_cg(c, Hcg, ycg, rho=CG.N0, mod=CG.mod, T=T, x_hat=x_hat, hard=hard2, ws=ws["cg_ul"],
                          stream=sp)

    # Step schedule.  world == 1: the three solvers back to back on one stream, each launched with
    # DBP_OPT_OVERLAP_PREV so its CTAs fill the previous kernel's last wave (209.5 vs 211.9 us for the
    # two-stream plan admm_ul,admm_dl|cg_ul).  world > 1: sequential on one
    # stream (every solver issues NCCL allreduces on one communicator; two streams could order them
    # differently across ranks).
    concurrent = world == 1 and not args.sequential
    plan = args.plan or {1: "admm_ul,admm_dl,cg_ul", 2: "admm_ul,admm_dl|cg_ul", 3: "admm_ul|admm_dl|cg_ul"}[args.streams]
    plan = [lane.split(",") for lane in plan.split("|")]
    assert sorted(sum(plan, [])) == sorted(ORDER), "--plan must name each solver once"
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

    steps_ms = {}                                      # per-step event times of the last timed region

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
        steps_ms["step"] = [e0.elapsed_time(e1) for e0, e1 in ev]
        return sum(steps_ms["step"])                       # ms over K steps

    def timed_region(K, T, names, fn=None):
        fn = fn or solver
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)] for _ in range(K)]
        barrier()
        torch.cuda.synchronize()
        for k in range(K):
            flush_l2(k)
            ev[k][0].record(stream)
            for i, nm in enumerate(names):
                fn(nm, T)
                ev[k][i + 1].record(stream)
        torch.cuda.synchronize()
        barrier()
        m = np.array([[ev[k][i].elapsed_time(ev[k][i + 1]) for i in range(len(names))] for k in range(K)])
        steps_ms["region"] = m                             # [K][solver] ms, for the latency percentiles
        return m.sum(axis=0)  # ms summed over K steps, per solver

    for _ in range(args.warmup):
        for nm in ORDER:
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
    per = timed_region(args.steps, UL.T, ORDER)        # sequential: per-solver times + kernel timer
    seq_steps = steps_ms["region"]
    st1 = ctx.stats()
    ktimes = ctx.kernel_times(reset=True)
    ctx.set_option(dbp.OPT_KERNEL_TIMING, 0)
    kern_ms_rank = sum(v[1] for v in ktimes.values()) / args.steps       # this rank's kernel time per step
    step_ms_rank = float(np.sum(per)) / args.steps
    conc_ms = None
    overlap = False
    gpu_sample = None
    comm_stats = (st0, st1)                            # the timed-kernel region's counters (per-rank comm)
    if concurrent:                                     # the step as scheduled (headline)
        # consecutive solvers on a lane are independent frames: each may start in its predecessor's
        # last wave (programmatic dependent launch; outputs still ordered, include/dbp.h)
        overlap = not args.no_overlap
        ctx.set_option(dbp.OPT_OVERLAP_PREV, int(overlap))
        step_concurrent(UL.T, join[3])                 # warm the overlapped launch path
        st0 = ctx.stats()
        conc_ms = timed_concurrent(args.steps, UL.T)
        step_list = steps_ms["step"]
        if rank == 0 and not args.no_cpu_baseline:     # the step's outputs on the oracle sample (parity)
            ctx.sync()
            gpu_sample = tuple(t[:PARITY_SUB].cpu().numpy() for t in (s_hat, hard, x_hat, hard2)) + (
                xbf[:, :PARITY_SUB].cpu().numpy(),)
        st1 = ctx.stats()
        ctx.set_option(dbp.OPT_OVERLAP_PREV, 0)
    else:
        # world > 1: the headline is the sequential step WITHOUT the per-kernel event timer (which brackets
        # every launch and disables graph replay); the timed-kernel region above gives the breakdown
        st0 = ctx.stats()
        conc_ms = float(np.sum(timed_region(args.steps, UL.T, ORDER)))
        step_list = steps_ms["region"].sum(axis=1).tolist()
        st1 = ctx.stats()
    clocks = clk.stop()
    ctx.sync()

    # per-iteration latency: (L(T) - L(1)) / (T - 1), per solver
    K1 = min(args.steps, 200)
    per1 = timed_region(K1, 1, ORDER)
    per = mx(per)
    per1 = mx(per1)

    # ... and directly, per consensus round: the split path (one launch per round, the path world > 1 runs)
    # under the kernel event timer; at world 1 forced (no collective), at world > 1 the timed-kernel region
    split_iter = None
    if world == 1:
        ctx.set_option(dbp.OPT_FORCE_SPLIT, 1)
        for nm in ORDER:
            solver(nm, UL.T)
        ctx.sync()
        ctx.set_option(dbp.OPT_KERNEL_TIMING, 1)
        ctx.kernel_times(reset=True)
        for _ in range(K1):
            for nm in ORDER:
                solver(nm, UL.T)
        ctx.sync()
        kts = ctx.kernel_times(reset=True)
        ctx.set_option(dbp.OPT_KERNEL_TIMING, 0)
        ctx.set_option(dbp.OPT_FORCE_SPLIT, 0)
    else:
        kts = ktimes
    split_iter = {"how": "split path, per-launch device time of each per-round kernel (kernel event timer); "
                         + ("forced at world 1, no collective" if world == 1 else "this rank, world > 1"),
                  **{k: 1e3 * v[1] / max(v[0], 1) for k, v in kts.items()
                     if k in ("admm_step", "bf_step", "cg_step", "ss_ul_step", "ss_dl_step")}}

    def timed_fn(fn, K, flush_k=0):
        for _ in range(3):
            fn()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        barrier()
        torch.cuda.synchronize()
        for e0, e1 in evs:
            flush_l2(flush_k)
            e0.record(stream)
            fn()
            e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return float(mx([sum(e0.elapsed_time(e1) for e0, e1 in evs) / K])[0])

    # ---------------------------------------------------------------- world > 1 legs
    multi = None
    if world > 1:
        multi = {"nccl_comm": comm, "modes": {}}
        for nm in ORDER:                                  # the T = 1 region ran last: redo the T-round step
            solver(nm, UL.T)
        ctx.sync()
        ref_outs = (s_hat.cpu().numpy().copy(), x_hat.cpu().numpy().copy(), xbf.cpu().numpy().copy())
        rows = gather_rows([step_ms_rank, kern_ms_rank, step_ms_rank - kern_ms_rank,
                            (comm_stats[1]["allreduce_calls"] - comm_stats[0]["allreduce_calls"]) / args.steps],
                           world, dist, dev)
        multi["per_rank"] = [{"rank": r, "step_ms": v[0], "kernel_ms": v[1], "exposed_comm_ms": v[2],
                              "allreduce_calls_per_step": v[3]} for r, v in enumerate(rows)]

        def rel(a, b):
            return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))

        # (i) device-side consensus (NEXT-1) on the same step, cross-checked against the NCCL path.  Every
        # rank runs the same sequence of collectives whatever happens locally: solver errors are caught per
        # call, and the ranks agree (MIN over ranks) on success before any result is reduced.
        if not args.no_device_consensus:
            errs = []

            def dc_solver(nm, T):
                try:
                    solver(nm, T)
                except Exception as e:   # noqa: BLE001 -- a bounded timeout or launch error, never a hang
                    errs.append(str(e)[:300])

            def agree(ok):
                return bool(max_over_ranks([0.0 if ok else 1.0], world, dist, dev)[0] == 0.0)

            def synced():
                try:
                    ctx.sync()
                except Exception as e:   # noqa: BLE001
                    errs.append(str(e)[:300])
                return not errs

            ctx.set_option(dbp.OPT_DEVICE_CONSENSUS, 1)
            for _ in range(3):
                for nm in ORDER:
                    dc_solver(nm, UL.T)
            ok = agree(synced())
            pdc = None
            if ok:
                pdc = mx(timed_region(args.steps, UL.T, ORDER, fn=dc_solver))
                ok = agree(synced())
            ctx.set_option(dbp.OPT_DEVICE_CONSENSUS, 0)
            if ok:
                dc = (s_hat.cpu().numpy(), x_hat.cpu().numpy(), xbf.cpu().numpy())
                err = [rel(a, b) for a, b in zip(dc, ref_outs)]
                ms = float(pdc.sum()) / args.steps
                multi["modes"]["device_consensus"] = {
                    "ms_per_step": ms, "value": BITS_PER_STEP / (ms * 1e-3) / 1e9,
                    "rel_l2_vs_nccl": {"admm_ul": err[0], "cg_ul": err[1], "admm_dl": err[2]},
                    "solvers_ms": dict(zip(ORDER, (pdc / args.steps).tolist()))}
            else:
                multi["modes"]["device_consensus"] = {"error": (errs[0] if errs else "failed on another rank")}

        # (ii) world-1 solve of the whole frame on every rank (same GPU): rel-L2 <= 1e-5
        ctx1 = dbp.Context(device=local, rank=0, world=1)
        Hf, yf, Hcf, ycf, Hdf, sf = (to(a) for a in full)
        s1, _ = dbp.detect_admm(ctx1, Hf, yf, rho=UL.rho, N0=UL.N0, mod=UL.mod, T=UL.T)
        x1, _ = dbp.detect_cg(ctx1, Hcf, ycf, rho=CG.N0, mod=CG.mod, T=CG.T)
        b1 = dbp.beamform_admm(ctx1, Hdf, sf, rho=DL.rho, T=DL.T)
        ctx1.sync()
        e1 = [rel(ref_outs[0], s1.cpu().numpy()), rel(ref_outs[1], x1.cpu().numpy()),
              rel(ref_outs[2], b1[c0:c1].cpu().numpy())]
        worst = mx([max(e1)])[0]
        multi["vs_world1"] = {"rel_l2": {"admm_ul": e1[0], "cg_ul": e1[1], "admm_dl": e1[2]},
                              "max_over_ranks": float(worst), "ok": bool(worst <= 1e-5)}

        # (iii) subcarrier-sharded control: all clusters of N/G subcarriers per rank, no communication
        n0, n1 = rank * UL.N // world, (rank + 1) * UL.N // world
        shard = {k: to(np.ascontiguousarray(a[:, n0:n1] if a.ndim == 4 else a[n0:n1]))
                 for k, a in zip(("H", "y", "Hc", "yc", "Hd", "s"), full)}

        def ctrl(nm, T):
            if nm == "admm_ul":
                dbp.detect_admm(ctx1, shard["H"], shard["y"], rho=UL.rho, N0=UL.N0, mod=UL.mod, T=T)
            elif nm == "cg_ul":
                dbp.detect_cg(ctx1, shard["Hc"], shard["yc"], rho=CG.N0, mod=CG.mod, T=T)
            else:
                dbp.beamform_admm(ctx1, shard["Hd"], shard["s"], rho=DL.rho, T=T)

        for _ in range(3):
            for nm in ORDER:
                ctrl(nm, UL.T)
        pc = mx(timed_region(args.steps, UL.T, ORDER, fn=ctrl))
        ms = float(pc.sum()) / args.steps
        multi["modes"]["control_subcarrier_sharded"] = {
            "ms_per_step": ms, "value": BITS_PER_STEP / (ms * 1e-3) / 1e9, "scaling": "weak-equivalent",
            "subcarriers_per_rank": n1 - n0, "solvers_ms": dict(zip(ORDER, (pc / args.steps).tolist()))}
        del Hf, yf, Hcf, ycf, Hdf, sf, shard
        ctx1.close()

    # ---------------------------------------------------------------- world == 1 context legs
    baselines, table2, configs = {}, None, None
    if world == 1:
        # centralized baselines (Table I rows MMSE-UL / ZF-DL, the paper's comparison P789-792, P810)
        xb, hb, xz = torch.empty_like(s_hat), torch.empty_like(hard), torch.empty_like(xbf)
        wsb = {a: torch.empty(max(1, ctx.workspace_bytes(UL.C, UL.S, UL.U, UL.N, UL.N_sym, a)), dtype=torch.uint8,
                              device=dev) for a in ("mmse_ul", "zf_dl")}
        for nm, fn, bits in (("mmse_ul", lambda: dbp.detect_mmse(ctx, Hg, yg, N0=UL.N0, mod=UL.mod, x_hat=xb,
                                                                  hard=hb, ws=wsb["mmse_ul"]), UL.bits_per_frame),
                             ("zf_dl", lambda: dbp.precode_zf(ctx, Hdg, sg, x=xz, ws=wsb["zf_dl"]),
                              DL.bits_per_frame)):
            ms = timed_fn(fn, K1)
            baselines[nm] = {"ms": ms, "gbps": bits / (ms * 1e-3) / 1e9}

        # the paper's own Table II workload (P803-804: U=16, 64-QAM, N=1200, N_sym=7 per coherence
        # interval, T=5, B=1024 = 32 x 32) next to its printed K40-cluster cells -- context only
        if not args.no_table2:
            t2 = UL.scaled(N_sym=7)
            H7, y7 = gen_frame("ul", t2, 0, t2.C, workers=workers)
            Hd7, s7 = gen_frame("dl", t2.scaled(algo="admm_dl"), 0, t2.C, workers=workers)
            H7g, y7g, Hd7g, s7g = to(H7), to(y7), to(Hd7), to(s7)
            bits7 = t2.U * t2.N * t2.N_sym * 6
            paper = {"admm_ul": (21.53, 39.95, "P771"), "cg_ul": (13.61, 59.25, "P779"),
                     "admm_dl": (11.11, 77.40, "P787")}
            fns = {"admm_ul": lambda: dbp.detect_admm(ctx, H7g, y7g, rho=t2.rho, N0=t2.N0, mod="qam64", T=t2.T),
                   "cg_ul": lambda: dbp.detect_cg(ctx, H7g, y7g, rho=t2.N0, mod="qam64", T=t2.T),
                   "admm_dl": lambda: dbp.beamform_admm(ctx, Hd7g, s7g, rho=t2.rho, T=t2.T)}
            table2 = {"workload": "B=1024 (C=32 x S=32), U=16, 64-QAM, N=1200, N_sym=7, T=5 (PAPER.md P803-804)",
                      "paper_hw": "32 x Tesla K40 + Cray Aries MPI (P685, P799), CPU wall clock"}
            ctx.set_option(dbp.OPT_KERNEL_TIMING, 1)
            ctx.kernel_times(reset=True)
            for nm, fn in fns.items():
                ms = timed_fn(fn, 20, flush_k=1)
                pl, pt, cite = paper[nm]
                table2[nm] = {"ms": ms, "mbps": bits7 / (ms * 1e-3) / 1e6, "paper_ms": pl, "paper_mbps": pt,
                              "paper_cite": cite}
            table2["kernels"] = sorted(ctx.kernel_times(reset=True))
            ctx.set_option(dbp.OPT_KERNEL_TIMING, 0)
            del H7g, y7g, Hd7g, s7g

        # per-config entries (BASELINE configs; each solver timed alone, L2 flushed)
        if not args.no_configs:
            configs = {}
            cfgA, cfgB, cfgE = synth.CONFIGS["A"], synth.CONFIGS["B"], synth.CONFIGS["E"]
            HA, yA = gen_frame("ul", cfgA, 0, cfgA.C)
            HB, yB = gen_frame("ul", cfgB, 0, cfgB.C, workers=workers)
            HAg, yAg, HBg, yBg = to(HA), to(yA), to(HB), to(yB)
            entries = [
                ("A", "admm_ul", cfgA, lambda: dbp.detect_admm(ctx, HAg, yAg, rho=cfgA.rho, N0=cfgA.N0,
                                                               mod=cfgA.mod, T=cfgA.T)),
                ("B", "cg_ul", cfgB, lambda: dbp.detect_cg(ctx, HBg, yBg, rho=cfgB.N0, mod=cfgB.mod, T=cfgB.T)),
                ("C", "admm_ul", UL, lambda: solver("admm_ul", UL.T)),
                ("C_cg", "cg_ul", CG, lambda: solver("cg_ul", CG.T)),
                ("D", "admm_dl", DL, lambda: solver("admm_dl", DL.T)),
            ]
            for key, algo, cfg, fn in entries:
                ms = timed_fn(fn, K1)
                configs[key] = {"algo": algo, "ms": ms, "gbps": cfg.bits_per_frame / (ms * 1e-3) / 1e9,
                                "shape": f"C={cfg.C} S={cfg.S} U={cfg.U} N={cfg.N} {cfg.mod} T={cfg.T}"}
            del HAg, yAg, HBg, yBg
            # config E: one GPU's share at G = 8 (C_loc = 16 of 128 clusters, all 4800 subcarriers); the
            # compute of the share only -- the allreduce of the 8-GPU run is not included
            Ce = cfgE.C // 8
            HE, yE = gen_frame("ul", cfgE, 0, Ce, workers=workers)
            HEg, yEg = to(HE), to(yE)
            del HE, yE
            shareE = cfgE.scaled(C=Ce)
            for key, algo, fn in (("E_share_admm_ul", "admm_ul",
                                   lambda: dbp.detect_admm(ctx, HEg, yEg, rho=cfgE.rho, N0=cfgE.N0, mod=cfgE.mod,
                                                           T=cfgE.T)),
                                  ("E_share_cg_ul", "cg_ul",
                                   lambda: dbp.detect_cg(ctx, HEg, yEg, rho=cfgE.N0, mod=cfgE.mod, T=cfgE.T))):
                ms = timed_fn(fn, 20)
                configs[key] = {"algo": algo, "ms": ms, "gbps": cfgE.bits_per_frame / (ms * 1e-3) / 1e9,
                                "shape": f"per-GPU share of E at G=8: C_loc={Ce} (C=128) S=32 U=32 N=4800 "
                                         f"{cfgE.mod} T={cfgE.T}; gbps = the whole frame's bits / this GPU's "
                                         f"compute time (no allreduce)"}
            # the same share on the split path (what each rank runs at G = 8): the per-round iteration kernel
            # against the HBM roofline (north star: >= 60% in the iteration kernel).  Algorithmic bytes of
            # one ADMM round at gamma = 1 (w-only state): packed rho B^{-1} + y^reg + w read + w written per
            # pair (4992 B at UP = 32); the init round (t = 1) reads y^reg and writes w only
            ctx.set_option(dbp.OPT_FORCE_SPLIT, 1)
            for _ in range(2):
                dbp.detect_admm(ctx, HEg, yEg, rho=cfgE.rho, N0=cfgE.N0, mod=cfgE.mod, T=cfgE.T)
            ctx.sync()
            ctx.set_option(dbp.OPT_KERNEL_TIMING, 1)
            ctx.kernel_times(reset=True)
            for _ in range(10):
                flush_l2(0)
                dbp.detect_admm(ctx, HEg, yEg, rho=cfgE.rho, N0=cfgE.N0, mod=cfgE.mod, T=cfgE.T)
            ctx.sync()
            ktE = ctx.kernel_times(reset=True)
            ctx.set_option(dbp.OPT_KERNEL_TIMING, 0)
            ctx.set_option(dbp.OPT_FORCE_SPLIT, 0)
            if "admm_step" in ktE:
                cnt, tot = ktE["admm_step"]
                pairs = Ce * cfgE.N
                upE = 32
                rnd = pairs * (upE * (upE + 1) // 2 * 8 + 3 * upE * 8) + 2 * cfgE.N * upE * 8
                ini = pairs * 2 * upE * 8 + cfgE.N * upE * 8
                avg_bytes = (ini + (cfgE.T - 1) * rnd) / cfgE.T
                us = 1e3 * tot / max(cnt, 1)
                gbs = avg_bytes / (us * 1e-6) / 1e9
                hbm = float(peaks_hbm()) if peaks_hbm() else 6550.0
                configs["E_share_iteration_kernel"] = {
                    "kernel": "admm_step (k_admm_it, one launch per consensus round, split path)",
                    "avg_us": us, "algorithmic_bytes": avg_bytes, "achieved_GBps": gbs, "peak_GBps": hbm,
                    "frac": gbs / hbm, "shape": f"C_loc={Ce} S=32 U=32 N={cfgE.N}, T={cfgE.T} launches per call "
                                                "(init + 4 rounds), L2 flushed before each call"}
            del HEg, yEg
            _ = shareE

    # median and p95 of the step latency (and of each solver's, sequential region), max over ranks
    def pct(v):
        v = np.asarray(v, dtype=float)
        return [float(np.median(v)), float(np.percentile(v, 95))]
    lat = {"step": dict(zip(("median", "p95"), mx(pct(step_list)).tolist()))}
    for i, nm in enumerate(ORDER):
        lat[nm] = dict(zip(("median", "p95"), mx(pct(seq_steps[:, i])).tolist()))
    total_ms = float(per.sum())
    ms_seq = total_ms / args.steps
    ms_step = float(mx([conc_ms])[0]) / args.steps
    value = BITS_PER_STEP / (ms_step * 1e-3) / 1e9
    solvers = {}
    for i, nm in enumerate(ORDER):
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
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        Hh, yh, Hch, ych, Hdh, sh = pin(H), pin(y), pin(Hc), pin(yc), pin(Hd), pin(s)
        o1 = torch.empty(tuple(s_hat.shape), dtype=torch.complex64).pin_memory().numpy()
        o2 = torch.empty(tuple(hard.shape), dtype=torch.uint8).pin_memory().numpy()
        o3 = torch.empty(tuple(s_hat.shape), dtype=torch.complex64).pin_memory().numpy()
        o4 = torch.empty(tuple(hard.shape), dtype=torch.uint8).pin_memory().numpy()
        o5 = torch.empty(tuple(xbf.shape), dtype=torch.complex64).pin_memory().numpy()

        def e2e_step():
            dbp.detect_admm(ctx, Hh, yh, rho=UL.rho, N0=UL.N0, mod=UL.mod, T=UL.T, s_hat=o1, hard=o2)
            dbp.beamform_admm(ctx, Hdh, sh, rho=DL.rho, T=DL.T, x=o5)
            dbp.detect_cg(ctx, Hch, ych, rho=CG.N0, mod=CG.mod, T=CG.T, x_hat=o3, hard=o4)

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier()
        dt = float(mx([time.perf_counter() - t0])[0]) / args.e2e_steps
        h2d = Hh.nbytes + yh.nbytes + Hch.nbytes + ych.nbytes + Hdh.nbytes + sh.nbytes
        d2h = o1.nbytes + o2.nbytes + o3.nbytes + o4.nbytes + o5.nbytes
        e2e = {"value": BITS_PER_STEP / dt / 1e9, "unit": "Gbit/s", "ms_per_step": dt * 1e3,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "how": "same C-ABI calls on pinned host numpy buffers; library stages H2D/D2H on the stream; "
                      "host wall clock, max over ranks"}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()
        if gpu_sample is not None:
            parity = parity_report(gpu_sample)

    if rank == 0:
        launches = st1["kernel_launches"] - st0["kernel_launches"]
        line = {"metric": METRIC, "value": value, "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_sequential": ms_seq,
                "latency_ms": {"how": "median / p95 over the K timed steps (step: the scheduled step; solvers: the "
                               "sequential region), max over ranks", **lat},
                "schedule": (("one stream: " if len(plan) == 1 else "concurrent, one stream per lane: ")
                             + " | ".join(" then ".join(l) for l in plan)
                             + ("; a solver may start in its lane predecessor's last wave (DBP_OPT_OVERLAP_PREV)"
                                if overlap else "")
                             if concurrent else "sequential on one stream"),
                "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32",
                "dtype_note": "fp32 storage and arithmetic; CG-UL's cluster-summed Gram runs on fp16 tensor cores as an "
                              "exact power-of-two-scaled hi/lo split with fp32 accumulation (~2^-22 relative; see "
                              "parity)",
                "data": "synthetic (seeded Philox-4x32: i.i.d. Rayleigh "
                "CN(0,1) channels, uniform Gray QAM, AWGN)", "config": workload_config(world),
                "solvers": solvers, "configs": configs, "centralized_baselines": baselines or None,
                "paper_table2_context": table2, "multi_gpu": multi,
                "roofline": roof, "cpu_baseline": cpu, "parity": parity, "e2e": e2e,
                "per_iter_split_us": split_iter,
                "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
                "consensus_rounds_per_step": (st1["consensus_rounds"] - st0["consensus_rounds"]) / args.steps,
                "allreduce_calls_per_step": (st1["allreduce_calls"] - st0["allreduce_calls"]) / args.steps,
                "kernels": kern, "clocks": clocks}
        print(json.dumps(line), flush=True)
    ctx.close()
    for ex in _POOL.values():
        ex.shutdown(wait=False, cancel_futures=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
