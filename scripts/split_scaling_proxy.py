"""Per-GPU compute of the split (multi-GPU) path at world = G, measured on one GPU: the
rank-local problem has C_loc = C/G clusters, run with DBP_OPT_FORCE_SPLIT (the allreduce is a
no-op at world 1, so this is the compute part only; NCCL latency comes on top).
usage: python scripts/split_scaling_proxy.py [--config C] [--reps 20]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_04458_b200 import dbp, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--gs", default="1,2,4,8", help="world sizes to model")
a = ap.parse_args()
ctx = dbp.Context(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for G in (int(g) for g in a.gs.split(",")):
    cfg = synth.CONFIGS[a.config]
    loc = cfg.scaled(C=cfg.C // G)
    H, y, _ = synth.uplink_frame(loc)
    Hd, s = synth.downlink_frame(loc.scaled(algo="admm_dl"))
    H, y, Hd, s = (torch.from_numpy(v).cuda() for v in (H, y, Hd, s))
    o1, h1 = torch.empty((cfg.N, 1, cfg.U), dtype=torch.complex64, device="cuda"), \
        torch.empty((cfg.N, 1, cfg.U), dtype=torch.uint8, device="cuda")
    o2, h2 = torch.empty_like(o1), torch.empty_like(h1)
    o3 = torch.empty((loc.C, cfg.N, 1, cfg.S), dtype=torch.complex64, device="cuda")
    runs = {"admm_ul": lambda: dbp.detect_admm(ctx, H, y, N0=cfg.N0, mod=cfg.mod, T=cfg.T, s_hat=o1, hard=h1),
            "cg_ul": lambda: dbp.detect_cg(ctx, H, y, rho=cfg.N0, mod=cfg.mod, T=cfg.T, x_hat=o2, hard=h2),
            "admm_dl": lambda: dbp.beamform_admm(ctx, Hd, s, T=cfg.T, x=o3)}
    out = {}
    for split in (0, 1, 2):                      # fused; split (graphs); split, plain launches
        ctx.set_option(dbp.OPT_FORCE_SPLIT, int(split > 0))
        ctx.set_option(dbp.OPT_GRAPHS, int(split != 2))
        for nm, fn in runs.items():
            fn()
            ctx.sync()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
            for e0, e1 in ev:
                flush.fill_(1)
                e0.record()
                fn()
                e1.record()
            torch.cuda.synchronize()
            out[(nm, split)] = sum(e0.elapsed_time(e1) for e0, e1 in ev) / a.reps * 1e3
    ctx.set_option(dbp.OPT_FORCE_SPLIT, 0)
    ctx.set_option(dbp.OPT_GRAPHS, 1)
    print(f"G={G} C_loc={loc.C}: " + ", ".join(f"{nm} fused {out[(nm, 0)]:.1f} split+graphs {out[(nm, 1)]:.1f} "
                                               f"split {out[(nm, 2)]:.1f} us" for nm in runs), flush=True)
