"""Per-kernel device times (library event timing) for one solver on a config."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_04458_b200 import dbp, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--solver", default="admm")
ap.add_argument("--config", default="C")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--T", type=int, default=0)
ap.add_argument("--nofused", type=int, default=0)
ap.add_argument("--nsym", type=int, default=0)
ap.add_argument("--N", type=int, default=0)
ap.add_argument("--C", type=int, default=0)
ap.add_argument("--cgtc", type=int, default=1, help="DBP_OPT_CG_TENSOR")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.T:
    cfg = cfg.scaled(T=a.T)
if a.nsym:
    cfg = cfg.scaled(N_sym=a.nsym)
if a.N:
    cfg = cfg.scaled(N=a.N)
if a.C:
    cfg = cfg.scaled(C=a.C)
ctx = dbp.Context(0)
ctx.set_option(dbp.OPT_FORCE_SPLIT, a.split)
ctx.set_option(dbp.OPT_NO_FUSED, a.nofused)
ctx.set_option(dbp.OPT_CG_TENSOR, a.cgtc)
if a.solver == "bf":
    Hd, s = synth.downlink_frame(cfg)
    Hd, s = torch.from_numpy(Hd).cuda(), torch.from_numpy(s).cuda()
    run = lambda: dbp.beamform_admm(ctx, Hd, s, rho=cfg.rho, T=cfg.T)
else:
    H, y, _ = synth.uplink_frame(cfg)
    H, y = torch.from_numpy(H).cuda(), torch.from_numpy(y).cuda()
    if a.solver == "admm":
        run = lambda: dbp.detect_admm(ctx, H, y, rho=cfg.rho, N0=cfg.N0, mod=cfg.mod, T=cfg.T)
    else:
        run = lambda: dbp.detect_cg(ctx, H, y, rho=cfg.N0, mod=cfg.mod, T=cfg.T)
for _ in range(3):
    run()
ctx.sync()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ctx.set_option(dbp.OPT_KERNEL_TIMING, 1)
ctx.kernel_times(reset=True)
for _ in range(a.reps):
    flush.fill_(1)
    flush.view(torch.int64).sum()
    run()
kt = ctx.kernel_times(reset=True)
print(a.solver, a.config, f"T={cfg.T}", {k: round(v[1] / v[0] * 1e3, 1) for k, v in kt.items()}, "us")
