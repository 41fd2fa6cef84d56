"""Run one solver on a BASELINE config a few times (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_04458_b200 import dbp, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--solver", default="admm", choices=["admm", "cg", "bf"])
ap.add_argument("--config", default="C")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--C", type=int, default=0)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.C:
    cfg = cfg.scaled(C=a.C)
ctx = dbp.Context(0)
ctx.set_option(dbp.OPT_FORCE_SPLIT, a.split)
if a.solver == "bf":
    Hd, s = synth.downlink_frame(cfg)
    Hd, s = torch.from_numpy(Hd).cuda(), torch.from_numpy(s).cuda()
    for _ in range(a.reps):
        dbp.beamform_admm(ctx, Hd, s, rho=cfg.rho, T=cfg.T)
else:
    H, y, _ = synth.uplink_frame(cfg)
    H, y = torch.from_numpy(H).cuda(), torch.from_numpy(y).cuda()
    for _ in range(a.reps):
        if a.solver == "admm":
            dbp.detect_admm(ctx, H, y, rho=cfg.rho, N0=cfg.N0, mod=cfg.mod, T=cfg.T)
        else:
            dbp.detect_cg(ctx, H, y, rho=cfg.N0, mod=cfg.mod, T=cfg.T)
ctx.sync()
print("ok")
