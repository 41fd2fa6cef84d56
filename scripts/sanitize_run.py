"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck): every solver on
config A and on config C / D shapes at N = 40 (several CTAs, a ragged tail), on the fused,
two-kernel and split paths, plus the centralized baselines and the device-consensus self-peer
mode.  Prints one line per case; the sanitizer's own report is the verdict."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_04458_b200 import dbp, synth  # noqa: E402

ctx = dbp.Context(0)
cases = [synth.CONFIGS["A"], synth.CONFIGS["C"].scaled(N=40), synth.CONFIGS["E"].scaled(N=3, C=8),
         synth.CONFIGS["C"].scaled(N=6, N_sym=3)]
for path in ("fused", "twokernel", "split", "xcons"):
    ctx.set_option(dbp.OPT_FORCE_SPLIT, int(path == "split"))
    ctx.set_option(dbp.OPT_NO_FUSED, int(path == "twokernel"))
    ctx.set_option(dbp.OPT_DEVICE_CONSENSUS, 2 if path == "xcons" else 0)
    for cfg in cases:
        H, y, _ = synth.uplink_frame(cfg)
        Hd, s = synth.downlink_frame(cfg)
        Hg, yg, Hdg, sg = (torch.from_numpy(a).cuda() for a in (H, y, Hd, s))
        dbp.detect_admm(ctx, Hg, yg, rho=cfg.rho, N0=cfg.N0, mod=cfg.mod, T=cfg.T)
        dbp.detect_cg(ctx, Hg, yg, rho=cfg.N0, mod=cfg.mod, T=cfg.T)
        dbp.beamform_admm(ctx, Hdg, sg, rho=cfg.rho, T=cfg.T)
        if path == "fused":
            dbp.detect_mmse(ctx, Hg, yg, N0=cfg.N0, mod=cfg.mod)
            dbp.precode_zf(ctx, Hdg, sg)
        ctx.sync()
        print(path, cfg.name, f"C={cfg.C} U={cfg.U} N={cfg.N} J={cfg.N_sym}", "ok", flush=True)
ctx.close()
