"""Per-kernel times of the three solvers at the paper's Table II workload (N_sym = 7, 64-QAM, B = 1024)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_04458_b200 import dbp, synth  # noqa: E402

cfg = synth.CONFIGS["C"].scaled(N_sym=7)
ctx = dbp.Context(0)
H, y, _ = synth.uplink_frame(cfg)
Hd, s = synth.downlink_frame(cfg.scaled(algo="admm_dl"))
H, y, Hd, s = (torch.from_numpy(v).cuda() for v in (H, y, Hd, s))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for nm, fn in {"admm_ul": lambda: dbp.detect_admm(ctx, H, y, N0=cfg.N0, mod="qam64", T=5),
               "cg_ul": lambda: dbp.detect_cg(ctx, H, y, rho=cfg.N0, mod="qam64", T=5),
               "admm_dl": lambda: dbp.beamform_admm(ctx, Hd, s, T=5)}.items():
    fn()
    ctx.sync()
    ctx.set_option(dbp.OPT_KERNEL_TIMING, 1)
    ctx.kernel_times(reset=True)
    for _ in range(10):
        flush.fill_(1)
        fn()
    kt = ctx.kernel_times(reset=True)
    ctx.set_option(dbp.OPT_KERNEL_TIMING, 0)
    print(nm, {k: round(v[1] / v[0] * 1e3, 1) for k, v in kt.items()}, "us")
