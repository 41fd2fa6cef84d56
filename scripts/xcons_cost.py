"""Fused ADMM-UL / ADMM-DL time with and without the device-side consensus exchange (self-peer, world 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_04458_b200 import dbp, synth  # noqa: E402

cfg = synth.CONFIGS["C"]
ctx = dbp.Context(0)
H, y, _ = synth.uplink_frame(cfg)
Hd, s = synth.downlink_frame(synth.CONFIGS["D"])
H, y, Hd, s = (torch.from_numpy(v).cuda() for v in (H, y, Hd, s))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fns = {"admm_ul": lambda: dbp.detect_admm(ctx, H, y, N0=cfg.N0, mod=cfg.mod, T=cfg.T),
       "admm_dl": lambda: dbp.beamform_admm(ctx, Hd, s, T=cfg.T)}
for mode in (0, 2):
    ctx.set_option(dbp.OPT_DEVICE_CONSENSUS, mode)
    for nm, fn in fns.items():
        fn()
        ctx.sync()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
        for e0, e1 in ev:
            flush.fill_(1)
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        print(f"device_consensus={mode} {nm}: {sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1e3:.1f} us")
