"""Programmatic dependent launch probe: config C/D solvers back to back on one stream, with and
without DBP_OPT_OVERLAP_PREV (independent frames; L2 flushed before each step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_04458_b200 import dbp, synth  # noqa: E402

torch.zeros(1, device="cuda")
ctx = dbp.Context(0)
UL, DL = synth.CONFIGS["C"], synth.CONFIGS["D"]
H, y, _ = synth.uplink_frame(UL)
Hd, s = synth.downlink_frame(DL)
H, y, Hd, s = (torch.from_numpy(a).cuda() for a in (H, y, Hd, s))
H2, y2 = H.clone(), y.clone()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
plans = {"ul,dl": ["ul", "dl"], "ul,dl,cg": ["ul", "dl", "cg"], "cg,ul,dl": ["cg", "ul", "dl"],
         "ul,ul": ["ul", "ul2"]}


def run(nm):
    if nm == "ul":
        dbp.detect_admm(ctx, H, y, rho=UL.rho, N0=UL.N0, mod=UL.mod, T=UL.T)
    elif nm == "ul2":
        dbp.detect_admm(ctx, H2, y2, rho=UL.rho, N0=UL.N0, mod=UL.mod, T=UL.T)
    elif nm == "dl":
        dbp.beamform_admm(ctx, Hd, s, rho=DL.rho, T=DL.T)
    else:
        dbp.detect_cg(ctx, H2, y2, rho=UL.N0, mod=UL.mod, T=UL.T)


for name, seq in plans.items():
    for ov in (0, 1):
        ctx.set_option(dbp.OPT_OVERLAP_PREV, ov)
        for _ in range(5):
            for nm in seq:
                run(nm)
        K = 200
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        torch.cuda.synchronize()
        for e0, e1 in ev:
            flush.fill_(1)
            e0.record()
            for nm in seq:
                run(nm)
            e1.record()
        torch.cuda.synchronize()
        print(f"{name:10s} overlap={ov}: {sum(a.elapsed_time(b) for a, b in ev) / K * 1000:.1f} us")
