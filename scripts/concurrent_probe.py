"""Step time of the bench workload (configs C + D, T = 5): the three solvers back to back on one
stream vs. the uplink pair on one stream and the downlink solver on a second, concurrently
(the DL kernel's CTAs fill the UL kernels' wave tails).  L2 flushed between steps, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_04458_b200 import dbp, synth  # noqa: E402

UL, DL = synth.CONFIGS["C"], synth.CONFIGS["D"]
ctx = dbp.Context(0)
H, y, _ = synth.uplink_frame(UL)
Hd, s = synth.downlink_frame(DL)
Hg, yg, Hdg, sg = (torch.from_numpy(a).cuda() for a in (H, y, Hd, s))
main = torch.cuda.current_stream()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty((), dtype=torch.int64, device="cuda")
outs = {}


def ul(st):
    outs["a"] = dbp.detect_admm(ctx, Hg, yg, rho=UL.rho, N0=UL.N0, mod=UL.mod, T=UL.T, stream=st.cuda_stream)
    outs["c"] = dbp.detect_cg(ctx, Hg, yg, rho=UL.N0, mod=UL.mod, T=UL.T, stream=st.cuda_stream)


def dl(st):
    outs["b"] = dbp.beamform_admm(ctx, Hdg, sg, rho=DL.rho, T=DL.T, stream=st.cuda_stream)


def step(conc):
    if not conc:
        ul(main)
        dl(main)
        return
    e = torch.cuda.Event()
    e.record(main)
    sa.wait_event(e)
    sb.wait_event(e)
    ul(sa)
    dl(sb)
    ea, eb = torch.cuda.Event(), torch.cuda.Event()
    ea.record(sa)
    eb.record(sb)
    main.wait_event(ea)
    main.wait_event(eb)


for conc in (False, True, False, True):
    for _ in range(5):
        step(conc)
    torch.cuda.synchronize()
    tot = 0.0
    K = 50
    for k in range(K):
        flush.fill_(k & 0xFF)
        torch.sum(flush.view(torch.int64), dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        step(conc)
        e1.record(main)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    print("concurrent" if conc else "sequential", f"{tot / K * 1e3:.1f} us/step")
