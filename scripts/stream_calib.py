"""Calibrate plain HBM streaming of the config-C channel (torch kernels) vs libdbp's Gram kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_04458_b200 import synth  # noqa: E402

H, y, _ = synth.uplink_frame(synth.CONFIGS["C"])
Hg = torch.from_numpy(H).cuda()
x = torch.view_as_real(Hg).reshape(-1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
for name, fn in [("sum", lambda: x.sum()), ("copy", lambda: out.copy_(x))]:
    for _ in range(3):
        fn()
    ts = []
    for _ in range(10):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    nbytes = x.numel() * 4 * (2 if name == "copy" else 1)
    print(f"{name}: {ms*1e3:.1f} us  {nbytes/ms/1e6:.0f} GB/s")
