"""Read-bandwidth references for one config-C channel tensor (157 MB): torch reductions over it,
L2 flushed before each (device events)."""
import torch

x = torch.randn(32 * 1200 * 32 * 16 * 2, device="cuda")          # config C H as floats
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty((), device="cuda")
for name, fn in {"sum": lambda: x.sum(), "amax": lambda: torch.amax(x.view(-1, 1024), dim=1)}.items():
    for _ in range(3):
        fn()
    ts = []
    for _ in range(20):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    ts.sort()
    print(f"{name}: {ts[len(ts) // 2]:.1f} us median, {x.numel() * 4 / ts[len(ts) // 2] / 1e3:.0f} GB/s")
