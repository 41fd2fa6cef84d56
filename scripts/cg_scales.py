"""k_cg_tc vs the FP32 CG paths and the fp64 oracle on clusters at powers of two apart."""
import numpy as np, torch, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle
from paper_1702_04458_b200 import dbp, synth
torch.zeros(1, device="cuda")
ctx = dbp.Context(0)
cfg = synth.CONFIGS["C"].scaled(N=11, C=8)
for spread in (-40, 24, 0):
    H, y, _ = synth.uplink_frame(cfg)
    f = np.float32(2.0) ** (spread * np.arange(cfg.C) / cfg.C); f = f / f.max()
    H = (H * f[:, None, None, None]).astype(np.complex64); y = (y * f[:, None, None, None]).astype(np.complex64)
    x_ref, _ = oracle.detect_cg(H, y, rho=cfg.N0, mod=cfg.mod, T=cfg.T)
    for path, (sp, nf, tc) in {"tc": (0, 0, 1), "fp32": (0, 0, 0), "two": (0, 1, 0), "split": (1, 0, 0)}.items():
        ctx.set_option(dbp.OPT_FORCE_SPLIT, sp); ctx.set_option(dbp.OPT_NO_FUSED, nf); ctx.set_option(dbp.OPT_CG_TENSOR, tc)
        x, _ = dbp.detect_cg(ctx, torch.from_numpy(H).cuda(), torch.from_numpy(y).cuda(), rho=cfg.N0, mod=cfg.mod, T=cfg.T)
        ctx.sync(); x = x.cpu().numpy()
        print(spread, path, np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))
