"""Uncoded BER harness (the methodology of Fig. 2 / Fig. 3,
P628-676, on the i.i.d. Rayleigh substitute channel, SPEC S471-488).

Runs the library's GPU solvers (the product path, through the C ABI) on seeded
synthetic frames over an SNR sweep and counts uncoded bit errors against the
transmitted Gray labels:
  uplink:   ADMM-UL (T = 1, 2, 3, 5), CG-UL (T = 1, 2, 3, 5), centralized MMSE-UL
  downlink: ADMM-DL (T = 1, 2, 3, 5) and centralized ZF-DL; the user side
            receives y = sum_c H_c^d x_c + n (eq. (2), P172), n ~ CN(0, N0_dl),
            and slices y.  Downlink SNR is the per-user Es/N0 of the
            unit-energy symbols, N0_dl = 10^(-SNR/10) (ZF delivers y = s + n);
            uplink SNR follows the configs, N0 = U Es 10^(-SNR/10).
usage: python scripts/ber_harness.py [--out FILE] [--N 300]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1702_04458_b200 import synth  # noqa: E402

BPS = {"bpsk": 1, "qpsk": 2, "qam16": 4, "qam64": 6}


def _bit_errors(a: np.ndarray, b: np.ndarray) -> int:
    x = np.bitwise_xor(a.astype(np.uint8), b.astype(np.uint8))
    return int(np.unpackbits(x[..., None], axis=-1).sum())


def ber_sweep(dbp, ctx, torch, ul_cfg, dl_cfg, snrs, Ts=(1, 2, 3, 5)):
    """-> {"uplink": {name: [ber per snr]}, "downlink": {...}, "snr_db": snrs}"""
    out = {"snr_db": list(snrs), "uplink": {}, "downlink": {}, "bits_per_point": {}}
    dev = "cuda"
    for k, snr in enumerate(snrs):
        cfg = ul_cfg.scaled(snr_db=snr, seed=ul_cfg.seed + 1000 * k)
        H, y, s = synth.uplink_frame(cfg)
        truth = dbp.slice_bits(ctx, torch.from_numpy(s.astype(np.complex64)).to(dev), cfg.mod).cpu().numpy()
        nbits = truth.size * BPS[cfg.mod]
        out["bits_per_point"]["uplink"] = nbits
        Hg, yg = torch.from_numpy(H).to(dev), torch.from_numpy(y).to(dev)
        runs = {}
        for T in Ts:
            runs[f"admm_T{T}"] = lambda T=T: dbp.detect_admm(ctx, Hg, yg, N0=cfg.N0, mod=cfg.mod, T=T)[1]
            runs[f"cg_T{T}"] = lambda T=T: dbp.detect_cg(ctx, Hg, yg, rho=cfg.N0, mod=cfg.mod, T=T)[1]
        runs["mmse"] = lambda: dbp.detect_mmse(ctx, Hg, yg, N0=cfg.N0, mod=cfg.mod)[1]
        for name, fn in runs.items():
            hard = fn()
            ctx.sync()
            out["uplink"].setdefault(name, []).append(_bit_errors(hard.cpu().numpy(), truth) / nbits)

        dcfg = dl_cfg.scaled(snr_db=snr, seed=dl_cfg.seed + 1000 * k)
        Hd, sd = synth.downlink_frame(dcfg)
        truth_d = dbp.slice_bits(ctx, torch.from_numpy(sd).to(dev), dcfg.mod).cpu().numpy()
        nbits_d = truth_d.size * BPS[dcfg.mod]
        out["bits_per_point"]["downlink"] = nbits_d
        Hdg, sdg = torch.from_numpy(Hd).to(dev), torch.from_numpy(sd).to(dev)
        rng = np.random.default_rng(dcfg.seed)
        n0_dl = 10.0 ** (-snr / 10.0)
        noise = np.sqrt(n0_dl / 2) * (rng.standard_normal(sd.shape) + 1j * rng.standard_normal(sd.shape))
        druns = {f"bf_T{T}": (lambda T=T: dbp.beamform_admm(ctx, Hdg, sdg, T=T)) for T in Ts}
        druns["zf"] = lambda: dbp.precode_zf(ctx, Hdg, sdg)
        for name, fn in druns.items():
            x = fn()
            ctx.sync()
            # y = sum_c H_c^d x_c + n  (eq. (2), P172) -- the users' receive vectors
            yd = torch.einsum("cnus,cnjs->nju", Hdg, x).cpu().numpy() + noise
            hard = dbp.slice_bits(ctx, torch.from_numpy(yd.astype(np.complex64)).to(dev), dcfg.mod).cpu().numpy()
            out["downlink"].setdefault(name, []).append(_bit_errors(hard, truth_d) / nbits_d)
    return out


def default_configs(N=300):
    ul = synth.Config("ber-ul", "admm_ul", C=8, S=16, U=16, N=N, mod="qam16", seed=1702047000)
    dl = synth.Config("ber-dl", "admm_dl", C=8, S=16, U=16, N=N, mod="qam16", seed=1702048000)
    return ul, dl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--N", type=int, default=300)
    a = ap.parse_args()
    import torch
    from paper_1702_04458_b200 import dbp
    ctx = dbp.Context(device=0)
    ul, dl = default_configs(a.N)
    res = ber_sweep(dbp, ctx, torch, ul, dl, [4, 8, 12, 16, 20])
    res["config"] = {"uplink": f"U={ul.U} S={ul.S} C={ul.C} B={ul.B} N={ul.N} {ul.mod}",
                     "downlink": f"U={dl.U} S={dl.S} C={dl.C} B={dl.B} N={dl.N} {dl.mod}",
                     "channel": "i.i.d. Rayleigh CN(0,1), perfect CSI (SPEC S88)", "rho": 1.0, "gamma": 1.0}
    txt = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
