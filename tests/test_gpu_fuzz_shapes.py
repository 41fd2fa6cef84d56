"""Seeded random shapes through every solver and path against the fp64 oracle: C, S, U, N, N_sym,
alphabet and SNR drawn per case inside the library's limits (U <= 32, S <= 64), so the kernels'
shape dispatch (fused / tensor-core / folded / lane-row / split, padding of U and S, partial
cluster blocks and CTAs) is exercised beyond the hand-picked cases of test_gpu_parity.py.  Same
bar: rel-L2 <= 1e-4 over the output and per subcarrier; hard bits exact except at ties."""
import numpy as np
import pytest

from paper_1702_04458_b200 import synth

from .test_gpu_parity import CG_PATHS, PATHS, TOL, check_hard, rel, set_path

pytestmark = pytest.mark.gpu

MODS = ["bpsk", "qpsk", "qam16", "qam64"]


def shapes(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n):
        U = int(rng.integers(1, 33))
        S = int(rng.integers(max(1, U // 2), 65))
        C = int(rng.integers(1, 25))
        N = int(rng.integers(1, 30))
        J = int(rng.choice([1, 1, 1, 2, 3, 7]))
        mod = MODS[int(rng.integers(0, 4))] if U > 1 else "qpsk"
        snr = float(rng.uniform(8.0, 30.0))
        out.append(synth.Config(f"fz{k}", "admm_ul", C=C, S=S, U=U, N=N, N_sym=J, mod=mod, snr_db=snr,
                                T=int(rng.integers(1, 7)), seed=1702049000 + k))
    return out


CASES = shapes(40, 1702)


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    from paper_1702_04458_b200 import dbp
    ctx = dbp.Context(device=0)
    yield dbp, ctx, oracle, torch
    ctx.close()


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: f"{c.name}-C{c.C}S{c.S}U{c.U}N{c.N}J{c.N_sym}{c.mod}T{c.T}")
def test_fuzz_all_solvers(env, cfg):
    dbp, ctx, oracle, torch = env
    H, y, _ = synth.uplink_frame(cfg)
    Hg, yg = torch.from_numpy(H).cuda(), torch.from_numpy(y).cuda()
    s_ref, h_ref = oracle.detect_admm(H, y, rho=cfg.rho, N0=cfg.N0, mod=cfg.mod, T=cfg.T)
    x_ref, hx_ref = oracle.detect_cg(H, y, rho=cfg.N0, mod=cfg.mod, T=cfg.T)
    dl = cfg.scaled(algo="admm_dl")
    Hd, s = synth.downlink_frame(dl)
    Hdg, sg = torch.from_numpy(Hd).cuda(), torch.from_numpy(s).cuda()
    b_ref = oracle.beamform_admm(Hd, s, rho=dl.rho, T=dl.T)
    for path in CG_PATHS:
        set_path(env, path)
        if path != "fp32":
            sh, hd = dbp.detect_admm(ctx, Hg, yg, rho=cfg.rho, N0=cfg.N0, mod=cfg.mod, T=cfg.T)
            xb = dbp.beamform_admm(ctx, Hdg, sg, rho=dl.rho, T=dl.T)
            ctx.sync()
            assert rel(sh.cpu().numpy(), s_ref) < TOL, ("admm", path)
            check_hard(hd.cpu().numpy(), h_ref, s_ref, cfg.mod)
            assert rel(xb.cpu().numpy(), b_ref) < TOL, ("bf", path)
        xh, hx = dbp.detect_cg(ctx, Hg, yg, rho=cfg.N0, mod=cfg.mod, T=cfg.T)
        ctx.sync()
        assert rel(xh.cpu().numpy(), x_ref) < TOL, ("cg", path)
        check_hard(hx.cpu().numpy(), hx_ref, x_ref, cfg.mod)
    set_path(env, "fused")
    assert set(PATHS) <= set(CG_PATHS)
