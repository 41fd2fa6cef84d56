"""The real library at world 2 on one GPU: two processes, each a rank of the cluster-partitioned
path (its own contiguous block of clusters, P149-155), with a true per-round consensus exchange
-- the partial sums cross processes through the library's host allreduce hook
(dbp_set_allreduce_hook) over torch.distributed gloo, in place of NCCL (NCCL refuses two ranks
on one device).  Every other part is the world > 1 product path: partition, per-round launches,
round / collective counts, replicated updates.  Checked against the fp64 oracle (the paper's
bar), against a world-1 solve (rel-L2 <= 1e-5, SURVEY 8(c) "across GPU counts") and rank
against rank (bitwise identical replicated outputs)."""
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_1702_04458_b200 import synth

pytestmark = pytest.mark.gpu

CASES = {
    "C": synth.CONFIGS["C"].scaled(N=24),
    "Cj3": synth.CONFIGS["C"].scaled(N=10, N_sym=3, mod="qam16"),
    "ss": synth.Config("ss", "admm_ul", C=6, S=8, U=16, N=12, mod="qam16", snr_db=20),   # S x S form
    # UP = 32 (config E's users): staged split-path rounds and the tensor-core G_loc at UP = 32
    "u32": synth.CONFIGS["E"].scaled(N=6, C=4),
}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_1702_04458_b200 import dbp
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = dbp.Context(device=0, rank=rank, world=world, unique_id=None)

    def hook(arr):
        t = torch.from_numpy(arr)
        dist.all_reduce(t)                       # sum over ranks, identical bits everywhere

    ctx.set_allreduce_hook(hook)
    res = {}
    for name, cfg in CASES.items():
        c0, c1 = synth.cluster_range(cfg.C, rank, world)
        H, y, _ = synth.uplink_frame(cfg, c0, c1)
        Hd, s = synth.downlink_frame(cfg.scaled(algo="admm_dl"), c0, c1)
        Hg, yg, Hdg, sg = (torch.from_numpy(a).cuda() for a in (H, y, Hd, s))
        regs = ["mmse", "box"] if name == "C" else ["mmse"]
        for reg in regs:
            st0 = ctx.stats()
            sh, hard = dbp.detect_admm(ctx, Hg, yg, rho=cfg.rho, N0=cfg.N0, reg=reg, mod=cfg.mod, T=cfg.T)
            ctx.sync()
            st1 = ctx.stats()
            res[f"{name}_admm_{reg}"] = sh.cpu().numpy()
            res[f"{name}_admm_{reg}_hard"] = hard.cpu().numpy()
            res[f"{name}_admm_{reg}_calls"] = np.array(st1["allreduce_calls"] - st0["allreduce_calls"])
        st0 = ctx.stats()
        xh, _ = dbp.detect_cg(ctx, Hg, yg, rho=cfg.N0, mod=cfg.mod, T=cfg.T)
        ctx.sync()
        st1 = ctx.stats()
        res[f"{name}_cg"] = xh.cpu().numpy()
        res[f"{name}_cg_calls"] = np.array(st1["allreduce_calls"] - st0["allreduce_calls"])
        x = dbp.beamform_admm(ctx, Hdg, sg, rho=cfg.rho, T=cfg.T, eps=0.1 if name == "C" else 0.0)
        ctx.sync()
        st2 = ctx.stats()
        res[f"{name}_bf"] = x.cpu().numpy()
        res[f"{name}_bf_calls"] = np.array(st2["allreduce_calls"] - st1["allreduce_calls"])
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    ctx.close()
    dist.destroy_process_group()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def two_ranks():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    out = tempfile.mkdtemp(prefix="dbp_w2_")
    mp.start_processes(_rank_main, args=(2, _port(), out), nprocs=2, join=True, start_method="spawn")
    return [dict(np.load(os.path.join(out, f"rank{r}.npz"))) for r in range(2)]


@pytest.mark.parametrize("name", list(CASES))
def test_world2_matches_oracle_and_world1(two_ranks, name):
    import oracle
    import torch

    from paper_1702_04458_b200 import dbp
    cfg = CASES[name]
    r0, r1 = two_ranks
    H, y, _ = synth.uplink_frame(cfg)
    Hd, s = synth.downlink_frame(cfg.scaled(algo="admm_dl"))
    ctx = dbp.Context(device=0)
    Hg, yg, Hdg, sg = (torch.from_numpy(a).cuda() for a in (H, y, Hd, s))
    T = cfg.T
    for reg in (["mmse", "box"] if name == "C" else ["mmse"]):
        k = f"{name}_admm_{reg}"
        assert np.array_equal(r0[k], r1[k]) and np.array_equal(r0[k + "_hard"], r1[k + "_hard"])
        s_ref, _ = oracle.detect_admm(H, y, rho=cfg.rho, N0=cfg.N0, reg=reg, mod=cfg.mod, T=T)
        assert rel(r0[k], s_ref) < 1e-4
        s1, _ = dbp.detect_admm(ctx, Hg, yg, rho=cfg.rho, N0=cfg.N0, reg=reg, mod=cfg.mod, T=T)
        assert rel(r0[k], s1.cpu().numpy()) < 1e-5
        assert int(r0[k + "_calls"]) == T                            # one allreduce per round (P311)
    k = f"{name}_cg"
    assert np.array_equal(r0[k], r1[k])
    x_ref, _ = oracle.detect_cg(H, y, rho=cfg.N0, mod=cfg.mod, T=T)
    assert rel(r0[k], x_ref) < 1e-4
    x1, _ = dbp.detect_cg(ctx, Hg, yg, rho=cfg.N0, mod=cfg.mod, T=T)
    assert rel(r0[k], x1.cpu().numpy()) < 1e-5
    assert int(r0[k + "_calls"]) == T + 1                            # y^MRC + one per iteration
    eps = 0.1 if name == "C" else 0.0
    xb = np.concatenate([r0[f"{name}_bf"], r1[f"{name}_bf"]])         # rank-local x_c, clusters in order
    assert rel(xb, oracle.beamform_admm(Hd, s, rho=cfg.rho, T=T, eps=eps)) < 1e-4
    b1 = dbp.beamform_admm(ctx, Hdg, sg, rho=cfg.rho, T=T, eps=eps)
    ctx.sync()
    assert rel(xb, b1.cpu().numpy()) < 1e-5
    assert int(r0[f"{name}_bf_calls"]) == T - 1
    ctx.close()
