"""world_size-2 gloo coverage of the N > 1 path (no GPU).

libdbp shards clusters over ranks and exchanges only the N x N_sym x U
consensus partial sums by an allreduce per round (P744-746).
These tests run that exact dataflow in fp64 on CPU -- rank-local clusters,
one gloo allreduce of the partial sum per consensus round, replicated prox /
CG updates on every rank -- and check that it reproduces the single-process
oracle (which sums all C clusters itself), plus the bench's host logic:
sharded input generation, the NCCL unique-id broadcast pattern and the
max-over-ranks timing reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1702_04458_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _admm_ul_rank(H, y, C, rho, N0, Es, T):
    """Split-path ADMM-UL (Alg. 1) for this rank's clusters; returns s_hat [N][J][U]."""
    Cl, N, S, U = H.shape
    J = y.shape[2]
    Hd = H.astype(np.complex128)
    Binv = np.linalg.inv(np.einsum("cnsu,cnsv->cnuv", Hd.conj(), Hd) + rho * np.eye(U))
    yreg = np.einsum("cnuv,cnjv->cnju", Binv, np.einsum("cnsu,cnjs->cnju", Hd.conj(), y.astype(np.complex128)))
    lam = np.zeros_like(yreg)
    z = yreg.copy()
    w = _allreduce(z.sum(axis=0))                                 # init consensus
    s = w / (N0 / (rho * Es) + C)
    for _ in range(2, T + 1):
        lam = lam + (z - s[None])
        z = yreg + rho * np.einsum("cnuv,cnjv->cnju", Binv, s[None] - lam)
        w = _allreduce((z + lam).sum(axis=0))                     # one allreduce per round
        s = w / (N0 / (rho * Es) + C)
    return s


def _cg_rank(H, y, rho, T):
    Hd = H.astype(np.complex128)
    r = _allreduce(np.einsum("cnsu,cnjs->nju", Hd.conj(), y.astype(np.complex128)))   # y^MRC
    p = r.copy()
    x = np.zeros_like(r)
    for _ in range(T):
        w = _allreduce(np.einsum("cnsu,cnsv,njv->nju", Hd.conj(), Hd, p))
        e = rho * p + w
        rr = np.sum(np.abs(r) ** 2, axis=-1, keepdims=True)
        live = rr > 0
        alpha = np.where(live, rr / np.where(live, np.real(np.sum(p.conj() * e, -1, keepdims=True)), 1), 0)
        x = x + alpha * p
        rn = r - alpha * e
        rr1 = np.sum(np.abs(rn) ** 2, axis=-1, keepdims=True)
        beta = np.where(live, rr1 / np.where(live, rr, 1), 0)
        p = np.where(live, rn + beta * p, p)
        r = np.where(live, rn, r)
    return x


def _bf_rank(Hd, s, C, S, rho, T):
    Hx = Hd.astype(np.complex128)
    U = Hx.shape[2]
    Binv = np.linalg.inv(np.einsum("cnus,cnvs->cnuv", Hx, Hx.conj()) + np.eye(U) / rho)
    sv = s.astype(np.complex128)
    z = np.broadcast_to(max(U / (C * S), 1 / C) * sv[None], (Hx.shape[0],) + sv.shape).copy()
    lam = np.zeros_like(z)
    x = np.einsum("cnus,cnuv,cnjv->cnjs", Hx.conj(), Binv, z + lam)
    for _ in range(2, T + 1):
        m = np.einsum("cnus,cnjs->cnju", Hx, x)
        wc = m - lam
        w = _allreduce(wc.sum(axis=0))
        z = wc + (sv - w)[None] / C
        lam = lam - (m - z)
        x = np.einsum("cnus,cnuv,cnjv->cnjs", Hx.conj(), Binv, z + lam)
    return x


def _central_rank(H, y, N0, Hd, s):
    """Centralized baselines, rank-local Gram sums + ONE allreduce of [Gram | matched filter]."""
    Hx = H.astype(np.complex128)
    G = _allreduce(np.einsum("cnsu,cnsv->nuv", Hx.conj(), Hx))
    b = _allreduce(np.einsum("cnsu,cnjs->nju", Hx.conj(), y.astype(np.complex128)))
    x = np.linalg.solve(G + N0 * np.eye(G.shape[-1]), b.transpose(0, 2, 1)).transpose(0, 2, 1)
    Hdx = Hd.astype(np.complex128)
    B = _allreduce(np.einsum("cnus,cnvs->nuv", Hdx, Hdx.conj()))
    r = np.linalg.solve(B, s.astype(np.complex128).transpose(0, 2, 1)).transpose(0, 2, 1)
    xz = np.einsum("cnus,nju->cnjs", Hdx.conj(), r)                       # rank-local x_c
    return x, xz


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        cfg = synth.CONFIGS["C"].scaled(N=6, C=4, N_sym=2)
        c0, c1 = synth.cluster_range(cfg.C, rank, world)
        H, y, _ = synth.uplink_frame(cfg, c0, c1)
        out["s"] = _admm_ul_rank(H, y, cfg.C, cfg.rho, cfg.N0, 1.0, cfg.T)
        out["x"] = _cg_rank(H, y, cfg.N0, cfg.T)
        dcfg = synth.CONFIGS["D"].scaled(N=5, C=4)
        d0, d1 = synth.cluster_range(dcfg.C, rank, world)
        Hd, s = synth.downlink_frame(dcfg, d0, d1)
        out["bf"] = _bf_rank(Hd, s, dcfg.C, dcfg.S, dcfg.rho, dcfg.T)
        out["shard"] = (c0, c1)
        out["mmse"], out["zf"] = _central_rank(H, y, cfg.N0, Hd, s)
        # bench bootstrap: rank 0's id reaches every rank; device time is max over ranks
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        out["uid_ok"] = obj[0] == bytes(range(128))
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["tmax"] = float(t)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def two_rank_results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_split_dataflow_matches_oracle(two_rank_results, oracle_mod):
    cfg = synth.CONFIGS["C"].scaled(N=6, C=4, N_sym=2)
    H, y, _ = synth.uplink_frame(cfg)
    s_ref, _ = oracle_mod.detect_admm(H, y, rho=cfg.rho, N0=cfg.N0, mod=cfg.mod, T=cfg.T)
    x_ref, _ = oracle_mod.detect_cg(H, y, rho=cfg.N0, mod=cfg.mod, T=cfg.T)
    for r in (0, 1):   # replicated outputs, identical on both ranks
        assert np.allclose(two_rank_results[r]["s"], s_ref, atol=1e-10, rtol=0)
        assert np.allclose(two_rank_results[r]["x"], x_ref, atol=1e-10, rtol=0)
    dcfg = synth.CONFIGS["D"].scaled(N=5, C=4)
    Hd, s = synth.downlink_frame(dcfg)
    x_bf = oracle_mod.beamform_admm(Hd, s, rho=dcfg.rho, T=dcfg.T)
    got = np.concatenate([two_rank_results[0]["bf"], two_rank_results[1]["bf"]], axis=0)   # rank-local x_c
    assert np.allclose(got, x_bf, atol=1e-10, rtol=0)


def test_bootstrap_host_logic(two_rank_results):
    assert two_rank_results[0]["shard"] == (0, 2) and two_rank_results[1]["shard"] == (2, 4)
    assert two_rank_results[0]["uid_ok"] and two_rank_results[1]["uid_ok"]
    assert two_rank_results[0]["tmax"] == two_rank_results[1]["tmax"] == 2.0


def test_centralized_dataflow_matches_oracle(two_rank_results, oracle_mod):
    cfg = synth.CONFIGS["C"].scaled(N=6, C=4, N_sym=2)
    H, y, _ = synth.uplink_frame(cfg)
    x_ref, _ = oracle_mod.mmse_centralized(H, y, N0=cfg.N0)
    for r in (0, 1):
        assert np.allclose(two_rank_results[r]["mmse"], x_ref, atol=1e-10, rtol=0)
    dcfg = synth.CONFIGS["D"].scaled(N=5, C=4)
    Hd, s = synth.downlink_frame(dcfg)
    got = np.concatenate([two_rank_results[0]["zf"], two_rank_results[1]["zf"]], axis=0)
    assert np.allclose(got, oracle_mod.zf_centralized(Hd, s), atol=1e-10, rtol=0)
