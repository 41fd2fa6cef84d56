"""Pins of the centralized baselines in the oracle (NEXT-3; Table I rows
MMSE-UL / ZF-DL, P594-595) against closed forms computed independently
with numpy on the stacked full-array channel, SPEC's worked examples, and the
decentralized algorithms' limits."""
import numpy as np
import pytest

from paper_1702_04458_b200 import synth

from tests.pins import rel


def stacked_ul(H, n, j=0, y=None):
    """Full uplink array at subcarrier n: H (B x U) = [H_1; ...; H_C], y (B)."""
    Hn = np.concatenate([H[c, n].astype(np.complex128) for c in range(H.shape[0])], axis=0)
    yn = None if y is None else np.concatenate([y[c, n, j].astype(np.complex128) for c in range(H.shape[0])])
    return Hn, yn


def stacked_dl(Hd, n):
    """Full downlink matrix at subcarrier n: H (U x B) = [H_1^d, ..., H_C^d]."""
    return np.concatenate([Hd[c, n].astype(np.complex128) for c in range(Hd.shape[0])], axis=1)


@pytest.mark.parametrize("cfg", [synth.CONFIGS["A"], synth.CONFIGS["C"].scaled(N=3, N_sym=2),
                                 synth.Config("s<u", "admm_ul", C=4, S=3, U=6, N=4, mod="qpsk", snr_db=10)])
def test_mmse_equals_regularized_solve(oracle_mod, cfg):
    H, y, _ = synth.uplink_frame(cfg)
    x, _ = oracle_mod.mmse_centralized(H, y, N0=cfg.N0, Es=1.0, mod=cfg.mod)
    for n in range(cfg.N):
        for j in range(cfg.N_sym):
            Hn, yn = stacked_ul(H, n, j, y)
            ref = np.linalg.solve(Hn.conj().T @ Hn + cfg.N0 * np.eye(cfg.U), Hn.conj().T @ yn)   # P212-218
            assert rel(x[n, j], ref) < 1e-11


def test_zf_detection_is_least_squares(oracle_mod):
    cfg = synth.CONFIGS["C"].scaled(N=4)
    H, y, _ = synth.uplink_frame(cfg)
    x, _ = oracle_mod.mmse_centralized(H, y, N0=0.0)
    for n in range(cfg.N):
        Hn, yn = stacked_ul(H, n, 0, y)
        assert rel(x[n, 0], np.linalg.lstsq(Hn, yn, rcond=None)[0]) < 1e-10


def test_mmse_identity_channel(oracle_mod):
    """SPEC S224: H = I_U, N0 = 0 -> x = y."""
    U = 5
    H = np.broadcast_to(np.eye(U, dtype=np.complex64), (1, 3, U, U)).copy()
    rng = np.random.default_rng(1)
    y = (rng.standard_normal((1, 3, 1, U)) + 1j * rng.standard_normal((1, 3, 1, U))).astype(np.complex64)
    x, _ = oracle_mod.mmse_centralized(H, y, N0=0.0)
    assert np.allclose(x[:, 0], y[0, :, 0].astype(np.complex128), atol=1e-12)


def test_decentralized_admm_converges_to_centralized(oracle_mod):
    """SPEC S242: C = 1, MMSE, t_max = 200 -> mmse_centralized to 1e-6 (and for C = 4 with more rounds)."""
    for C, T in ((1, 200), (4, 600)):
        cfg = synth.CONFIGS["A"].scaled(C=C, N=4)
        H, y, _ = synth.uplink_frame(cfg)
        s, _ = oracle_mod.detect_admm(H, y, rho=1.0, N0=cfg.N0, mod=cfg.mod, T=T)
        x, _ = oracle_mod.mmse_centralized(H, y, N0=cfg.N0)
        assert rel(s, x) < 1e-6


def test_cg_reaches_centralized_in_u_steps(oracle_mod):
    cfg = synth.CONFIGS["A"].scaled(N=4)
    H, y, _ = synth.uplink_frame(cfg)
    xc, _ = oracle_mod.detect_cg(H, y, rho=cfg.N0, T=cfg.U, mod=cfg.mod)
    x, _ = oracle_mod.mmse_centralized(H, y, N0=cfg.N0)
    assert rel(xc, x) < 1e-9


@pytest.mark.parametrize("cfg", [synth.CONFIGS["D"].scaled(N=3), synth.CONFIGS["A"].scaled(algo="admm_dl", N_sym=2)])
def test_zf_precoder_exact_and_minimum_norm(oracle_mod, cfg):
    Hd, s = synth.downlink_frame(cfg)
    x = oracle_mod.zf_centralized(Hd, s)
    for n in range(cfg.N):
        Hn = stacked_dl(Hd, n)
        for j in range(cfg.N_sym):
            xn = np.concatenate([x[c, n, j] for c in range(cfg.C)])
            assert np.linalg.norm(Hn @ xn - s[n, j]) < 1e-10 * max(1.0, np.linalg.norm(s[n, j]))   # S307
            assert rel(xn, np.linalg.pinv(Hn) @ s[n, j].astype(np.complex128)) < 1e-9                # S308


def test_zf_orthonormal_rows(oracle_mod):
    """SPEC S306: H with orthonormal rows -> x = H^H s."""
    rng = np.random.default_rng(2)
    U, S, C = 3, 4, 2
    Q, _ = np.linalg.qr(rng.standard_normal((C * S, U)) + 1j * rng.standard_normal((C * S, U)))
    Hfull = Q.conj().T                                   # U x B with orthonormal rows
    Hd = np.stack([Hfull[:, c * S:(c + 1) * S] for c in range(C)])[:, None].astype(np.complex64)
    s = (rng.standard_normal((1, 1, U)) + 1j * rng.standard_normal((1, 1, U))).astype(np.complex64)
    x = oracle_mod.zf_centralized(Hd, s)
    xn = np.concatenate([x[c, 0, 0] for c in range(C)])
    Hf = np.concatenate([Hd[c, 0].astype(np.complex128) for c in range(C)], axis=1)
    assert rel(xn, Hf.conj().T @ np.linalg.solve(Hf @ Hf.conj().T, s[0, 0])) < 1e-12
    assert rel(xn, Hf.conj().T @ s[0, 0]) < 1e-6          # fp32 rounding of the stored orthonormal rows


def test_bf_admm_converges_to_zf(oracle_mod):
    cfg = synth.CONFIGS["D"].scaled(N=2, C=4)
    Hd, s = synth.downlink_frame(cfg)
    x = oracle_mod.beamform_admm(Hd, s, rho=1.0, T=1000)      # geometric: 0.11 at T=50, 4e-8 at T=1000
    assert rel(x, oracle_mod.zf_centralized(Hd, s)) < 1e-6


def test_rank_deficient_raises(oracle_mod):
    H = np.zeros((1, 2, 4, 3), dtype=np.complex64)
    y = np.zeros((1, 2, 1, 4), dtype=np.complex64)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.mmse_centralized(H, y, N0=0.0)
