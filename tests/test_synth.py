"""Seeded input generator: determinism, shard independence, moments (no GPU)."""
import numpy as np

from paper_1702_04458_b200 import synth


def test_philox_known_answer():
    # Random123 Philox-4x32-10 known-answer vector: ctr = key = 0
    out = synth.philox4x32(np.array([0], dtype=np.uint64), 0, 0)
    assert [int(o[0]) for o in out] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_channel_moments_and_shards():
    cfg = synth.CONFIGS["B"].scaled(N=64)
    H = synth.uplink_channel(cfg)
    assert abs(np.mean(H)) < 0.01 and abs(np.mean(np.abs(H) ** 2) - 1) < 0.02
    part = synth.uplink_channel(cfg, 2, 5, 10, 30)
    assert np.array_equal(part, H[2:5, 10:30])
    H2, y2, s2 = synth.uplink_frame(cfg, 2, 5, 10, 30)
    Hf, yf, sf = synth.uplink_frame(cfg)
    assert np.array_equal(y2, yf[2:5, 10:30]) and np.array_equal(s2, sf[10:30])


def test_symbols_on_alphabet():
    for mod, (m, norm) in synth._LEVELS.items():
        s = synth.qam_symbols(0, 4096, 1, 5, mod)
        k = (s.real * np.sqrt(norm) + (m - 1)) / 2
        assert np.allclose(k, np.round(k)) and round(k.min()) == 0 and round(k.max()) == m - 1
        assert abs(np.mean(np.abs(s) ** 2) - 1) < 0.05


def test_downlink_reciprocity():
    cfg = synth.CONFIGS["D"].scaled(N=8, C=4)
    Hd, s = synth.downlink_frame(cfg)
    H = synth.uplink_channel(cfg)
    assert np.array_equal(Hd, np.swapaxes(H, 2, 3))   # H^d = (H^u)^T (P174)


def test_cluster_range():
    assert synth.cluster_range(32, 3, 8) == (12, 16)
    import pytest
    with pytest.raises(ValueError):
        synth.cluster_range(6, 0, 4)
