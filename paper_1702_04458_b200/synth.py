"""Seeded synthetic inputs shared by the tests, the bench and the oracle legs.

This module holds NO arithmetic of the method (no Gram, inverse, ADMM, CG or
slicing): it only draws random numbers and applies the channel model of the
paper's system description, y = H s + n (P144, eq. (1) P152-154) and
reciprocity H^d = (H^u)^T (P174).

Generator (SURVEY 8(d) "Inputs"): counter-based Philox-4x32-10 keyed by the
64-bit seed; the counter is (flat element index, stream id).  Streams: 0 = H,
1 = uplink symbols, 2 = uplink noise, 3 = downlink symbols.  Because the
counter is the *global* flat index, a rank that generates only its own
clusters gets exactly the values a single-process run would hold for them.

Normals: Box-Muller on two 53-bit uniforms per complex entry, so CN(0, 1)
entries are (r cos t + i r sin t)/sqrt(2).  Symbols: uniform over the Gray
QAM alphabet with Es = 1 (reading 17).  Noise variance N0 = U * Es *
10^(-SNR/10) (reading 16, SPEC S504).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)

STREAM_H, STREAM_SYM_UL, STREAM_NOISE, STREAM_SYM_DL = 0, 1, 2, 3
BITS = {"bpsk": 1, "qpsk": 2, "qam16": 4, "qam64": 6}
_LEVELS = {"bpsk": (2, 1.0), "qpsk": (2, 2.0), "qam16": (4, 10.0), "qam64": (8, 42.0)}


def philox4x32(idx: np.ndarray, stream: int, seed: int):
    """Philox-4x32-10 on counters (idx_lo, idx_hi, stream, 0), key = seed."""
    idx = np.asarray(idx, dtype=np.uint64)
    c0 = idx & _MASK
    c1 = idx >> np.uint64(32)
    c2 = np.full_like(c0, np.uint64(stream) & _MASK)
    c3 = np.zeros_like(c0)
    k0 = np.uint64(seed) & _MASK
    k1 = (np.uint64(seed) >> np.uint64(32)) & _MASK
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    return c0, c1, c2, c3


def _u53(a, b):
    return (((a << np.uint64(32)) | b) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def cnormal(start: int, count: int, stream: int, seed: int, chunk: int = 1 << 22) -> np.ndarray:
    """count CN(0,1) draws for flat indices [start, start+count), complex128."""
    out = np.empty(count, dtype=np.complex128)
    for o in range(0, count, chunk):
        n = min(chunk, count - o)
        x0, x1, x2, x3 = philox4x32(np.arange(start + o, start + o + n, dtype=np.uint64), stream, seed)
        u1, u2 = _u53(x0, x1), _u53(x2, x3)
        r = np.sqrt(-2.0 * np.log1p(-u1))
        t = 2.0 * np.pi * u2
        out[o:o + n] = (r * np.cos(t) + 1j * (r * np.sin(t))) * np.sqrt(0.5)
    return out


def qam_symbols(start: int, count: int, stream: int, seed: int, mod: str) -> np.ndarray:
    """Uniform Gray-QAM symbols with Es = 1 (complex128)."""
    m, norm = _LEVELS[mod]
    x0, x1, _, _ = philox4x32(np.arange(start, start + count, dtype=np.uint64), stream, seed)
    ki = (x0 % np.uint64(m)).astype(np.float64)
    kq = (x1 % np.uint64(m)).astype(np.float64)
    re = (2 * ki - (m - 1)) / np.sqrt(norm)
    if mod == "bpsk":
        return re.astype(np.complex128)
    im = (2 * kq - (m - 1)) / np.sqrt(norm)
    return re + 1j * im


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration."""
    name: str
    algo: str            # "admm_ul", "cg_ul", "admm_dl"
    C: int
    S: int
    U: int
    N: int
    mod: str
    T: int = 5
    N_sym: int = 1
    snr_db: float = 25.0
    rho: float = 1.0
    seed: int = 1702044580
    gpus: tuple = field(default=(1,))

    @property
    def B(self) -> int:
        return self.C * self.S

    @property
    def N0(self) -> float:
        return self.U * 10.0 ** (-self.snr_db / 10.0)

    @property
    def bits_per_frame(self) -> int:
        return self.U * self.N * self.N_sym * BITS[self.mod]

    def scaled(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    "A": Config("A", "admm_ul", C=2, S=16, U=4, N=16, mod="qpsk", T=5, snr_db=10.0,
                seed=1702044580, gpus=(1, 2)),
    "B": Config("B", "cg_ul", C=8, S=16, U=16, N=1200, mod="qam16", T=5, snr_db=15.0,
                seed=1702044581, gpus=(1, 2, 4, 8)),
    "C": Config("C", "admm_ul", C=32, S=32, U=16, N=1200, mod="qam64", T=5, snr_db=25.0,
                seed=1702044582, gpus=(1, 2, 4, 8)),
    "D": Config("D", "admm_dl", C=32, S=32, U=16, N=1200, mod="qam16", T=5,
                seed=1702044583, gpus=(1, 2, 4, 8)),
    "E": Config("E", "admm_ul", C=128, S=32, U=32, N=4800, mod="qam64", T=5, snr_db=25.0,
                seed=1702044584, gpus=(8, 1, 2, 4)),
}


def uplink_channel(cfg: Config, c0: int = 0, c1: int | None = None, n0: int = 0,
                   n1: int | None = None) -> np.ndarray:
    """H^u clusters [c0, c1) x subcarriers [n0, n1): complex64 [c][n][S][U]."""
    c1 = cfg.C if c1 is None else c1
    n1 = cfg.N if n1 is None else n1
    per_c = cfg.N * cfg.S * cfg.U
    per_n = cfg.S * cfg.U
    out = np.empty((c1 - c0, n1 - n0, cfg.S, cfg.U), dtype=np.complex64)
    for c in range(c0, c1):
        start = c * per_c + n0 * per_n
        out[c - c0] = cnormal(start, (n1 - n0) * per_n, STREAM_H, cfg.seed).reshape(
            n1 - n0, cfg.S, cfg.U)
    return out


def uplink_symbols(cfg: Config, n0: int = 0, n1: int | None = None) -> np.ndarray:
    """Transmitted uplink symbols s^u [n][Nsym][U] (complex128, exact alphabet points)."""
    n1 = cfg.N if n1 is None else n1
    per_n = cfg.N_sym * cfg.U
    return qam_symbols(n0 * per_n, (n1 - n0) * per_n, STREAM_SYM_UL, cfg.seed,
                       cfg.mod).reshape(n1 - n0, cfg.N_sym, cfg.U)


def uplink_frame(cfg: Config, c0: int = 0, c1: int | None = None, n0: int = 0,
                 n1: int | None = None, noise: bool = True):
    """(H [c][n][S][U] c64, y [c][n][Nsym][S] c64, s [n][Nsym][U] c128).

    y_c = H_c s + n_c (eq. (1), P152) computed in float64 from the
    float32-rounded H, then rounded to float32.
    """
    c1 = cfg.C if c1 is None else c1
    n1 = cfg.N if n1 is None else n1
    H = uplink_channel(cfg, c0, c1, n0, n1)
    s = uplink_symbols(cfg, n0, n1)
    y = np.einsum("cnsu,nju->cnjs", H.astype(np.complex128), s, optimize=True)
    if noise and cfg.N0 > 0:
        per_c = cfg.N * cfg.N_sym * cfg.S
        per_n = cfg.N_sym * cfg.S
        for c in range(c0, c1):
            start = c * per_c + n0 * per_n
            nz = cnormal(start, (n1 - n0) * per_n, STREAM_NOISE, cfg.seed)
            y[c - c0] += np.sqrt(cfg.N0) * nz.reshape(n1 - n0, cfg.N_sym, cfg.S)
    return H, y.astype(np.complex64), s


def downlink_frame(cfg: Config, c0: int = 0, c1: int | None = None, n0: int = 0,
                   n1: int | None = None):
    """(Hd [c][n][U][S] c64 = per-pair transpose of H^u (P174), s [n][Nsym][U] c64)."""
    n1 = cfg.N if n1 is None else n1
    H = uplink_channel(cfg, c0, c1, n0, n1)
    Hd = np.ascontiguousarray(np.swapaxes(H, 2, 3))
    per_n = cfg.N_sym * cfg.U
    s = qam_symbols(n0 * per_n, (n1 - n0) * per_n, STREAM_SYM_DL, cfg.seed,
                    cfg.mod).reshape(n1 - n0, cfg.N_sym, cfg.U)
    return Hd, s.astype(np.complex64)


def cluster_range(C: int, rank: int, world: int):
    """Contiguous cluster block of a rank; C % world == 0 required."""
    if world < 1 or C % world:
        raise ValueError(f"C={C} not divisible by world={world}")
    per = C // world
    return rank * per, (rank + 1) * per
