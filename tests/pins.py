"""Independent reference computations that pin the oracle (test-only).

Nothing here calls ``oracle/``: these are textbook closed forms and generic
solvers (numpy / scipy) for the problems the paper states, used as anchors
other than the oracle itself.
"""
from __future__ import annotations

import numpy as np


def stack_uplink(Hc: np.ndarray) -> np.ndarray:
    """[C][S][U] cluster blocks -> B x U full H (row-wise partition, eq. (1) P151)."""
    C, S, U = Hc.shape
    return Hc.astype(np.complex128).reshape(C * S, U)


def mmse(H: np.ndarray, y: np.ndarray, N0: float, Es: float = 1.0) -> np.ndarray:
    """Centralized MMSE equalizer (E0) with g = N0/(2Es)||s||^2 (P212)."""
    U = H.shape[1]
    return np.linalg.solve(H.conj().T @ H + (N0 / Es) * np.eye(U), H.conj().T @ y)


def ls(H: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Zero-forcing (least squares) equalizer, g = 0 (P212)."""
    return np.linalg.lstsq(H, y, rcond=None)[0]


def zf_precoder(Hd: np.ndarray, s: np.ndarray) -> np.ndarray:
    """ZF beamformer x = H^H (H H^H)^{-1} s, the eps = 0 solution of (P0) (P431)."""
    return Hd.conj().T @ np.linalg.solve(Hd @ Hd.conj().T, s)


def textbook_cg(A: np.ndarray, b: np.ndarray, T: int):
    """Hestenes-Stiefel CG on A x = b, x0 = 0; returns iterates x_0..x_T."""
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    xs = [x.copy()]
    for _ in range(T):
        rr = np.vdot(r, r).real
        if rr == 0:
            xs.append(x.copy())
            continue
        Ap = A @ p
        a = rr / np.vdot(p, Ap).real
        x = x + a * p
        r = r - a * Ap
        p = r + (np.vdot(r, r).real / rr) * p
        xs.append(x.copy())
    return xs


def krylov_minimizer(A: np.ndarray, b: np.ndarray, t: int) -> np.ndarray:
    """argmin over x in K_t(A, b) of (x - x*)^H A (x - x*), x* = A^{-1} b.

    The characterising optimality property of CG iterate t (Hestenes-Stiefel);
    computed by Galerkin projection on an orthonormal Krylov basis.
    """
    K = [b]
    for _ in range(t - 1):
        K.append(A @ K[-1])
    Q, _ = np.linalg.qr(np.stack(K, axis=1))
    c = np.linalg.solve(Q.conj().T @ A @ Q, Q.conj().T @ b)
    return Q @ c


def box_ls(H: np.ndarray, y: np.ndarray, r: float) -> np.ndarray:
    """Box-constrained equalizer (E0) with g = chi(s in box of radius r) (P213-218),
    solved on the real-stacked system by scipy's bounded least squares."""
    from scipy.optimize import lsq_linear
    A = np.block([[H.real, -H.imag], [H.imag, H.real]])
    b = np.concatenate([y.real, y.imag])
    res = lsq_linear(A, b, bounds=(-r, r), method="bvls", tol=1e-14)
    U = H.shape[1]
    return res.x[:U] + 1j * res.x[U:]


def box_ls_real(H: np.ndarray, y: np.ndarray, r: float) -> np.ndarray:
    """BPSK box equalizer (P344): s real in [-r, r]^U minimising ||y - H s||; the complex
    system stacked as [Re H; Im H] s = [Re y; Im y], scipy bounded least squares."""
    from scipy.optimize import lsq_linear
    A = np.concatenate([H.real, H.imag], axis=0)
    b = np.concatenate([y.real, y.imag])
    res = lsq_linear(A, b, bounds=(-r, r), method="bvls", tol=1e-14)
    return res.x + 0j


def constellation(mod: str) -> np.ndarray:
    """All points of the Es = 1 Gray alphabet (reading 17)."""
    m, norm = {"bpsk": (2, 1.0), "qpsk": (2, 2.0), "qam16": (4, 10.0), "qam64": (8, 42.0)}[mod]
    lv = (2 * np.arange(m) - (m - 1)) / np.sqrt(norm)
    if mod == "bpsk":
        return lv.astype(np.complex128)
    return (lv[:, None] + 1j * lv[None, :]).ravel()


def gray_bits_of_point(pt: complex, mod: str) -> int:
    """Gray label of an alphabet point: per axis level index k -> k ^ (k >> 1), [I | Q]."""
    m, norm = {"bpsk": (2, 1.0), "qpsk": (2, 2.0), "qam16": (4, 10.0), "qam64": (8, 42.0)}[mod]
    bpa = {2: 1, 4: 2, 8: 3}[m]
    ki = int(round((pt.real * np.sqrt(norm) + (m - 1)) / 2))
    gi = ki ^ (ki >> 1)
    if mod == "bpsk":
        return gi
    kq = int(round((pt.imag * np.sqrt(norm) + (m - 1)) / 2))
    return (gi << bpa) | (kq ^ (kq >> 1))


def brute_force_ml(H: np.ndarray, y: np.ndarray, mod: str) -> np.ndarray:
    """Exhaustive ML detection over the alphabet^U (tiny U only)."""
    pts = constellation(mod)
    U = H.shape[1]
    grids = np.meshgrid(*([pts] * U), indexing="ij")
    cand = np.stack([g.ravel() for g in grids], axis=1)        # [M^U][U]
    d = np.linalg.norm(y[None, :] - cand @ H.T, axis=1)
    return cand[np.argmin(d)]


def rel(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
