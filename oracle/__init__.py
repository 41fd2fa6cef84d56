"""Plain double-precision CPU oracle for arXiv 1702.04458 Algorithms 1-3.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1702_04458_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``oracle/dbp_oracle.c`` (plain C99, ``double
complex``); this module only compiles it (gcc, no fast-math) and marshals
numpy arrays.  Inputs are the same complex64 arrays the GPU path consumes,
promoted to double inside the C code (SURVEY 8(c) "Form").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dbp_oracle.c")
_HDR = os.path.join(_HERE, "dbp_oracle.h")
_SO = os.path.join(_HERE, "_dbp_oracle.so")
_lock = threading.Lock()
_lib = None

REG = {"mmse": 0, "zf": 1, "box": 2}
MOD = {"bpsk": 1, "qpsk": 2, "qam16": 4, "qam64": 6}
MODE = {"paper": -1, "uu": 0, "ss": 1}


class Dims(ctypes.Structure):
    _fields_ = [("C", ctypes.c_int32), ("S", ctypes.c_int32), ("U", ctypes.c_int32),
                ("N", ctypes.c_int32), ("N_sym", ctypes.c_int32)]


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile the oracle shared library in-tree (idempotent)."""
    with _lock:
        stale = (not os.path.exists(_SO) or
                 os.path.getmtime(_SO) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
        if force or stale:
            tmp = _SO + f".tmp{os.getpid()}"
            cmd = ["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared",
                   "-fno-fast-math", "-ffp-contract=off", "-Wall", "-o", tmp, _SRC, "-lm"]
            subprocess.run(cmd, check=True)
            os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        d, i, i64 = ctypes.c_double, ctypes.c_int, ctypes.c_int64
        sig = {
            "dbpo_hpd_inverse": [i, P, P],
            "dbpo_slice": [i, i64, P, P],
            "dbpo_detect_admm": [P, P, P, d, d, d, d, i, i, i, i, P, P],
            "dbpo_detect_admm_trace": [P, P, P, d, d, d, d, i, i, i, i, i, i, P, P, P],
            "dbpo_detect_cg": [P, P, P, d, i, i, P, P],
            "dbpo_detect_cg_trace": [P, P, P, d, i, i, i, P, P, P],
            "dbpo_beamform_admm": [P, P, P, d, d, d, i, i, P],
            "dbpo_beamform_admm_trace": [P, P, P, d, d, d, i, i, i, i, P, P, P, P],
            "dbpo_mmse_centralized": [P, P, P, d, d, i, P, P],
            "dbpo_zf_centralized": [P, P, P, P],
        }
        for name, args in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex64)


def _check(st: int, what: str):
    if st == 1:
        raise OracleError(f"{what}: invalid argument")
    if st == 3:
        raise OracleError(f"{what}: matrix not Hermitian positive definite")
    if st != 0:
        raise OracleError(f"{what}: status {st}")


def hpd_inverse(G) -> np.ndarray:
    G = np.ascontiguousarray(G, dtype=np.complex128)
    n = G.shape[0]
    out = np.empty_like(G)
    _check(_load().dbpo_hpd_inverse(n, _ptr(G), _ptr(out)), "hpd_inverse")
    return out


def slice_bits(x, mod: str) -> np.ndarray:
    """Gray bits of the nearest constellation point, decided in fp32."""
    x = _c64(x)
    out = np.empty(x.shape, dtype=np.uint8)
    _check(_load().dbpo_slice(MOD[mod], x.size, _ptr(x), _ptr(out)), "slice")
    return out


def _dims(H, y_or_s, uplink=True):
    C, N = H.shape[0], H.shape[1]
    if uplink:
        S, U = H.shape[2], H.shape[3]
        J = y_or_s.shape[2]
    else:
        U, S = H.shape[2], H.shape[3]
        J = y_or_s.shape[1]
    return Dims(C, S, U, N, J)


def detect_admm(H, y, *, rho=1.0, gamma=1.0, N0=0.0, Es=1.0, reg="mmse", mod="qam64",
                T=5, mode="paper"):
    """Algorithm 1.  H [C][N][S][U], y [C][N][Nsym][S] -> (s_hat [N][Nsym][U] c128, hard u8)."""
    H, y = _c64(H), _c64(y)
    d = _dims(H, y)
    s_hat = np.empty((d.N, d.N_sym, d.U), dtype=np.complex128)
    hard = np.empty((d.N, d.N_sym, d.U), dtype=np.uint8)
    st = _load().dbpo_detect_admm(ctypes.byref(d), _ptr(H), _ptr(y), rho, gamma, N0, Es,
                                  REG[reg], MOD[mod], T, MODE[mode], _ptr(s_hat), _ptr(hard))
    _check(st, "detect_admm")
    return s_hat, hard


def detect_admm_trace(H, y, *, rho=1.0, gamma=1.0, N0=0.0, Es=1.0, reg="mmse", mod="qam64",
                      T=5, mode="paper", n=0, j=0):
    """Iterates of Alg. 1 at (n, j): s [T][U], z [T][C][U], lam [T][C][U]."""
    H, y = _c64(H), _c64(y)
    d = _dims(H, y)
    s = np.empty((T, d.U), dtype=np.complex128)
    z = np.empty((T, d.C, d.U), dtype=np.complex128)
    lam = np.empty((T, d.C, d.U), dtype=np.complex128)
    st = _load().dbpo_detect_admm_trace(ctypes.byref(d), _ptr(H), _ptr(y), rho, gamma, N0, Es,
                                        REG[reg], MOD[mod], T, MODE[mode], n, j,
                                        _ptr(s), _ptr(z), _ptr(lam))
    _check(st, "detect_admm_trace")
    return s, z, lam


def detect_cg(H, y, *, rho=0.0, mod="qam64", T=5):
    """Algorithm 2.  -> (x_hat [N][Nsym][U] c128, hard u8)."""
    H, y = _c64(H), _c64(y)
    d = _dims(H, y)
    x = np.empty((d.N, d.N_sym, d.U), dtype=np.complex128)
    hard = np.empty((d.N, d.N_sym, d.U), dtype=np.uint8)
    _check(_load().dbpo_detect_cg(ctypes.byref(d), _ptr(H), _ptr(y), rho, MOD[mod], T,
                                  _ptr(x), _ptr(hard)), "detect_cg")
    return x, hard


def detect_cg_trace(H, y, *, rho=0.0, T=5, n=0, j=0):
    """x, r, p for t = 0..T at (n, j): each [T+1][U]."""
    H, y = _c64(H), _c64(y)
    d = _dims(H, y)
    x = np.empty((T + 1, d.U), dtype=np.complex128)
    r = np.empty_like(x)
    p = np.empty_like(x)
    _check(_load().dbpo_detect_cg_trace(ctypes.byref(d), _ptr(H), _ptr(y), rho, T, n, j,
                                        _ptr(x), _ptr(r), _ptr(p)), "detect_cg_trace")
    return x, r, p


def beamform_admm(Hd, s, *, rho=1.0, gamma=1.0, eps=0.0, T=5, mode="paper"):
    """Algorithm 3.  Hd [C][N][U][S], s [N][Nsym][U] -> x [C][N][Nsym][S] c128."""
    Hd, s = _c64(Hd), _c64(s)
    d = _dims(Hd, s, uplink=False)
    x = np.empty((d.C, d.N, d.N_sym, d.S), dtype=np.complex128)
    _check(_load().dbpo_beamform_admm(ctypes.byref(d), _ptr(Hd), _ptr(s), rho, gamma, eps, T,
                                      MODE[mode], _ptr(x)), "beamform_admm")
    return x


def beamform_admm_trace(Hd, s, *, rho=1.0, gamma=1.0, eps=0.0, T=5, mode="paper", n=0, j=0):
    """x [T][C][S], z [T][C][U], lam [T][C][U], w [T][C][U] at (n, j)."""
    Hd, s = _c64(Hd), _c64(s)
    d = _dims(Hd, s, uplink=False)
    x = np.empty((T, d.C, d.S), dtype=np.complex128)
    z = np.empty((T, d.C, d.U), dtype=np.complex128)
    lam = np.empty_like(z)
    w = np.empty_like(z)
    _check(_load().dbpo_beamform_admm_trace(ctypes.byref(d), _ptr(Hd), _ptr(s), rho, gamma, eps,
                                            T, MODE[mode], n, j, _ptr(x), _ptr(z), _ptr(lam),
                                            _ptr(w)), "beamform_admm_trace")
    return x, z, lam, w


def mmse_centralized(H, y, *, N0=0.0, Es=1.0, mod="qam64"):
    """Centralized MMSE-UL (N0 = 0: ZF) over all clusters -> (x_hat [N][Nsym][U] c128, hard u8)."""
    H, y = _c64(H), _c64(y)
    d = _dims(H, y)
    x = np.empty((d.N, d.N_sym, d.U), dtype=np.complex128)
    hard = np.empty((d.N, d.N_sym, d.U), dtype=np.uint8)
    _check(_load().dbpo_mmse_centralized(ctypes.byref(d), _ptr(H), _ptr(y), N0, Es, MOD[mod], _ptr(x),
                                         _ptr(hard)), "mmse_centralized")
    return x, hard


def zf_centralized(Hd, s):
    """Centralized ZF-DL precoder x_c = H_c^H (sum_c H_c H_c^H)^{-1} s -> x [C][N][Nsym][S] c128."""
    Hd, s = _c64(Hd), _c64(s)
    d = _dims(Hd, s, uplink=False)
    x = np.empty((d.C, d.N, d.N_sym, d.S), dtype=np.complex128)
    _check(_load().dbpo_zf_centralized(ctypes.byref(d), _ptr(Hd), _ptr(s), _ptr(x)), "zf_centralized")
    return x
