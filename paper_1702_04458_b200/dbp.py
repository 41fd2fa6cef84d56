"""ctypes binding of libdbp (include/dbp.h) -- argument marshalling only.

Every step of the hot path runs in libdbp's sm_100a kernels; this module
converts torch tensors (device pointers, the caller's current CUDA stream) or
numpy arrays (host pointers, staged by the library inside the call) into the
C-ABI arguments and raises ``DbpError`` on a non-OK status.  There is no CPU
fallback: if ``libdbp.so`` is missing or no GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DBP_LIB") or os.path.join(_HERE, "libdbp.so")   # DBP_LIB: tuning variants

STATUS = {0: "DBP_OK", 1: "DBP_ERR_INVALID_ARG", 2: "DBP_ERR_UNSUPPORTED", 3: "DBP_ERR_NOT_HPD",
          4: "DBP_ERR_CUDA", 5: "DBP_ERR_NCCL", 6: "DBP_ERR_WORKSPACE"}
REG = {"mmse": 0, "zf": 1, "box": 2}
MOD = {"bpsk": 1, "qpsk": 2, "qam16": 4, "qam64": 6}
ALGO = {"admm_ul": 0, "cg_ul": 1, "admm_dl": 2, "mmse_ul": 3, "zf_dl": 4}
OPT_FORCE_SPLIT = 1
OPT_KERNEL_TIMING = 2
OPT_NO_FUSED = 3
OPT_DEVICE_CONSENSUS = 4
OPT_MODE = 5
OPT_GRAPHS = 6
OPT_CG_TENSOR = 7
OPT_OVERLAP_PREV = 8

EXPORTS = ["dbp_get_unique_id", "dbp_ctx_create", "dbp_ctx_destroy", "dbp_set_option", "dbp_get_stats",
           "dbp_last_error", "dbp_workspace_bytes", "dbp_detect_admm", "dbp_detect_cg",
           "dbp_beamform_admm", "dbp_slice", "dbp_sync", "dbp_get_kernel_times", "dbp_complexity",
           "dbp_detect_mmse", "dbp_precode_zf", "dbp_get_comm_info", "dbp_set_allreduce_hook"]
CPLX_ALGO = {"admm_dl": 0, "admm_ul": 1, "cg_ul": 2, "zf_dl": 3, "mmse_ul": 4}
CPLX_MODE = {"SxS": 0, "UxU": 1, None: 1}
CPLX_METRIC = {"TM": 0, "AR": 1}


class DbpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Dims(ctypes.Structure):
    _fields_ = [("C", ctypes.c_int32), ("S", ctypes.c_int32), ("U", ctypes.c_int32),
                ("N", ctypes.c_int32), ("N_sym", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("allreduce_calls", ctypes.c_int64), ("allreduce_bytes", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("consensus_rounds", ctypes.c_int64),
                ("graph_replays", ctypes.c_int64)]


class KernelTime(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 40), ("launches", ctypes.c_int64), ("total_ms", ctypes.c_double)]


_lib = None


def load() -> ctypes.CDLL:
    """Load libdbp.so (raises if it was not built; no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DbpError(4, f"{LIB_PATH} not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P, I, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
    S, I64 = ctypes.c_size_t, ctypes.c_int64
    sigs = {
        "dbp_get_unique_id": [P],
        "dbp_ctx_create": [P, I, I, I, P],
        "dbp_ctx_destroy": [P],
        "dbp_set_option": [P, I, I64],
        "dbp_get_stats": [P, P],
        "dbp_workspace_bytes": [P, P, I, P],
        "dbp_detect_admm": [P, P, P, P, F, F, F, F, I, I, ctypes.c_int32, P, P, P, S, P],
        "dbp_detect_cg": [P, P, P, P, F, I, ctypes.c_int32, P, P, P, S, P],
        "dbp_beamform_admm": [P, P, P, P, F, F, F, ctypes.c_int32, P, P, S, P],
        "dbp_slice": [P, I, I64, P, P, P],
        "dbp_sync": [P, P],
        "dbp_get_kernel_times": [P, P, I, P, I],
        "dbp_complexity": [I, I, I, I64, I64, I64, I64, P],
        "dbp_detect_mmse": [P, P, P, P, F, F, I, P, P, P, S, P],
        "dbp_precode_zf": [P, P, P, P, P, P, S, P],
        "dbp_get_comm_info": [P, P, P],
        "dbp_set_allreduce_hook": [P, P, P],
    }
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.dbp_last_error.argtypes = []
    lib.dbp_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(st: int):
    if st != 0:
        raise DbpError(st, load().dbp_last_error().decode())


def get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(load().dbp_get_unique_id(buf))
    return bytes(buf)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        return ctypes.c_void_p(x.data_ptr())
    return x.ctypes.data_as(ctypes.c_void_p)


def _stream(stream, ref):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    if ref is not None and _is_torch(ref) and ref.is_cuda:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream(ref.device).cuda_stream)
    return ctypes.c_void_p(0)


def _empty_like_io(ref, shape, kind):
    """Output buffer on the same side (device tensor / host array) as `ref`."""
    if _is_torch(ref):
        import torch
        dt = torch.complex64 if kind == "c" else torch.uint8
        return torch.empty(shape, dtype=dt, device=ref.device)
    return np.empty(shape, dtype=np.complex64 if kind == "c" else np.uint8)


def _check_args(ctx, spec, ws=None):
    """Validate every array against the dims the C ABI will be told (the library trusts them):
    spec = [(name, array or None, expected shape, 'c' complex64 | 'u' uint8), ...].  All arrays
    must be on one side -- torch tensors on ctx's CUDA device, or host (numpy / CPU) arrays --
    C-contiguous, and of the exact shape and dtype; raises ValueError otherwise."""
    kinds = set()
    for name, x, shape, kind in spec:
        if x is None:
            continue
        shp = tuple(int(v) for v in x.shape)
        if shp != tuple(shape):
            raise ValueError(f"{name}: shape {shp}, expected {tuple(shape)}")
        dt = str(x.dtype)
        want = "complex64" if kind == "c" else "uint8"
        if not dt.endswith(want):
            raise ValueError(f"{name}: dtype {dt}, expected {want}")
        if _is_torch(x):
            if not x.is_contiguous():
                raise ValueError(f"{name}: must be contiguous")
            if x.is_cuda:
                if x.device.index != ctx.device:
                    raise ValueError(f"{name}: on {x.device}, the context is on cuda:{ctx.device}")
                kinds.add("device")
            else:
                kinds.add("host")
        else:
            if not x.flags["C_CONTIGUOUS"]:
                raise ValueError(f"{name}: must be C-contiguous")
            kinds.add("host")
    if len(kinds) > 1:
        raise ValueError("all arrays of one call must be device tensors or all host arrays")
    if ws is not None:
        if not (_is_torch(ws) and ws.is_cuda and ws.device.index == ctx.device):
            raise ValueError(f"ws must be a CUDA tensor on cuda:{ctx.device}")
        if not ws.is_contiguous():
            raise ValueError("ws must be contiguous")


def _dims4(x, name):
    if len(x.shape) != 4:
        raise ValueError(f"{name}: expected 4 dims, got shape {tuple(x.shape)}")
    return tuple(int(v) for v in x.shape)


def _dim(x, i, name):
    if len(x.shape) <= i:
        raise ValueError(f"{name}: shape {tuple(x.shape)} has no dim {i}")
    return int(x.shape[i])


HOOK_T = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_float), ctypes.c_int64, ctypes.c_void_p)


class Context:
    """One libdbp context (one per rank); NCCL communicator when world > 1."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, unique_id: bytes | None = None):
        lib = load()
        self._h = ctypes.c_void_p()
        uid = None
        if unique_id is not None:
            uid = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(lib.dbp_ctx_create(ctypes.byref(self._h), device, rank, world, uid))
        self.device, self.rank, self.world = device, rank, world

    def close(self):
        if self._h:
            load().dbp_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, opt: int, value: int):
        _check(load().dbp_set_option(self._h, opt, value))

    def stats(self) -> dict:
        s = Stats()
        _check(load().dbp_get_stats(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def set_allreduce_hook(self, fn):
        """Host consensus exchange for a context created with world > 1 and no unique id:
        fn(arr) receives the round's partial sums as a float32 numpy array (a view of the
        library's pinned buffer) and must replace them in place by their sum over all ranks."""
        def _cb(ptr, n, user):
            try:
                fn(np.ctypeslib.as_array(ptr, shape=(int(n),)))
                return 0
            except Exception:                       # noqa: BLE001 -- reported as DBP_ERR_NCCL
                return 1
        self._hook = HOOK_T(_cb)                    # keep the trampoline alive with the context
        _check(load().dbp_set_allreduce_hook(self._h, self._hook, None))

    def comm_info(self) -> dict:
        """{'nranks': ncclCommCount, 'rank': ncclCommUserRank} of the consensus communicator."""
        n, r = ctypes.c_int(), ctypes.c_int()
        _check(load().dbp_get_comm_info(self._h, ctypes.byref(n), ctypes.byref(r)))
        return {"nranks": n.value, "rank": r.value}

    def workspace_bytes(self, C, S, U, N, N_sym, algo: str) -> int:
        d = Dims(C, S, U, N, N_sym)
        out = ctypes.c_size_t()
        _check(load().dbp_workspace_bytes(self._h, ctypes.byref(d), ALGO[algo], ctypes.byref(out)))
        return out.value

    def kernel_times(self, reset: bool = False) -> dict:
        """{name: (launches, total_ms)} recorded under OPT_KERNEL_TIMING (blocks on the events)."""
        arr = (KernelTime * 64)()
        n = ctypes.c_int()
        _check(load().dbp_get_kernel_times(self._h, arr, 64, ctypes.byref(n), int(reset)))
        return {arr[i].name.decode(): (arr[i].launches, arr[i].total_ms) for i in range(n.value)}

    def sync(self, stream=None):
        _check(load().dbp_sync(self._h, _stream(stream, None) if stream is not None else _cur_stream()))


def _cur_stream():
    try:
        import torch
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    except Exception:
        pass
    return ctypes.c_void_p(0)


def detect_admm(ctx: Context, H, y, *, rho=1.0, gamma=1.0, N0=0.0, Es=1.0, reg="mmse", mod="qam64", T=5,
                s_hat=None, hard=None, want_hard=True, ws=None, stream=None):
    """Algorithm 1.  H [C_loc][N][S][U], y [C_loc][N][N_sym][S] -> (s_hat [N][N_sym][U], hard)."""
    C_loc, N, S, U = _dims4(H, "H")
    J = _dim(y, 2, "y")
    if s_hat is None:
        s_hat = _empty_like_io(H, (N, J, U), "c")
    if hard is None and want_hard:
        hard = _empty_like_io(H, (N, J, U), "u")
    _check_args(ctx, [("H", H, (C_loc, N, S, U), "c"), ("y", y, (C_loc, N, J, S), "c"),
                      ("s_hat", s_hat, (N, J, U), "c"), ("hard", hard, (N, J, U), "u")], ws)
    d = Dims(C_loc * ctx.world, S, U, N, J)
    wsb = 0 if ws is None else (ws.numel() * ws.element_size() if _is_torch(ws) else ws.nbytes)
    _check(load().dbp_detect_admm(ctx._h, ctypes.byref(d), _ptr(H), _ptr(y), rho, gamma, N0, Es, REG[reg],
                                  MOD[mod], T, _ptr(s_hat), _ptr(hard), _ptr(ws), wsb, _stream(stream, H)))
    return s_hat, hard


def detect_cg(ctx: Context, H, y, *, rho=0.0, mod="qam64", T=5, x_hat=None, hard=None, want_hard=True,
              ws=None, stream=None):
    """Algorithm 2.  -> (x_hat [N][N_sym][U], hard)."""
    C_loc, N, S, U = _dims4(H, "H")
    J = _dim(y, 2, "y")
    if x_hat is None:
        x_hat = _empty_like_io(H, (N, J, U), "c")
    if hard is None and want_hard:
        hard = _empty_like_io(H, (N, J, U), "u")
    _check_args(ctx, [("H", H, (C_loc, N, S, U), "c"), ("y", y, (C_loc, N, J, S), "c"),
                      ("x_hat", x_hat, (N, J, U), "c"), ("hard", hard, (N, J, U), "u")], ws)
    d = Dims(C_loc * ctx.world, S, U, N, J)
    wsb = 0 if ws is None else (ws.numel() * ws.element_size() if _is_torch(ws) else ws.nbytes)
    _check(load().dbp_detect_cg(ctx._h, ctypes.byref(d), _ptr(H), _ptr(y), rho, MOD[mod], T, _ptr(x_hat),
                                _ptr(hard), _ptr(ws), wsb, _stream(stream, H)))
    return x_hat, hard


def beamform_admm(ctx: Context, Hd, s, *, rho=1.0, gamma=1.0, eps=0.0, T=5, x=None, ws=None, stream=None):
    """Algorithm 3.  Hd [C_loc][N][U][S], s [N][N_sym][U] -> x [C_loc][N][N_sym][S]."""
    C_loc, N, U, S = _dims4(Hd, "Hd")
    J = _dim(s, 1, "s")
    if x is None:
        x = _empty_like_io(Hd, (C_loc, N, J, S), "c")
    _check_args(ctx, [("Hd", Hd, (C_loc, N, U, S), "c"), ("s", s, (N, J, U), "c"),
                      ("x", x, (C_loc, N, J, S), "c")], ws)
    d = Dims(C_loc * ctx.world, S, U, N, J)
    wsb = 0 if ws is None else (ws.numel() * ws.element_size() if _is_torch(ws) else ws.nbytes)
    _check(load().dbp_beamform_admm(ctx._h, ctypes.byref(d), _ptr(Hd), _ptr(s), rho, gamma, eps, T, _ptr(x),
                                    _ptr(ws), wsb, _stream(stream, Hd)))
    return x


def detect_mmse(ctx: Context, H, y, *, N0=0.0, Es=1.0, mod="qam64", x_hat=None, hard=None, want_hard=True,
                ws=None, stream=None):
    """Centralized MMSE-UL detection (N0 = 0: ZF) over all clusters.  -> (x_hat [N][N_sym][U], hard)."""
    C_loc, N, S, U = _dims4(H, "H")
    J = _dim(y, 2, "y")
    if x_hat is None:
        x_hat = _empty_like_io(H, (N, J, U), "c")
    if hard is None and want_hard:
        hard = _empty_like_io(H, (N, J, U), "u")
    _check_args(ctx, [("H", H, (C_loc, N, S, U), "c"), ("y", y, (C_loc, N, J, S), "c"),
                      ("x_hat", x_hat, (N, J, U), "c"), ("hard", hard, (N, J, U), "u")], ws)
    d = Dims(C_loc * ctx.world, S, U, N, J)
    wsb = 0 if ws is None else (ws.numel() * ws.element_size() if _is_torch(ws) else ws.nbytes)
    _check(load().dbp_detect_mmse(ctx._h, ctypes.byref(d), _ptr(H), _ptr(y), N0, Es, MOD[mod], _ptr(x_hat),
                                  _ptr(hard), _ptr(ws), wsb, _stream(stream, H)))
    return x_hat, hard


def precode_zf(ctx: Context, Hd, s, *, x=None, ws=None, stream=None):
    """Centralized ZF-DL precoding x_c = H_c^H (sum_c H_c H_c^H)^{-1} s -> x [C_loc][N][N_sym][S]."""
    C_loc, N, U, S = _dims4(Hd, "Hd")
    J = _dim(s, 1, "s")
    if x is None:
        x = _empty_like_io(Hd, (C_loc, N, J, S), "c")
    _check_args(ctx, [("Hd", Hd, (C_loc, N, U, S), "c"), ("s", s, (N, J, U), "c"),
                      ("x", x, (C_loc, N, J, S), "c")], ws)
    d = Dims(C_loc * ctx.world, S, U, N, J)
    wsb = 0 if ws is None else (ws.numel() * ws.element_size() if _is_torch(ws) else ws.nbytes)
    _check(load().dbp_precode_zf(ctx._h, ctypes.byref(d), _ptr(Hd), _ptr(s), _ptr(x), _ptr(ws), wsb,
                                 _stream(stream, Hd)))
    return x


def complexity(algo: str, mode, metric: str, U: int, S: int, C: int, T: int = 1) -> dict:
    """Table I (P566-595) real-multiplication counts: preprocessing, first and each
    subsequent iteration, and total(T) (host-only; see include/dbp.h)."""
    out = (ctypes.c_int64 * 4)()
    _check(load().dbp_complexity(CPLX_ALGO[algo], CPLX_MODE[mode], CPLX_METRIC[metric], U, S, C, T, out))
    return {"pre": out[0], "first": out[1], "next": out[2], "total": out[3]}


def slice_bits(ctx: Context, x, mod: str, out=None, stream=None):
    """Hard slicer (P210) on device or host complex64 data."""
    if out is None:
        out = _empty_like_io(x, tuple(x.shape), "u")
    _check_args(ctx, [("x", x, tuple(int(v) for v in x.shape), "c"), ("out", out, tuple(int(v) for v in x.shape), "u")])
    n = x.numel() if _is_torch(x) else x.size
    _check(load().dbp_slice(ctx._h, MOD[mod], n, _ptr(x), _ptr(out), _stream(stream, x)))
    return out
