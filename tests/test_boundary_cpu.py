"""C-ABI library: builds, loads and exports every symbol include/dbp.h declares
(no compute calls without a GPU); host-side validation paths that need no
device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dbp.h")).read()
    return sorted(set(re.findall(r"^(?:dbp_status|const char\*)\s+(dbp_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1702_04458_b200 import build, dbp
    build.build()
    return dbp.load()


def test_header_declares_expected_api():
    syms = declared_symbols()
    for s in ["dbp_detect_admm", "dbp_detect_cg", "dbp_beamform_admm", "dbp_ctx_create", "dbp_sync",
              "dbp_workspace_bytes", "dbp_get_unique_id", "dbp_last_error", "dbp_slice"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_1702_04458_b200 import dbp
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(dbp.EXPORTS) == declared_symbols()


def test_library_is_sm100a(lib):
    import subprocess
    from paper_1702_04458_b200 import dbp
    out = subprocess.run(["cuobjdump", "--list-elf", dbp.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_context_is_rejected_without_gpu(lib):
    from paper_1702_04458_b200 import dbp
    d = dbp.Dims(2, 16, 4, 16, 1)
    out = ctypes.c_size_t()
    assert lib.dbp_workspace_bytes(None, ctypes.byref(d), 0, ctypes.byref(out)) == 1
    assert b"ctx" in lib.dbp_last_error()
    assert lib.dbp_detect_admm(None, ctypes.byref(d), None, None, 1.0, 1.0, 0.1, 1.0, 0, 2, 5,
                               None, None, None, 0, None) == 1
    assert lib.dbp_sync(None, None) == 1
    assert lib.dbp_get_unique_id(None) == 1


def test_product_package_does_not_import_oracle():
    """The product path never touches oracle/ (DESIGN.md section 4)."""
    pkg = os.path.join(ROOT, "paper_1702_04458_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "dbp_oracle" not in txt, f


def test_binding_validates_shapes_and_dtypes():
    """the wrappers check every array against the dims passed to the C ABI (which
    trusts them) before any call -- a mismatched y / output buffer / dtype raises ValueError
    instead of an out-of-bounds device or host access."""
    import types

    import numpy as np
    import pytest as _pt

    from paper_1702_04458_b200 import dbp
    ctx = types.SimpleNamespace(device=0, world=1, rank=0)
    C, N, S, U = 2, 5, 8, 4
    H = np.zeros((C, N, S, U), np.complex64)
    y = np.zeros((C, N, 1, S), np.complex64)
    Hd = np.zeros((C, N, U, S), np.complex64)
    s = np.zeros((N, 1, U), np.complex64)
    bad = [
        lambda: dbp.detect_admm(ctx, H, y[:, :4]),                                    # y: fewer subcarriers
        lambda: dbp.detect_admm(ctx, H, np.zeros((C, N, 1, S + 1), np.complex64)),    # y: wrong S
        lambda: dbp.detect_admm(ctx, H, y, s_hat=np.zeros((N, 1, U - 1), np.complex64)),
        lambda: dbp.detect_admm(ctx, H, y, hard=np.zeros((N, 1, U), np.complex64)),   # hard must be uint8
        lambda: dbp.detect_admm(ctx, H.astype(np.complex128), y),
        lambda: dbp.detect_cg(ctx, H, y.astype(np.uint8)),                            # uint8 for a complex input
        lambda: dbp.detect_cg(ctx, H, y, x_hat=np.zeros((N + 1, 1, U), np.complex64)),
        lambda: dbp.beamform_admm(ctx, Hd, s[:3]),
        lambda: dbp.beamform_admm(ctx, Hd, s, x=np.zeros((C, N, 1, S - 1), np.complex64)),
        lambda: dbp.detect_mmse(ctx, H[:, :, :, :3], y),
        lambda: dbp.precode_zf(ctx, Hd, np.zeros((N, 1, U + 1), np.complex64)),
        lambda: dbp.detect_admm(ctx, np.asfortranarray(H), y),                        # not C-contiguous
        lambda: dbp.detect_admm(ctx, H[0], y),                                        # 3-D H
    ]
    for f in bad:
        with _pt.raises(ValueError):
            f()


def test_missing_library_fails_loudly():
    """No CPU fallback: with the shared library absent the binding raises (DbpError), it never
    computes anything itself."""
    import subprocess
    import sys
    code = ("from paper_1702_04458_b200 import dbp\n"
            "try:\n"
            "    dbp.load()\n"
            "except dbp.DbpError as e:\n"
            "    print('raised', e)\n"
            "else:\n"
            "    print('loaded')\n")
    env = dict(os.environ, DBP_LIB=os.path.join(ROOT, "build_var", "does_not_exist.so"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("raised") and "not built" in r.stdout, r.stdout + r.stderr


def test_binding_option_constants_match_header():
    """Every DBP_OPT_* value of include/dbp.h has the same value as the binding's OPT_* constant."""
    from paper_1702_04458_b200 import dbp
    src = open(os.path.join(ROOT, "include", "dbp.h")).read()
    opts = dict((k, int(v)) for k, v in re.findall(r"DBP_OPT_(\w+)\s*=\s*(\d+)", src))
    assert len(opts) >= 8
    for k, v in opts.items():
        assert getattr(dbp, "OPT_" + k) == v, k


def test_set_option_rejects_unknown_without_gpu(lib):
    assert lib.dbp_set_option(None, 8, 1) == 1              # null context: invalid argument
