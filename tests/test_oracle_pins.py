"""Pins of the oracle against what the paper and mathematics fix (no GPU).

Each test anchors an oracle function to something other than itself:
closed forms (MMSE, LS, ZF), generic solvers (scipy bounded LS), the
optimality conditions of the sub-problems (E1)-(E3), (P1)-(P3) stated in the
paper, Krylov optimality of CG, worked examples (tests/golden), brute force,
and invariances.  See DESIGN.md section 4 for the list per function.
"""
import json
import os

import numpy as np
import pytest

from tests import pins

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rand_ul(rng, C, S, U, N=1, J=1, snr_db=20.0, mod="qpsk", noise=True):
    H = ((rng.standard_normal((C, N, S, U)) + 1j * rng.standard_normal((C, N, S, U))) /
         np.sqrt(2)).astype(np.complex64)
    pts = pins.constellation(mod)
    s = pts[rng.integers(0, len(pts), size=(N, J, U))]
    y = np.einsum("cnsu,nju->cnjs", H.astype(np.complex128), s)
    N0 = U * 10 ** (-snr_db / 10)
    if noise:
        y = y + np.sqrt(N0 / 2) * (rng.standard_normal(y.shape) + 1j * rng.standard_normal(y.shape))
    return H, y.astype(np.complex64), s, N0


def full_H(H, n=0):
    return pins.stack_uplink(H[:, n])


def full_y(y, n=0, j=0):
    return y[:, n, j, :].astype(np.complex128).reshape(-1)


# ------------------------------------------------------------------ linalg

@pytest.mark.parametrize("ex", GOLD["hpd_inverse"], ids=lambda e: e["cite"][:14])
def test_hpd_inverse_golden(oracle_mod, ex):
    M = np.array(ex["M_re"]) + 1j * np.array(ex["M_im"])
    ref = np.array(ex["inv_re"]) + 1j * np.array(ex["inv_im"])
    assert np.allclose(oracle_mod.hpd_inverse(M), ref, atol=1e-14)


def test_hpd_inverse_residual_and_error(oracle_mod):
    rng = np.random.default_rng(1)
    for n in (1, 4, 16, 33, 64):
        A = rng.standard_normal((n + 3, n)) + 1j * rng.standard_normal((n + 3, n))
        G = A.conj().T @ A + 0.5 * np.eye(n)
        Gi = oracle_mod.hpd_inverse(G)
        assert np.max(np.abs(G @ Gi - np.eye(n))) < 1e-9     # SPEC S62
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.hpd_inverse(np.array([[1.0, 2.0], [2.0, 1.0]], dtype=complex))  # indefinite
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.hpd_inverse(np.array([[np.nan, 0], [0, 1.0]], dtype=complex))


# ------------------------------------------------------------------ slicer

@pytest.mark.parametrize("ex", GOLD["slice"], ids=lambda e: e["cite"][:14])
def test_slice_golden(oracle_mod, ex):
    b = oracle_mod.slice_bits(np.array([ex["x_re"] + 1j * ex["x_im"]]), ex["mod"])
    assert int(b[0]) == ex["bits"]


@pytest.mark.parametrize("mod", ["bpsk", "qpsk", "qam16", "qam64"])
def test_slice_brute_force(oracle_mod, mod):
    """Nearest point by exhaustive search (SPEC S170), Gray labels of the points."""
    rng = np.random.default_rng(7)
    x = (rng.standard_normal(20000) + 1j * rng.standard_normal(20000)) * 0.8
    if mod == "bpsk":
        x = x.real + 0j
    x = x.astype(np.complex64)
    pts = pins.constellation(mod)
    xd = x.astype(np.complex128)
    near = pts[np.argmin(np.abs(xd[:, None] - pts[None, :]), axis=1)]
    want = np.array([pins.gray_bits_of_point(p, mod) for p in near])
    got = oracle_mod.slice_bits(x, mod)
    assert np.array_equal(got, want)
    # every alphabet point maps to its own label; adjacent points differ in one bit
    labels = oracle_mod.slice_bits(pts.astype(np.complex64), mod)
    assert np.array_equal(labels, [pins.gray_bits_of_point(p, mod) for p in pts])
    dmin = np.min(np.abs(pts[:, None] - pts[None, :]) + 10 * np.eye(len(pts)))
    for a in range(len(pts)):
        for b in range(len(pts)):
            if a != b and abs(abs(pts[a] - pts[b]) - dmin) < 1e-9:
                assert bin(int(labels[a]) ^ int(labels[b])).count("1") == 1


# --------------------------------------------------------------- Algorithm 1

def test_admm_1x1_worked_example(oracle_mod):
    ex = GOLD["admm_1x1"]
    H = np.full((1, 1, 1, 1), ex["H"], dtype=np.complex64)
    y = np.full((1, 1, 1, 1), ex["y"], dtype=np.complex64)
    s, z, lam = oracle_mod.detect_admm_trace(H, y, rho=ex["rho"], N0=ex["N0"], Es=ex["Es"],
                                             T=1, mod="qpsk")
    assert abs(z[0, 0, 0] - ex["z1"]) < 1e-15 and abs(s[0, 0] - ex["s1"]) < 1e-15


@pytest.mark.parametrize("C", [1, 4])
def test_admm_converges_to_mmse(oracle_mod, C):
    """SPEC acceptance 1 (U=8, B=32, rho=1) -> centralized MMSE (P212).  The error
    decays geometrically (5e-3 @ T=50 ... 1e-15 @ T=800); T=400 gives < 1e-8."""
    rng = np.random.default_rng(11 + C)
    S = 32 // C
    for _ in range(5):
        H, y, _, N0 = rand_ul(rng, C, S, 8, N=2, J=2, snr_db=10)
        s_hat, _ = oracle_mod.detect_admm(H, y, rho=1.0, N0=N0, T=400, mod="qpsk")
        for n in range(2):
            for j in range(2):
                ref = pins.mmse(full_H(H, n), full_y(y, n, j), N0)
                assert pins.rel(s_hat[n, j], ref) < 1e-8


def test_admm_zf_converges_to_ls(oracle_mod):
    rng = np.random.default_rng(3)
    H, y, _, _ = rand_ul(rng, 4, 8, 6, snr_db=5)
    s_hat, _ = oracle_mod.detect_admm(H, y, reg="zf", rho=1.0, T=400, mod="qpsk")
    assert pins.rel(s_hat[0, 0], pins.ls(full_H(H), full_y(y))) < 1e-6


BOX_MODS = ["bpsk", "qpsk", "qam16", "qam64"]


def box_r(mod):
    """Box radius from the alphabet itself (largest per-axis coordinate, P343, reading 17)."""
    return float(np.max(pins.constellation(mod).real))


@pytest.mark.parametrize("mod", BOX_MODS)
def test_admm_box_converges_to_bounded_ls(oracle_mod, mod):
    """(E2-BOX) (P339-343): fixed point = box-constrained LS (scipy bvls) on the radius of
    each alphabet; BPSK (P344): real-valued s, the real-stacked system with Im(s) = 0."""
    rng = np.random.default_rng(5)
    r = box_r(mod)
    hits = 0
    for _ in range(4):
        H, y, _, _ = rand_ul(rng, 2, 4, 4, snr_db=0, mod=mod)
        s_hat, _ = oracle_mod.detect_admm(H, y, reg="box", rho=1.0, T=3000, mod=mod)
        if mod == "bpsk":
            ref = pins.box_ls_real(full_H(H), full_y(y), r)
            assert np.all(s_hat[0, 0].imag == 0)
        else:
            ref = pins.box_ls(full_H(H), full_y(y), r)
        hits += np.any(np.abs(np.abs(ref.real) - r) < 1e-9) + np.any(np.abs(np.abs(ref.imag) - r) < 1e-9)
        assert pins.rel(s_hat[0, 0], ref) < 1e-5
    assert hits > 0  # the box is active in at least one instance


@pytest.mark.parametrize("S,U", [(4, 8), (8, 8), (16, 8)])
def test_admm_mode_equivalence(oracle_mod, S, U):
    """Eq. (3) (U x U) vs eq. (4) (S x S, Woodbury): same iterates (SPEC acceptance 5)."""
    rng = np.random.default_rng(S)
    H, y, _, N0 = rand_ul(rng, 3, S, U, N=2, J=2)
    for T in (1, 2, 7):
        a, _ = oracle_mod.detect_admm(H, y, rho=0.7, N0=N0, T=T, mode="uu", mod="qpsk")
        b, _ = oracle_mod.detect_admm(H, y, rho=0.7, N0=N0, T=T, mode="ss", mod="qpsk")
        assert pins.rel(a, b) < 1e-9


@pytest.mark.parametrize("reg,mod", [("mmse", "qpsk"), ("zf", "qpsk")] + [("box", m) for m in BOX_MODS])
def test_admm_steps_satisfy_E1_E2_E3(oracle_mod, reg, mod):
    """Every iterate satisfies the optimality conditions of (E1), (E2)/Lemma 1 and
    the update (E3) as reordered by Alg. 1 (P238-249, P304-312, P356-357).  BOX runs
    every alphabet's radius (P343) at 0 dB so the clamp is active; BPSK projects onto
    the real segment [-1, 1] (P344)."""
    rng = np.random.default_rng(17)
    C, S, U, rho, gamma, T = 3, 6, 4, 0.8, 1.0, 6
    H, y, _, N0 = rand_ul(rng, C, S, U, snr_db=0 if reg == "box" else 5, mod=mod)
    s, z, lam = oracle_mod.detect_admm_trace(H, y, rho=rho, gamma=gamma, N0=N0, reg=reg, T=T,
                                             mod=mod)
    Hc = [H[c, 0].astype(np.complex128) for c in range(C)]
    yc = [y[c, 0, 0].astype(np.complex128) for c in range(C)]
    r = box_r(mod)
    clipped = 0
    for t in range(T):
        for c in range(C):
            sp = s[t - 1] if t > 0 else np.zeros(U)
            # (E1): H^H (H z - y) - rho (s - z - lam) = 0   (t = 1: s = 0, lam = 0)
            g = Hc[c].conj().T @ (Hc[c] @ z[t, c] - yc[c]) - rho * (sp - z[t, c] - lam[t, c])
            assert np.linalg.norm(g) < 1e-10
            if t > 0:  # Alg. 1 line 12 (E3 reordered)
                assert np.allclose(lam[t, c], lam[t - 1, c] + gamma * (z[t - 1, c] - s[t - 1]),
                                   atol=1e-12)
        w = sum(z[t, c] + lam[t, c] for c in range(C))
        if reg == "mmse":   # (E2) with g = N0/(2Es)||s||^2: N0 s + rho sum_c (s - w_c) = 0
            assert np.linalg.norm(N0 * s[t] + rho * (C * s[t] - w)) < 1e-10
        elif reg == "zf":
            assert np.linalg.norm(C * s[t] - w) < 1e-10
        else:               # projection of v = w/C onto the box (Lemma 1 + P343; BPSK P344)
            v = w / C
            if mod == "bpsk":
                want = np.clip(v.real, -r, r) + 0j
                clipped += int(np.sum(np.abs(v.real) > r))
            else:
                want = np.clip(v.real, -r, r) + 1j * np.clip(v.imag, -r, r)
                clipped += int(np.sum(np.abs(v.real) > r) + np.sum(np.abs(v.imag) > r))
            assert np.allclose(s[t], want, atol=1e-12)
    if reg == "box":
        assert clipped > 0   # the radius constant is exercised, not just the identity branch


def test_admm_invariances(oracle_mod):
    """Linearity in y, cluster-unitary invariance, user permutation."""
    rng = np.random.default_rng(23)
    C, S, U = 4, 6, 4
    H, y1, _, N0 = rand_ul(rng, C, S, U, N=2)
    _, y2, _, _ = rand_ul(rng, C, S, U, N=2)
    kw = dict(rho=1.3, N0=N0, T=4, mod="qpsk")
    a, _ = oracle_mod.detect_admm(H, y1, **kw)
    b, _ = oracle_mod.detect_admm(H, y2, **kw)
    ab, _ = oracle_mod.detect_admm(H, (0.5 * y1.astype(np.complex128) - 2j * y2).astype(np.complex64), **kw)
    assert pins.rel(ab, 0.5 * a - 2j * b) < 1e-6  # fp32 rounding of the combined input
    Q = np.linalg.qr(rng.standard_normal((C, S, S)) + 1j * rng.standard_normal((C, S, S)))[0]
    HQ = np.einsum("cab,cnbu->cnau", Q, H.astype(np.complex128))
    yQ = np.einsum("cab,cnjb->cnja", Q, y1.astype(np.complex128))
    q, _ = oracle_mod.detect_admm(HQ.astype(np.complex64), yQ.astype(np.complex64), **kw)
    assert pins.rel(q, a) < 1e-6
    perm = rng.permutation(U)
    p, _ = oracle_mod.detect_admm(np.ascontiguousarray(H[..., perm]), y1, **kw)
    assert pins.rel(p, a[..., perm]) < 1e-12


def test_admm_noise_free_matches_ml(oracle_mod):
    """Noise-free tiny QPSK: brute-force ML = transmitted s = slice(ADMM-ZF)."""
    rng = np.random.default_rng(29)
    for _ in range(10):
        H, y, s, _ = rand_ul(rng, 2, 4, 3, noise=False)
        ml = pins.brute_force_ml(full_H(H), full_y(y), "qpsk")
        assert np.allclose(ml, s[0, 0])
        s_hat, hard = oracle_mod.detect_admm(H, y, reg="zf", T=300, mod="qpsk")
        assert np.array_equal(hard[0, 0], [pins.gray_bits_of_point(p, "qpsk") for p in ml])


# --------------------------------------------------------------- Algorithm 2

def test_cg_exact_after_U_steps(oracle_mod):
    """SPEC acceptance 2 / S260: T = U iterations solve (rho I + H^H H) x = H^H y."""
    rng = np.random.default_rng(31)
    for C in (1, 4):
        H, y, _, N0 = rand_ul(rng, C, 32 // C, 8, N=2, J=2)
        x, _ = oracle_mod.detect_cg(H, y, rho=N0, T=8, mod="qpsk")
        for n in range(2):
            for j in range(2):
                assert pins.rel(x[n, j], pins.mmse(full_H(H, n), full_y(y, n, j), N0)) < 1e-10


def test_cg_matches_centralized_textbook_cg(oracle_mod):
    """Decentralized CG = centralized CG iterate by iterate (north star; eq. (7) P379)."""
    rng = np.random.default_rng(37)
    H, y, _, N0 = rand_ul(rng, 4, 8, 8)
    T = 6
    x, r, p = oracle_mod.detect_cg_trace(H, y, rho=N0, T=T)
    Hf, yf = full_H(H), full_y(y)
    A = N0 * np.eye(8) + Hf.conj().T @ Hf
    ref = pins.textbook_cg(A, Hf.conj().T @ yf, T)
    for t in range(T + 1):
        assert pins.rel(x[t], ref[t]) < 1e-12
        assert pins.rel(r[t], Hf.conj().T @ yf - A @ x[t]) < 1e-9   # r is the true residual


def test_cg_krylov_optimality(oracle_mod):
    """x^(t) minimises the A-norm error over K_t(A, y^MRC) for every finite t."""
    rng = np.random.default_rng(41)
    H, y, _, N0 = rand_ul(rng, 2, 16, 8, snr_db=10)
    x, _, _ = oracle_mod.detect_cg_trace(H, y, rho=N0, T=7)
    Hf, yf = full_H(H), full_y(y)
    A = N0 * np.eye(8) + Hf.conj().T @ Hf
    for t in range(1, 8):
        assert pins.rel(x[t], pins.krylov_minimizer(A, Hf.conj().T @ yf, t)) < 1e-8


def test_cg_special_cases(oracle_mod):
    rng = np.random.default_rng(43)
    # orthonormal columns, rho = 0: system matrix = I, exact after one step (S261)
    Q = np.linalg.qr(rng.standard_normal((16, 4)) + 1j * rng.standard_normal((16, 4)))[0]
    H = Q.reshape(2, 1, 8, 4).astype(np.complex64)
    y = (rng.standard_normal((2, 1, 1, 8)) + 1j * rng.standard_normal((2, 1, 1, 8))).astype(np.complex64)
    x, _ = oracle_mod.detect_cg(H, y, rho=0.0, T=1, mod="qpsk")
    assert pins.rel(x[0, 0], full_H(H).conj().T @ full_y(y)) < 1e-6
    # y = 0 -> x = 0, with r = 0 freezing the iteration (reading 4)
    x0, _ = oracle_mod.detect_cg(H, np.zeros_like(y), rho=0.1, T=3, mod="qpsk")
    assert np.all(x0 == 0)
    # homogeneity x(a y) = a x(y) for complex a (SURVEY 8(c) invariants)
    H, y, _, N0 = rand_ul(rng, 2, 8, 8)
    a, _ = oracle_mod.detect_cg(H, y, rho=N0, T=3, mod="qpsk")
    b, _ = oracle_mod.detect_cg(H, (y.astype(np.complex128) * (0.5 + 0.25j)).astype(np.complex64),
                                rho=N0, T=3, mod="qpsk")
    assert pins.rel(b, (0.5 + 0.25j) * a) < 1e-6


# --------------------------------------------------------------- Algorithm 3

def rand_dl(rng, C, S, U, N=1, J=1, mod="qam16"):
    Hd = ((rng.standard_normal((C, N, U, S)) + 1j * rng.standard_normal((C, N, U, S))) /
          np.sqrt(2)).astype(np.complex64)
    pts = pins.constellation(mod)
    s = pts[rng.integers(0, len(pts), size=(N, J, U))].astype(np.complex64)
    return Hd, s


def full_Hd(Hd, n=0):
    return np.concatenate([Hd[c, n].astype(np.complex128) for c in range(Hd.shape[0])], axis=1)


def test_bf_converges_to_zf(oracle_mod):
    """SPEC acceptance 3: U=8, B=32, C=4, eps=0, rho=1, T=300 -> ZF (P431) to 1e-3."""
    rng = np.random.default_rng(53)
    for _ in range(5):
        Hd, s = rand_dl(rng, 4, 8, 8, mod="qpsk")
        x = oracle_mod.beamform_admm(Hd, s, rho=1.0, T=300)
        xf = np.concatenate([x[c, 0, 0] for c in range(4)])
        ref = pins.zf_precoder(full_Hd(Hd), s[0, 0].astype(np.complex128))
        assert pins.rel(xf, ref) < 1e-3
        assert pins.rel(full_Hd(Hd) @ xf, s[0, 0]) < 1e-3


@pytest.mark.parametrize("eps", [0.0, 0.3])
def test_bf_steps_satisfy_P1_P2_P3(oracle_mod, eps):
    """(P1) stationarity, (P2) = Lemma 2 projection KKT, (P3) update (P453-455, P538)."""
    rng = np.random.default_rng(59)
    C, S, U, rho, gamma, T = 3, 6, 4, 0.9, 1.0, 6
    Hd, s = rand_dl(rng, C, S, U)
    x, z, lam, w = oracle_mod.beamform_admm_trace(Hd, s, rho=rho, gamma=gamma, eps=eps, T=T)
    Hc = [Hd[c, 0].astype(np.complex128) for c in range(C)]
    sv = s[0, 0].astype(np.complex128)
    for t in range(T):
        for c in range(C):
            # (P1): x + rho H^H (H x - z - lam) = 0
            g = x[t, c] + rho * Hc[c].conj().T @ (Hc[c] @ x[t, c] - z[t, c] - lam[t, c])
            assert np.linalg.norm(g) < 1e-10
        if t == 0:
            continue
        wc = np.stack([Hc[c] @ x[t - 1, c] - lam[t - 1, c] for c in range(C)])
        assert np.allclose(wc, w[t], atol=1e-12)                          # Alg. 3 line 12
        d = z[t] - wc                                                     # projection step
        assert np.allclose(d, d[0][None, :], atol=1e-12)                  # same for every c
        res = sv - z[t].sum(axis=0)
        if eps == 0:
            assert np.linalg.norm(res) < 1e-12                            # sum_c z_c = s
        else:
            assert np.linalg.norm(res) <= eps * (1 + 1e-12)
            mu = np.vdot(res, d[0]) / max(np.vdot(res, res).real, 1e-300)
            assert np.linalg.norm(d[0] - mu * res) < 1e-10 and mu.real >= -1e-12
            if np.linalg.norm(sv - wc.sum(axis=0)) <= eps:
                assert np.allclose(d, 0)
        for c in range(C):                                                # (P3), line 15
            m = Hc[c] @ x[t - 1, c]
            assert np.allclose(lam[t, c], lam[t - 1, c] - gamma * (m - z[t, c]), atol=1e-12)


def test_bf_consensus_project_golden(oracle_mod):
    ex = GOLD["consensus_project"]
    Hd = np.zeros((ex["C"], 1, 2, 3), dtype=np.complex64)        # x_c = 0 -> w_c = -lambda_c = 0
    s = np.array(ex["s"], dtype=np.complex64).reshape(1, 1, 2)
    _, z, _, _ = oracle_mod.beamform_admm_trace(Hd, s, rho=1.0, T=2)
    assert np.allclose(z[1], np.array(ex["z"])[None, :], atol=1e-15)


@pytest.mark.parametrize("ex", GOLD["bf_init_scale"], ids=lambda e: e["cite"][:14])
def test_bf_init_scale_golden(oracle_mod, ex):
    rng = np.random.default_rng(61)
    Hd, s = rand_dl(rng, ex["C"], ex["S"], ex["U"])
    _, z, _, _ = oracle_mod.beamform_admm_trace(Hd, s, T=1)
    assert np.allclose(z[0], ex["scale"] * s[0, 0][None, :].astype(np.complex128), atol=1e-15)


def test_bf_first_iteration_is_local(oracle_mod):
    """T = 1 needs no consensus (P811): x_c^(1) depends on cluster c's data only."""
    rng = np.random.default_rng(67)
    Hd, s = rand_dl(rng, 4, 8, 4)
    x1 = oracle_mod.beamform_admm(Hd, s, T=1)
    Hd2 = Hd.copy()
    Hd2[2] = rng.standard_normal(Hd2[2].shape)
    x2 = oracle_mod.beamform_admm(Hd2, s, T=1)
    assert np.array_equal(x1[[0, 1, 3]], x2[[0, 1, 3]]) and not np.allclose(x1[2], x2[2])
    x3 = oracle_mod.beamform_admm(Hd2, s, T=2)
    assert not np.allclose(x3[0], x2[0])                  # from t = 2 on, consensus couples


@pytest.mark.parametrize("S,U", [(4, 8), (8, 8), (16, 8)])
def test_bf_mode_equivalence(oracle_mod, S, U):
    rng = np.random.default_rng(71 + S)
    Hd, s = rand_dl(rng, 3, S, U, N=2, J=2)
    for T in (1, 3):
        a = oracle_mod.beamform_admm(Hd, s, rho=0.8, T=T, mode="uu")
        b = oracle_mod.beamform_admm(Hd, s, rho=0.8, T=T, mode="ss")
        assert pins.rel(a, b) < 1e-8


def test_bf_invariances(oracle_mod):
    rng = np.random.default_rng(73)
    C, S, U = 3, 8, 4
    Hd, s1 = rand_dl(rng, C, S, U)
    _, s2 = rand_dl(rng, C, S, U)
    a = oracle_mod.beamform_admm(Hd, s1, T=4)
    b = oracle_mod.beamform_admm(Hd, s2, T=4)
    ab = oracle_mod.beamform_admm(Hd, (2 * s1 + 1j * s2).astype(np.complex64), T=4)
    assert pins.rel(ab, 2 * a + 1j * b) < 1e-6
    Q = np.linalg.qr(rng.standard_normal((C, S, S)) + 1j * rng.standard_normal((C, S, S)))[0]
    HQ = np.einsum("cnus,cst->cnut", Hd.astype(np.complex128), Q).astype(np.complex64)
    q = oracle_mod.beamform_admm(HQ, s1, T=4)
    back = np.einsum("cst,cnjt->cnjs", Q, q)     # H_c -> H_c Q_c gives x_c = Q_c x'_c
    assert pins.rel(back, a) < 1e-5
