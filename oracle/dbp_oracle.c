/*
 * dbp_oracle.c -- plain, slow, obviously-correct double-precision oracle for
 * Algorithms 1-3 of Li et al., "Decentralized Baseband Processing for Massive
 * MU-MIMO Systems", arXiv 1702.04458.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py.  Never part of the product
 * path; shares no code with paper_1702_04458_b200/csrc/.
 *
 * Every algorithm is written step by step in the paper's order and notation,
 * one subcarrier n and one symbol j at a time, clusters c = 0..C-1 summed in
 * that fixed order (SPEC S398).  No blocking, no fusion, no reordering.  The
 * only parallelism is an OpenMP loop over independent subcarriers (P706).
 *
 * Parity pins (tests/test_oracle_*.py): see DESIGN.md section 4.  No function
 * here is "parity unpinned".
 */
#include "dbp_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cd;

/* ---------------------------------------------------------------- helpers */

static cd ldf(const float* p, size_t idx) { return (double)p[2 * idx] + I * (double)p[2 * idx + 1]; }
static cd ldd(const double* p, size_t idx) { return p[2 * idx] + I * p[2 * idx + 1]; }
static void std_(double* p, size_t idx, cd v) { p[2 * idx] = creal(v); p[2 * idx + 1] = cimag(v); }

/* y = A x, A: r x k row-major */
static void matvec(int r, int k, const cd* A, const cd* x, cd* y) {
    for (int i = 0; i < r; ++i) {
        cd acc = 0;
        for (int j = 0; j < k; ++j) acc += A[i * k + j] * x[j];
        y[i] = acc;
    }
}

/* y = A^H x, A: r x k row-major, y has k entries */
static void matvec_h(int r, int k, const cd* A, const cd* x, cd* y) {
    for (int j = 0; j < k; ++j) {
        cd acc = 0;
        for (int i = 0; i < r; ++i) acc += conj(A[i * k + j]) * x[i];
        y[j] = acc;
    }
}

/* G = A^H A + delta I  (k x k), A: r x k */
static void gram_cols(int r, int k, const cd* A, double delta, cd* G) {
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
            cd acc = 0;
            for (int s = 0; s < r; ++s) acc += conj(A[s * k + i]) * A[s * k + j];
            G[i * k + j] = acc + (i == j ? delta : 0.0);
        }
}

/* G = A A^H + delta I  (r x r), A: r x k */
static void gram_rows(int r, int k, const cd* A, double delta, cd* G) {
    for (int i = 0; i < r; ++i)
        for (int j = 0; j < r; ++j) {
            cd acc = 0;
            for (int s = 0; s < k; ++s) acc += A[i * k + s] * conj(A[j * k + s]);
            G[i * r + j] = acc + (i == j ? delta : 0.0);
        }
}

/* Cholesky G = L L^H, L lower triangular with real positive diagonal.
 * Returns 0, or 3 if a pivot is <= 0 or non-finite (SPEC S44, S68-69). */
static int cholesky(int n, const cd* G, cd* L) {
    for (int i = 0; i < n * n; ++i) L[i] = 0;
    for (int j = 0; j < n; ++j) {
        double d = creal(G[j * n + j]);
        for (int k = 0; k < j; ++k) d -= creal(L[j * n + k] * conj(L[j * n + k]));
        if (!(d > 0.0) || !isfinite(d)) return 3;
        double ljj = sqrt(d);
        L[j * n + j] = ljj;
        for (int i = j + 1; i < n; ++i) {
            cd acc = G[i * n + j];
            for (int k = 0; k < j; ++k) acc -= L[i * n + k] * conj(L[j * n + k]);
            L[i * n + j] = acc / ljj;
        }
    }
    return 0;
}

/* G^{-1} for Hermitian positive-definite G: Cholesky, then for each unit
 * vector e_k a forward substitution L u = e_k and a backward substitution
 * L^H x = u (P704: "matrix inversions via the Cholesky factorization followed
 * by forward-backward substitution"). */
static int hpd_inverse(int n, const cd* G, cd* Ginv) {
    cd* L = malloc(sizeof(cd) * n * n);
    cd* u = malloc(sizeof(cd) * n);
    cd* x = malloc(sizeof(cd) * n);
    int st = cholesky(n, G, L);
    if (st == 0) {
        for (int k = 0; k < n; ++k) {
            for (int i = 0; i < n; ++i) {
                cd acc = (i == k) ? 1.0 : 0.0;
                for (int m = 0; m < i; ++m) acc -= L[i * n + m] * u[m];
                u[i] = acc / L[i * n + i];
            }
            for (int i = n - 1; i >= 0; --i) {
                cd acc = u[i];
                for (int m = i + 1; m < n; ++m) acc -= conj(L[m * n + i]) * x[m];
                x[i] = acc / conj(L[i * n + i]);
            }
            for (int i = 0; i < n; ++i) Ginv[i * n + k] = x[i];
        }
    }
    free(L); free(u); free(x);
    return st;
}

int dbpo_hpd_inverse(int n, const double* G, double* Ginv) {
    if (n < 1 || !G || !Ginv) return 1;
    cd* g = malloc(sizeof(cd) * n * n);
    cd* gi = malloc(sizeof(cd) * n * n);
    for (int i = 0; i < n * n; ++i) g[i] = ldd(G, i);
    int st = hpd_inverse(n, g, gi);
    if (st == 0) for (int i = 0; i < n * n; ++i) std_(Ginv, i, gi[i]);
    free(g); free(gi);
    return st;
}

/* ------------------------------------------------------------ constellation */

/* Gray QAM with Es = 1 (reading 17): per-axis levels (2k-(m-1))/sqrt(norm),
 * m levels per axis.  Returns levels per axis (1 axis for BPSK). */
static int axis_levels(int mod, float* scale, int* naxes) {
    switch (mod) {
        case DBPO_BPSK:  *scale = 1.0f;        *naxes = 1; return 2;
        case DBPO_QPSK:  *scale = 1.41421356f; *naxes = 2; return 2; /* sqrt(2)  */
        case DBPO_QAM16: *scale = 3.16227766f; *naxes = 2; return 4; /* sqrt(10) */
        case DBPO_QAM64: *scale = 6.48074070f; *naxes = 2; return 8; /* sqrt(42) */
        default: return 0;
    }
}

/* Box radius r = largest per-axis coordinate (P343, reading 17). */
static double box_radius(int mod) {
    switch (mod) {
        case DBPO_BPSK:  return 1.0;
        case DBPO_QPSK:  return 1.0 / sqrt(2.0);
        case DBPO_QAM16: return 3.0 / sqrt(10.0);
        case DBPO_QAM64: return 7.0 / sqrt(42.0);
        default: return 0.0;
    }
}

/* Nearest level index on one axis, decided in fp32 (reading 19):
 * k = clamp(ceil((x*scale + m)/2) - 1, 0, m-1); exact ties go down. */
static int slice_axis(float x, int m, float scale) {
    volatile float t = x * scale;           /* no contraction into an fma */
    volatile float u = (t + (float)m) * 0.5f;
    float k = ceilf(u) - 1.0f;
    if (!(k >= 0.0f)) return 0;             /* also catches NaN */
    if (k > (float)(m - 1)) return m - 1;
    return (int)k;
}

static unsigned gray(unsigned k) { return k ^ (k >> 1); }

int dbpo_slice(int mod, int64_t count, const float* x, uint8_t* bits) {
    float scale; int naxes;
    int m = axis_levels(mod, &scale, &naxes);
    if (!m || count < 0 || (count && (!x || !bits))) return 1;
    int bpa = (m == 2) ? 1 : (m == 4) ? 2 : 3;
    for (int64_t i = 0; i < count; ++i) {
        unsigned gi = gray((unsigned)slice_axis(x[2 * i], m, scale));
        if (naxes == 1) { bits[i] = (uint8_t)gi; continue; }
        unsigned gq = gray((unsigned)slice_axis(x[2 * i + 1], m, scale));
        bits[i] = (uint8_t)((gi << bpa) | gq);
    }
    return 0;
}

/* ---------------------------------------------------------- argument checks */

static int dims_ok(const dbpo_dims* d) {
    return d && d->C >= 1 && d->S >= 1 && d->U >= 1 && d->N >= 1 && d->N_sym >= 1;
}

static int use_ss_mode(int mode, int S, int U) {
    if (mode == DBPO_MODE_SS) return 1;
    if (mode == DBPO_MODE_UU) return 0;
    return S <= U; /* Alg. 1 line 3 (P290), Alg. 3 line 3 (P500) */
}

/* ================================================= Algorithm 1: ADMM uplink */

/* Proximal step (E2), Lemma 1 (P325-344): s = prox_g(v), v = w / C.
 * MMSE uses Alg. 1 line 13 form s = (N0/(rho Es) + C)^{-1} w (P312). */
static cd prox_ul(cd w, int reg, int mod, int C, double rho, double N0, double Es) {
    if (reg == DBPO_REG_MMSE) return w / (N0 / (rho * Es) + (double)C);
    cd v = w / (double)C;
    if (reg == DBPO_REG_ZF) return v;                               /* (E2-ZF)   */
    double r = box_radius(mod);
    double re = creal(v), im = cimag(v);
    re = (re > 0 ? 1.0 : re < 0 ? -1.0 : 0.0) * fmin(fabs(re), r); /* (E2-BOX)  */
    im = (im > 0 ? 1.0 : im < 0 ? -1.0 : 0.0) * fmin(fabs(im), r);
    if (mod == DBPO_BPSK) im = 0.0;                                 /* BPSK, P344 */
    return re + I * im;
}

typedef struct {
    int C, S, U, ss;
    cd* Hn;    /* [C][S][U] for this subcarrier */
    cd* inv;   /* UxU mode: B_c^{-1} [C][U][U]; SxS mode: A_c^{-1} [C][S][S] */
} ul_pre;

/* Preprocessing, Alg. 1 lines 2-8 (P289-298). */
static int admm_ul_preprocess(ul_pre* P, double rho) {
    int C = P->C, S = P->S, U = P->U;
    int n = P->ss ? S : U;
    cd* G = malloc(sizeof(cd) * n * n);
    int st = 0;
    for (int c = 0; c < C && st == 0; ++c) {
        const cd* Hc = P->Hn + (size_t)c * S * U;
        if (P->ss) gram_rows(S, U, Hc, rho, G); /* A_c = H_c H_c^H + rho I_S (line 4) */
        else       gram_cols(S, U, Hc, rho, G); /* B_c = H_c^H H_c + rho I_U (line 7) */
        st = hpd_inverse(n, G, P->inv + (size_t)c * n * n);
    }
    free(G);
    return st;
}

/* y_c^reg (Alg. 1 line 5 or line 8). */
static void admm_ul_yreg(const ul_pre* P, int c, const cd* yc, cd* yreg) {
    int S = P->S, U = P->U;
    const cd* Hc = P->Hn + (size_t)c * S * U;
    if (P->ss) {
        cd* t = malloc(sizeof(cd) * S);
        matvec(S, S, P->inv + (size_t)c * S * S, yc, t); /* A_c^{-1} y_c   */
        matvec_h(S, U, Hc, t, yreg);                      /* H_c^H (.)      */
        free(t);
    } else {
        cd* t = malloc(sizeof(cd) * U);
        matvec_h(S, U, Hc, yc, t);                        /* H_c^H y_c      */
        matvec(U, U, P->inv + (size_t)c * U * U, t, yreg);/* B_c^{-1} (.)   */
        free(t);
    }
}

/* z_c = y_c^reg + E1-operator (s - lambda_c): Alg. 1 line 13 (S<=U) or 15. */
static void admm_ul_zupdate(const ul_pre* P, int c, const cd* yreg, const cd* d,
                            double rho, cd* z) {
    int S = P->S, U = P->U;
    const cd* Hc = P->Hn + (size_t)c * S * U;
    if (P->ss) {
        /* z = yreg + d - H^H A^{-1} H d   (eq. 4, P277) */
        cd* t1 = malloc(sizeof(cd) * S);
        cd* t2 = malloc(sizeof(cd) * S);
        cd* t3 = malloc(sizeof(cd) * U);
        matvec(S, U, Hc, d, t1);
        matvec(S, S, P->inv + (size_t)c * S * S, t1, t2);
        matvec_h(S, U, Hc, t2, t3);
        for (int u = 0; u < U; ++u) z[u] = yreg[u] + d[u] - t3[u];
        free(t1); free(t2); free(t3);
    } else {
        /* z = yreg + rho B^{-1} d   (eq. 3, P272) */
        cd* t = malloc(sizeof(cd) * U);
        matvec(U, U, P->inv + (size_t)c * U * U, d, t);
        for (int u = 0; u < U; ++u) z[u] = yreg[u] + rho * t[u];
        free(t);
    }
}

/* ADMM iterations of Alg. 1 (lines 9-21) for one (n, j). */
static void admm_ul_iterate(const ul_pre* P, const cd* ycs /* [C][S] */, double rho,
                            double gamma, double N0, double Es, int reg, int mod,
                            int T, cd* s, double* s_tr, double* z_tr, double* lam_tr) {
    int C = P->C, S = P->S, U = P->U;
    cd* yreg = malloc(sizeof(cd) * C * U);
    cd* z = malloc(sizeof(cd) * C * U);
    cd* lam = malloc(sizeof(cd) * C * U);
    cd* w = malloc(sizeof(cd) * U);
    cd* d = malloc(sizeof(cd) * U);
    for (int c = 0; c < C; ++c) admm_ul_yreg(P, c, ycs + (size_t)c * S, yreg + (size_t)c * U);

    /* Init (line 10): lambda_c = 0, z_c = y_c^reg, s = prox(sum_c z_c). */
    for (int u = 0; u < U; ++u) w[u] = 0;
    for (int c = 0; c < C; ++c)
        for (int u = 0; u < U; ++u) {
            lam[c * U + u] = 0;
            z[c * U + u] = yreg[c * U + u];
            w[u] += z[c * U + u];
        }
    for (int u = 0; u < U; ++u) s[u] = prox_ul(w[u], reg, mod, C, rho, N0, Es);
    if (s_tr) {
        for (int u = 0; u < U; ++u) std_(s_tr, u, s[u]);
        for (int i = 0; i < C * U; ++i) { std_(z_tr, i, z[i]); std_(lam_tr, i, lam[i]); }
    }

    for (int t = 2; t <= T; ++t) {                      /* line 11 */
        for (int u = 0; u < U; ++u) w[u] = 0;
        for (int c = 0; c < C; ++c) {
            cd* zc = z + (size_t)c * U;
            cd* lc = lam + (size_t)c * U;
            for (int u = 0; u < U; ++u) lc[u] = lc[u] + gamma * (zc[u] - s[u]); /* line 12 */
            for (int u = 0; u < U; ++u) d[u] = s[u] - lc[u];
            admm_ul_zupdate(P, c, yreg + (size_t)c * U, d, rho, zc);             /* lines 13-16 */
            for (int u = 0; u < U; ++u) w[u] += zc[u] + lc[u];                   /* lines 17-18 */
        }
        for (int u = 0; u < U; ++u) s[u] = prox_ul(w[u], reg, mod, C, rho, N0, Es); /* line 19 */
        if (s_tr) {
            size_t o = (size_t)(t - 1);
            for (int u = 0; u < U; ++u) std_(s_tr, o * U + u, s[u]);
            for (int i = 0; i < C * U; ++i) {
                std_(z_tr, o * C * U + i, z[i]);
                std_(lam_tr, o * C * U + i, lam[i]);
            }
        }
    }
    free(yreg); free(z); free(lam); free(w); free(d);
}

static int admm_ul_run(const dbpo_dims* d, const float* H, const float* y, double rho,
                       double gamma, double N0, double Es, int reg, int mod, int T,
                       int mode, double* s_hat, uint8_t* hard, int n_tr, int j_tr,
                       double* s_tr, double* z_tr, double* lam_tr) {
    if (!dims_ok(d) || !H || !y || T < 1 || !(rho > 0) || !(gamma > 0) || !(Es > 0) ||
        !(N0 >= 0) || reg < 0 || reg > 2)
        return 1;
    float sc; int nax;
    if (!axis_levels(mod, &sc, &nax)) return 1;
    const int C = d->C, S = d->S, U = d->U, N = d->N, J = d->N_sym;
    const int ss = use_ss_mode(mode, S, U);
    int status = 0;
#pragma omp parallel for schedule(dynamic) reduction(max : status)
    for (int n = 0; n < N; ++n) {
        if (s_tr && n != n_tr) continue;
        ul_pre P = {C, S, U, ss, NULL, NULL};
        int m = ss ? S : U;
        P.Hn = malloc(sizeof(cd) * C * S * U);
        P.inv = malloc(sizeof(cd) * C * m * m);
        cd* ycs = malloc(sizeof(cd) * C * S);
        cd* s = malloc(sizeof(cd) * U);
        for (int c = 0; c < C; ++c)
            for (int i = 0; i < S * U; ++i)
                P.Hn[(size_t)c * S * U + i] = ldf(H, ((size_t)c * N + n) * S * U + i);
        int st = admm_ul_preprocess(&P, rho);
        for (int j = 0; j < J && st == 0; ++j) {
            if (s_tr && j != j_tr) continue;
            for (int c = 0; c < C; ++c)
                for (int k = 0; k < S; ++k)
                    ycs[(size_t)c * S + k] = ldf(y, (((size_t)c * N + n) * J + j) * S + k);
            admm_ul_iterate(&P, ycs, rho, gamma, N0, Es, reg, mod, T, s,
                            s_tr, z_tr, lam_tr);
            if (s_hat)
                for (int u = 0; u < U; ++u) std_(s_hat, ((size_t)n * J + j) * U + u, s[u]);
            if (hard) {
                float f[64];
                for (int u = 0; u < U; ++u) { f[2 * u] = (float)creal(s[u]); f[2 * u + 1] = (float)cimag(s[u]); }
                dbpo_slice(mod, U, f, hard + ((size_t)n * J + j) * U);
            }
        }
        if (st > status) status = st;
        free(P.Hn); free(P.inv); free(ycs); free(s);
    }
    return status;
}

int dbpo_detect_admm(const dbpo_dims* d, const float* H, const float* y, double rho,
                     double gamma, double N0, double Es, int reg, int mod, int T, int mode,
                     double* s_hat, uint8_t* hard) {
    if (!s_hat || (d && d->U > 32)) return 1;
    return admm_ul_run(d, H, y, rho, gamma, N0, Es, reg, mod, T, mode, s_hat, hard,
                       -1, -1, NULL, NULL, NULL);
}

int dbpo_detect_admm_trace(const dbpo_dims* d, const float* H, const float* y, double rho,
                           double gamma, double N0, double Es, int reg, int mod, int T,
                           int mode, int n_tr, int j_tr, double* s_tr, double* z_tr,
                           double* lam_tr) {
    if (!s_tr || !z_tr || !lam_tr || !d || n_tr < 0 || n_tr >= d->N || j_tr < 0 ||
        j_tr >= d->N_sym)
        return 1;
    return admm_ul_run(d, H, y, rho, gamma, N0, Es, reg, mod, T, mode, NULL, NULL, n_tr,
                       j_tr, s_tr, z_tr, lam_tr);
}

/* ================================================== Algorithm 2: CG uplink */

/* One (n, j) of Alg. 2 (P383-413).  Readings: line 11 uses e^(t) (reading 1),
 * alpha = ||r||^2 / Re(p^H e) (reading 3), r = 0 freezes x (reading 4). */
static void cg_one(int C, int S, int U, const cd* Hn /* [C][S][U] */, const cd* ycs,
                   double rho, int T, cd* x, double* x_tr, double* r_tr, double* p_tr) {
    cd* r = malloc(sizeof(cd) * U);
    cd* p = malloc(sizeof(cd) * U);
    cd* w = malloc(sizeof(cd) * U);
    cd* e = malloc(sizeof(cd) * U);
    cd* t1 = malloc(sizeof(cd) * S);
    cd* t2 = malloc(sizeof(cd) * U);
    /* Preprocessing, lines 3-4: y^MRC = sum_c H_c^H y_c. */
    for (int u = 0; u < U; ++u) r[u] = 0;
    for (int c = 0; c < C; ++c) {
        matvec_h(S, U, Hn + (size_t)c * S * U, ycs + (size_t)c * S, t2);
        for (int u = 0; u < U; ++u) r[u] += t2[u];
    }
    /* Init, line 6: r = y^MRC, p = r, x = 0. */
    for (int u = 0; u < U; ++u) { p[u] = r[u]; x[u] = 0; }
    int stopped = 0;
    for (int t = 1; t <= T; ++t) {
        if (x_tr && t == 1)
            for (int u = 0; u < U; ++u) { std_(x_tr, u, x[u]); std_(r_tr, u, r[u]); std_(p_tr, u, p[u]); }
        double rr = 0;
        for (int u = 0; u < U; ++u) rr += creal(r[u] * conj(r[u]));
        if (rr == 0.0) stopped = 1;
        if (!stopped) {
            /* lines 9-11: w_c = H_c^H H_c p (two matvecs), w = sum_c w_c */
            for (int u = 0; u < U; ++u) w[u] = 0;
            for (int c = 0; c < C; ++c) {
                const cd* Hc = Hn + (size_t)c * S * U;
                matvec(S, U, Hc, p, t1);
                matvec_h(S, U, Hc, t1, t2);
                for (int u = 0; u < U; ++u) w[u] += t2[u];
            }
            for (int u = 0; u < U; ++u) e[u] = rho * p[u] + w[u];       /* line 13 */
            cd phe = 0;
            for (int u = 0; u < U; ++u) phe += conj(p[u]) * e[u];
            double alpha = rr / creal(phe);                              /* line 14 */
            for (int u = 0; u < U; ++u) x[u] = x[u] + alpha * p[u];      /* line 15 */
            for (int u = 0; u < U; ++u) r[u] = r[u] - alpha * e[u];      /* line 16 */
            double rr1 = 0;
            for (int u = 0; u < U; ++u) rr1 += creal(r[u] * conj(r[u]));
            double beta = rr1 / rr;                                      /* line 17 */
            for (int u = 0; u < U; ++u) p[u] = r[u] + beta * p[u];       /* line 18 */
        }
        if (x_tr)
            for (int u = 0; u < U; ++u) {
                std_(x_tr, (size_t)t * U + u, x[u]);
                std_(r_tr, (size_t)t * U + u, r[u]);
                std_(p_tr, (size_t)t * U + u, p[u]);
            }
    }
    if (x_tr && T == 0)
        for (int u = 0; u < U; ++u) { std_(x_tr, u, x[u]); std_(r_tr, u, r[u]); std_(p_tr, u, p[u]); }
    free(r); free(p); free(w); free(e); free(t1); free(t2);
}

static int cg_run(const dbpo_dims* d, const float* H, const float* y, double rho, int mod,
                  int T, double* x_hat, uint8_t* hard, int n_tr, int j_tr, double* x_tr,
                  double* r_tr, double* p_tr) {
    if (!dims_ok(d) || !H || !y || T < 1 || !(rho >= 0)) return 1;
    float sc; int nax;
    if (hard && !axis_levels(mod, &sc, &nax)) return 1;
    const int C = d->C, S = d->S, U = d->U, N = d->N, J = d->N_sym;
#pragma omp parallel for schedule(dynamic)
    for (int n = 0; n < N; ++n) {
        if (x_tr && n != n_tr) continue;
        cd* Hn = malloc(sizeof(cd) * C * S * U);
        cd* ycs = malloc(sizeof(cd) * C * S);
        cd* x = malloc(sizeof(cd) * U);
        for (int c = 0; c < C; ++c)
            for (int i = 0; i < S * U; ++i)
                Hn[(size_t)c * S * U + i] = ldf(H, ((size_t)c * N + n) * S * U + i);
        for (int j = 0; j < J; ++j) {
            if (x_tr && j != j_tr) continue;
            for (int c = 0; c < C; ++c)
                for (int k = 0; k < S; ++k)
                    ycs[(size_t)c * S + k] = ldf(y, (((size_t)c * N + n) * J + j) * S + k);
            cg_one(C, S, U, Hn, ycs, rho, T, x, x_tr, r_tr, p_tr);
            if (x_hat)
                for (int u = 0; u < U; ++u) std_(x_hat, ((size_t)n * J + j) * U + u, x[u]);
            if (hard) {
                float f[64];
                for (int u = 0; u < U; ++u) { f[2 * u] = (float)creal(x[u]); f[2 * u + 1] = (float)cimag(x[u]); }
                dbpo_slice(mod, U, f, hard + ((size_t)n * J + j) * U);
            }
        }
        free(Hn); free(ycs); free(x);
    }
    return 0;
}

int dbpo_detect_cg(const dbpo_dims* d, const float* H, const float* y, double rho, int mod,
                   int T, double* x_hat, uint8_t* hard) {
    if (!x_hat || (d && d->U > 32)) return 1;
    return cg_run(d, H, y, rho, mod, T, x_hat, hard, -1, -1, NULL, NULL, NULL);
}

int dbpo_detect_cg_trace(const dbpo_dims* d, const float* H, const float* y, double rho,
                         int T, int n_tr, int j_tr, double* x_tr, double* r_tr, double* p_tr) {
    if (!x_tr || !r_tr || !p_tr || !d || n_tr < 0 || n_tr >= d->N || j_tr < 0 ||
        j_tr >= d->N_sym)
        return 1;
    return cg_run(d, H, y, rho, DBPO_QPSK, T, NULL, NULL, n_tr, j_tr, x_tr, r_tr, p_tr);
}

/* ============================================ Algorithm 3: ADMM beamforming */

/* (P1) closed form, Alg. 3 line 8 / lines 17-21: x_c = A_c^{-1} H_c^H q (S<=U)
 * or H_c^H B_c^{-1} q (S>U), with q = z_c + lambda_c. */
static void bf_p1(int S, int U, int ss, const cd* Hc /* U x S */, const cd* inv,
                  const cd* q, cd* x) {
    if (ss) {
        cd* t = malloc(sizeof(cd) * S);
        matvec_h(U, S, Hc, q, t);   /* H_c^H q        */
        matvec(S, S, inv, t, x);    /* A_c^{-1} (.)   */
        free(t);
    } else {
        cd* t = malloc(sizeof(cd) * U);
        matvec(U, U, inv, q, t);    /* B_c^{-1} q     */
        matvec_h(U, S, Hc, t, x);   /* H_c^H (.)      */
        free(t);
    }
}

static void bf_one(int C, int S, int U, int ss, const cd* Hn /* [C][U][S] */,
                   const cd* inv, const cd* s, double gamma, double eps, int T,
                   cd* x /* [C][S] */, double* x_tr, double* z_tr, double* lam_tr,
                   double* w_tr) {
    const int B = C * S;
    const int m = ss ? S : U;
    cd* z = malloc(sizeof(cd) * C * U);
    cd* lam = malloc(sizeof(cd) * C * U);
    cd* mv = malloc(sizeof(cd) * C * U);
    cd* wc = malloc(sizeof(cd) * C * U);
    cd* w = malloc(sizeof(cd) * U);
    cd* q = malloc(sizeof(cd) * U);
    /* Init, lines 8-9: z_c = max{U/B, 1/C} s, lambda_c = 0, x_c = P1(z_c). */
    double a0 = fmax((double)U / (double)B, 1.0 / (double)C);
    for (int c = 0; c < C; ++c) {
        for (int u = 0; u < U; ++u) { z[c * U + u] = a0 * s[u]; lam[c * U + u] = 0; }
        for (int u = 0; u < U; ++u) q[u] = z[c * U + u] + lam[c * U + u];
        bf_p1(S, U, ss, Hn + (size_t)c * U * S, inv + (size_t)c * m * m, q, x + (size_t)c * S);
    }
    if (x_tr) {
        for (int i = 0; i < C * S; ++i) std_(x_tr, i, x[i]);
        for (int i = 0; i < C * U; ++i) { std_(z_tr, i, z[i]); std_(lam_tr, i, lam[i]); std_(w_tr, i, 0); }
    }
    for (int t = 2; t <= T; ++t) {                                   /* line 10 */
        for (int u = 0; u < U; ++u) w[u] = 0;
        for (int c = 0; c < C; ++c) {
            matvec(U, S, Hn + (size_t)c * U * S, x + (size_t)c * S, mv + (size_t)c * U); /* line 11 */
            for (int u = 0; u < U; ++u) {
                wc[c * U + u] = mv[c * U + u] - lam[c * U + u];                         /* line 12 */
                w[u] += wc[c * U + u];                                                 /* line 13 */
            }
        }
        /* line 14 / Lemma 2 (P538, proof P873-890, reading 8):
         * z_c = w_c + max{0, 1 - eps/||s - w||} (s - w)/C. */
        double f = 1.0;
        if (eps > 0) {
            double nrm = 0;
            for (int u = 0; u < U; ++u) nrm += creal((s[u] - w[u]) * conj(s[u] - w[u]));
            nrm = sqrt(nrm);
            f = (nrm > 0) ? fmax(0.0, 1.0 - eps / nrm) : 0.0;
        }
        for (int c = 0; c < C; ++c)
            for (int u = 0; u < U; ++u)
                z[c * U + u] = wc[c * U + u] + f * (s[u] - w[u]) / (double)C;
        for (int c = 0; c < C; ++c) {
            for (int u = 0; u < U; ++u)                                              /* line 15 */
                lam[c * U + u] = lam[c * U + u] - gamma * (mv[c * U + u] - z[c * U + u]);
            for (int u = 0; u < U; ++u) q[u] = z[c * U + u] + lam[c * U + u];
            bf_p1(S, U, ss, Hn + (size_t)c * U * S, inv + (size_t)c * m * m, q,     /* lines 16-21 */
                  x + (size_t)c * S);
        }
        if (x_tr) {
            size_t o = (size_t)(t - 1);
            for (int i = 0; i < C * S; ++i) std_(x_tr, o * C * S + i, x[i]);
            for (int i = 0; i < C * U; ++i) {
                std_(z_tr, o * C * U + i, z[i]);
                std_(lam_tr, o * C * U + i, lam[i]);
                std_(w_tr, o * C * U + i, wc[i]);
            }
        }
    }
    free(z); free(lam); free(mv); free(wc); free(w); free(q);
}

static int bf_run(const dbpo_dims* d, const float* Hd, const float* s, double rho,
                  double gamma, double eps, int T, int mode, double* xout, int n_tr,
                  int j_tr, double* x_tr, double* z_tr, double* lam_tr, double* w_tr) {
    if (!dims_ok(d) || !Hd || !s || T < 1 || !(rho > 0) || !(gamma > 0) || !(eps >= 0))
        return 1;
    const int C = d->C, S = d->S, U = d->U, N = d->N, J = d->N_sym;
    const int ss = use_ss_mode(mode, S, U);
    const int m = ss ? S : U;
    int status = 0;
#pragma omp parallel for schedule(dynamic) reduction(max : status)
    for (int n = 0; n < N; ++n) {
        if (x_tr && n != n_tr) continue;
        cd* Hn = malloc(sizeof(cd) * C * U * S);
        cd* inv = malloc(sizeof(cd) * C * m * m);
        cd* G = malloc(sizeof(cd) * m * m);
        cd* sv = malloc(sizeof(cd) * U);
        cd* x = malloc(sizeof(cd) * C * S);
        for (int c = 0; c < C; ++c)
            for (int i = 0; i < U * S; ++i)
                Hn[(size_t)c * U * S + i] = ldf(Hd, ((size_t)c * N + n) * U * S + i);
        /* Preprocessing, lines 2-6: inverses with rho^{-1} regularisation. */
        int st = 0;
        for (int c = 0; c < C && st == 0; ++c) {
            const cd* Hc = Hn + (size_t)c * U * S;
            if (ss) gram_cols(U, S, Hc, 1.0 / rho, G); /* A_c = H_c^H H_c + rho^-1 I_S */
            else    gram_rows(U, S, Hc, 1.0 / rho, G); /* B_c = H_c H_c^H + rho^-1 I_U */
            st = hpd_inverse(m, G, inv + (size_t)c * m * m);
        }
        for (int j = 0; j < J && st == 0; ++j) {
            if (x_tr && j != j_tr) continue;
            for (int u = 0; u < U; ++u) sv[u] = ldf(s, ((size_t)n * J + j) * U + u);
            bf_one(C, S, U, ss, Hn, inv, sv, gamma, eps, T, x, x_tr, z_tr, lam_tr, w_tr);
            if (xout)
                for (int c = 0; c < C; ++c)
                    for (int k = 0; k < S; ++k)
                        std_(xout, (((size_t)c * N + n) * J + j) * S + k, x[(size_t)c * S + k]);
        }
        if (st > status) status = st;
        free(Hn); free(inv); free(G); free(sv); free(x);
    }
    return status;
}

int dbpo_beamform_admm(const dbpo_dims* d, const float* Hd, const float* s, double rho,
                       double gamma, double eps, int T, int mode, double* x) {
    if (!x || (d && d->U > 32)) return 1;
    return bf_run(d, Hd, s, rho, gamma, eps, T, mode, x, -1, -1, NULL, NULL, NULL, NULL);
}

int dbpo_beamform_admm_trace(const dbpo_dims* d, const float* Hd, const float* s, double rho,
                             double gamma, double eps, int T, int mode, int n_tr, int j_tr,
                             double* x_tr, double* z_tr, double* lam_tr, double* w_tr) {
    if (!x_tr || !z_tr || !lam_tr || !w_tr || !d || n_tr < 0 || n_tr >= d->N || j_tr < 0 ||
        j_tr >= d->N_sym)
        return 1;
    return bf_run(d, Hd, s, rho, gamma, eps, T, mode, NULL, n_tr, j_tr, x_tr, z_tr, lam_tr,
                  w_tr);
}

/* ================================= centralized baselines (P210-218, P431, P594) */

/* MMSE-UL (P212-218; SPEC mmse_centralized S218-221): for the full array
 * H = [H_1; ...; H_C] (B x U, B = CS), x = (H^H H + (N0/Es) I_U)^{-1} H^H y,
 * with H^H H = sum_c H_c^H H_c and H^H y = sum_c H_c^H y_c summed in cluster
 * order.  N0 = 0 is ZF detection.  Solved by Cholesky + forward/backward
 * substitution (hpd_inverse, then one mat-vec). */
int dbpo_mmse_centralized(const dbpo_dims* d, const float* H, const float* y, double N0, double Es,
                          int mod, double* x_hat, uint8_t* hard) {
    if (!dims_ok(d) || !H || !y || !x_hat || !(N0 >= 0) || !(Es > 0) || d->U > 32) return 1;
    float sc; int nax;
    if (hard && !axis_levels(mod, &sc, &nax)) return 1;
    const int C = d->C, S = d->S, U = d->U, N = d->N, J = d->N_sym;
    int status = 0;
#pragma omp parallel for schedule(dynamic)
    for (int n = 0; n < N; ++n) {
        cd* G = malloc(sizeof(cd) * U * U);
        cd* Gc = malloc(sizeof(cd) * U * U);
        cd* Gi = malloc(sizeof(cd) * U * U);
        cd* Hc = malloc(sizeof(cd) * S * U);
        cd* yc = malloc(sizeof(cd) * S);
        cd* b = malloc(sizeof(cd) * U);
        cd* bc = malloc(sizeof(cd) * U);
        cd* x = malloc(sizeof(cd) * U);
        for (int i = 0; i < U * U; ++i) G[i] = 0;
        for (int c = 0; c < C; ++c) {
            for (int i = 0; i < S * U; ++i) Hc[i] = ldf(H, ((size_t)c * N + n) * S * U + i);
            gram_cols(S, U, Hc, 0.0, Gc);
            for (int i = 0; i < U * U; ++i) G[i] += Gc[i];
        }
        for (int u = 0; u < U; ++u) G[u * U + u] += N0 / Es;
        int st = hpd_inverse(U, G, Gi);
        for (int j = 0; j < J && st == 0; ++j) {
            for (int u = 0; u < U; ++u) b[u] = 0;
            for (int c = 0; c < C; ++c) {
                for (int i = 0; i < S * U; ++i) Hc[i] = ldf(H, ((size_t)c * N + n) * S * U + i);
                for (int k = 0; k < S; ++k) yc[k] = ldf(y, (((size_t)c * N + n) * J + j) * S + k);
                matvec_h(S, U, Hc, yc, bc);
                for (int u = 0; u < U; ++u) b[u] += bc[u];
            }
            matvec(U, U, Gi, b, x);
            for (int u = 0; u < U; ++u) std_(x_hat, ((size_t)n * J + j) * U + u, x[u]);
            if (hard) {
                float f[64];
                for (int u = 0; u < U; ++u) { f[2 * u] = (float)creal(x[u]); f[2 * u + 1] = (float)cimag(x[u]); }
                dbpo_slice(mod, U, f, hard + ((size_t)n * J + j) * U);
            }
        }
        if (st) {
#pragma omp critical
            status = st;
        }
        free(G); free(Gc); free(Gi); free(Hc); free(yc); free(b); free(bc); free(x);
    }
    return status;
}

/* ZF-DL (P431; SPEC zf_centralized S300-308): for the full downlink matrix
 * H = [H_1^d, ..., H_C^d] (U x B), x = H^H (H H^H)^{-1} s, i.e. r = (sum_c
 * H_c H_c^H)^{-1} s and x_c = H_c^H r per cluster.  x: [C][N][Nsym][S]. */
int dbpo_zf_centralized(const dbpo_dims* d, const float* Hd, const float* s, double* x) {
    if (!dims_ok(d) || !Hd || !s || !x || d->U > 32) return 1;
    const int C = d->C, S = d->S, U = d->U, N = d->N, J = d->N_sym;
    int status = 0;
#pragma omp parallel for schedule(dynamic)
    for (int n = 0; n < N; ++n) {
        cd* B = malloc(sizeof(cd) * U * U);
        cd* Bc = malloc(sizeof(cd) * U * U);
        cd* Bi = malloc(sizeof(cd) * U * U);
        cd* Hn = malloc(sizeof(cd) * C * U * S);
        cd* sv = malloc(sizeof(cd) * U);
        cd* r = malloc(sizeof(cd) * U);
        cd* xc = malloc(sizeof(cd) * S);
        for (int i = 0; i < U * U; ++i) B[i] = 0;
        for (int c = 0; c < C; ++c) {
            for (int i = 0; i < U * S; ++i) Hn[(size_t)c * U * S + i] = ldf(Hd, ((size_t)c * N + n) * U * S + i);
            gram_rows(U, S, Hn + (size_t)c * U * S, 0.0, Bc);
            for (int i = 0; i < U * U; ++i) B[i] += Bc[i];
        }
        int st = hpd_inverse(U, B, Bi);
        for (int j = 0; j < J && st == 0; ++j) {
            for (int u = 0; u < U; ++u) sv[u] = ldf(s, ((size_t)n * J + j) * U + u);
            matvec(U, U, Bi, sv, r);
            for (int c = 0; c < C; ++c) {
                matvec_h(U, S, Hn + (size_t)c * U * S, r, xc);
                for (int k = 0; k < S; ++k) std_(x, (((size_t)c * N + n) * J + j) * S + k, xc[k]);
            }
        }
        if (st) {
#pragma omp critical
            status = st;
        }
        free(B); free(Bc); free(Bi); free(Hn); free(sv); free(r); free(xc);
    }
    return status;
}
