/*
 * dbp_oracle.h -- plain double-precision CPU oracle for the decentralized
 * baseband processing hot path of Li et al., arXiv 1702.04458.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path under
 * paper_1702_04458_b200/csrc/.
 *
 * Citations: "P<n>" = /root/reference/PAPER.md line n (section / equation /
 * algorithm named beside it).  Readings of ambiguous passages follow
 * SURVEY.md section 8(c) and are listed in DESIGN.md section 3.
 *
 * Layouts (row-major, complex values interleaved re,im):
 *   H   [C][N][S][U]      uplink H_c^u          (float32 inputs, promoted to double)
 *   y   [C][N][Nsym][S]   uplink y_c^u
 *   Hd  [C][N][U][S]      downlink H_c^d = (H_c^u)^T (P174, P181)
 *   s   [N][Nsym][U]      downlink transmit vector s^d
 *   outputs are double complex interleaved.
 *
 * Return codes: 0 ok, 1 invalid argument, 3 not HPD (Cholesky pivot <= 0 or
 * non-finite).
 */
#ifndef DBP_ORACLE_H
#define DBP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { int32_t C, S, U, N, N_sym; } dbpo_dims;

enum { DBPO_REG_MMSE = 0, DBPO_REG_ZF = 1, DBPO_REG_BOX = 2 };       /* P212-218, P335-344 */
enum { DBPO_BPSK = 1, DBPO_QPSK = 2, DBPO_QAM16 = 4, DBPO_QAM64 = 6 }; /* value = bits/symbol */
enum { DBPO_MODE_PAPER = -1, DBPO_MODE_UU = 0, DBPO_MODE_SS = 1 };      /* P290, P500 */

/* Hermitian positive-definite inverse by Cholesky + forward/backward
 * substitution (P704; SPEC hpd_inverse).  G, Ginv: n x n double complex. */
int dbpo_hpd_inverse(int n, const double* G, double* Ginv);

/* Hard slicer: nearest constellation point per axis (P210), ties toward the
 * more negative level, Gray bits [I | Q] (readings 17-19).  Decided in fp32. */
int dbpo_slice(int mod, int64_t count, const float* x, uint8_t* bits);

/* Algorithm 1 (P282-318): decentralized ADMM uplink detection. */
int dbpo_detect_admm(const dbpo_dims* d, const float* H, const float* y,
                     double rho, double gamma, double N0, double Es, int reg,
                     int mod, int T, int mode, double* s_hat, uint8_t* hard);

/* Same, recording the iterates of subcarrier n_tr, symbol j_tr:
 * s_tr [T][U], z_tr [T][C][U], lam_tr [T][C][U]  (index t-1 for t = 1..T). */
int dbpo_detect_admm_trace(const dbpo_dims* d, const float* H, const float* y,
                           double rho, double gamma, double N0, double Es,
                           int reg, int mod, int T, int mode, int n_tr, int j_tr,
                           double* s_tr, double* z_tr, double* lam_tr);

/* Algorithm 2 (P383-413): decentralized CG uplink detection. */
int dbpo_detect_cg(const dbpo_dims* d, const float* H, const float* y,
                   double rho, int mod, int T, double* x_hat, uint8_t* hard);

/* x_tr, r_tr, p_tr: [T+1][U] for t = 0..T (iterations stopped early by the
 * r = 0 rule repeat the frozen state). */
int dbpo_detect_cg_trace(const dbpo_dims* d, const float* H, const float* y,
                         double rho, int T, int n_tr, int j_tr,
                         double* x_tr, double* r_tr, double* p_tr);

/* Algorithm 3 (P491-527): decentralized ADMM downlink beamforming.
 * x: [C][N][Nsym][S].  eps >= 0 applies Lemma 2 (P535-547). */
int dbpo_beamform_admm(const dbpo_dims* d, const float* Hd, const float* s,
                       double rho, double gamma, double eps, int T, int mode,
                       double* x);

/* x_tr [T][C][S], z_tr [T][C][U], lam_tr [T][C][U], w_tr [T][C][U]
 * (w_tr[t-1] = w_c^(t-1) of Alg. 3 line 12, zero for t = 1). */
int dbpo_beamform_admm_trace(const dbpo_dims* d, const float* Hd, const float* s,
                             double rho, double gamma, double eps, int T, int mode,
                             int n_tr, int j_tr, double* x_tr, double* z_tr,
                             double* lam_tr, double* w_tr);

/* Centralized baselines (Table I rows ZF-DL / MMSE-UL, P594-595):
 * MMSE-UL x = (H^H H + (N0/Es) I)^{-1} H^H y over all C clusters (N0 = 0: ZF),
 * x_hat [N][Nsym][U];  ZF-DL x_c = H_c^H (sum_c H_c H_c^H)^{-1} s,
 * x [C][N][Nsym][S].  Status 3 if the Gram is not HPD (rank deficiency). */
int dbpo_mmse_centralized(const dbpo_dims* d, const float* H, const float* y, double N0, double Es,
                          int mod, double* x_hat, uint8_t* hard);
int dbpo_zf_centralized(const dbpo_dims* d, const float* Hd, const float* s, double* x);

#ifdef __cplusplus
}
#endif
#endif
