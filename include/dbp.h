/*
 * dbp.h -- C ABI of libdbp, the B200-native (sm_100a) hot path of
 * "Decentralized Baseband Processing for Massive MU-MIMO Systems"
 * (K. Li, R. Sharan, Y. Chen, T. Goldstein, J. R. Cavallaro, C. Studer,
 * arXiv 1702.04458).  Citations "P<n>" are lines of PAPER.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  * Complex numbers are dbp_cf32 = {float re, im} (== torch.complex64 ==
 *    cuFloatComplex), stored row-major, interleaved.
 *  * Clusters are partitioned row-wise over ranks (P149-155): rank r of
 *    `world` owns clusters [r*C/world, (r+1)*C/world); C % world == 0.
 *    Every per-cluster array below holds only the caller rank's C_loc =
 *    C/world clusters; per-subcarrier consensus arrays are full and
 *    replicated on every rank.
 *  * Pointers may be DEVICE pointers (the normal case; torch owns them) or
 *    HOST pointers (pageable or pinned).  Host buffers are staged through a
 *    library-owned device buffer with cudaMemcpyAsync on `stream`, so the
 *    host->device and device->host copies are part of the call (used by the
 *    end-to-end measurement).  All pointers of one call must be of the same
 *    kind.  Alignment: 16 bytes for complex arrays.
 *  * `ws` is a caller-owned device workspace of at least
 *    dbp_workspace_bytes() bytes (NULL allowed when that size is 0).
 *  * All compute is enqueued asynchronously on `stream` (a cudaStream_t;
 *    NULL = legacy default stream).  Host-pointer calls synchronise `stream`
 *    before returning.
 *  * Ownership: the caller owns every buffer and the workspace; the library
 *    owns only the context, its NCCL communicator, the device error flag,
 *    host-I/O staging buffers and cached launch state.
 *  * Errors: invalid arguments are detected synchronously BEFORE any launch
 *    and return DBP_ERR_INVALID_ARG with nothing enqueued; shapes outside the
 *    supported envelope return DBP_ERR_UNSUPPORTED.  A non-positive or
 *    non-finite Cholesky pivot found on the device (SPEC S44) sets a device
 *    flag; dbp_sync() then returns DBP_ERR_NOT_HPD and the outputs of the
 *    calls since the last dbp_sync() are undefined.  dbp_last_error() gives a
 *    thread-local message for the last non-OK status.
 *  * Supported envelope (v1): 1 <= U <= 32 (users are zero-padded to the
 *    next of 4/8/16/32 internally, which is exact), 1 <= S <= 64, N_sym <= 16.
 *  * Empty frames: N = 0 (no subcarriers) is valid.  After the scalar
 *    arguments are validated the solvers return DBP_OK with nothing
 *    enqueued and no consensus round (N is the same on every rank, so all
 *    ranks skip together); data pointers may then be NULL.
 *  * Threading: a context is not thread-safe; use one per rank and thread.
 */
#ifndef DBP_H
#define DBP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { float re, im; } dbp_cf32;

typedef enum {
    DBP_OK = 0,
    DBP_ERR_INVALID_ARG = 1,
    DBP_ERR_UNSUPPORTED = 2,
    DBP_ERR_NOT_HPD = 3,
    DBP_ERR_CUDA = 4,
    DBP_ERR_NCCL = 5,
    DBP_ERR_WORKSPACE = 6
} dbp_status;

/* Regulariser g(s) of the equalisation problem (E0) (P205-218) and its
 * proximal step (E2-*) (P335-344).  BOX with DBP_BPSK is the real-line
 * projection of P344. */
typedef enum { DBP_REG_MMSE = 0, DBP_REG_ZF = 1, DBP_REG_BOX = 2 } dbp_reg;

/* Gray-mapped constellation O (P143), Es = 1; value = bits per symbol. */
typedef enum { DBP_BPSK = 1, DBP_QPSK = 2, DBP_QAM16 = 4, DBP_QAM64 = 6 } dbp_mod;

typedef enum { DBP_ALGO_ADMM_UL = 0, DBP_ALGO_CG_UL = 1, DBP_ALGO_ADMM_DL = 2, DBP_ALGO_MMSE_UL = 3,
               DBP_ALGO_ZF_DL = 4 } dbp_algo;

/* C = total clusters (all ranks), S = B_c antennas per cluster (P150),
 * U users, N subcarriers (N >= 0), N_sym symbols sharing one channel
 * (P706-709).  B = C*S. */
typedef struct { int32_t C, S, U, N, N_sym; } dbp_dims;

typedef struct dbp_ctx dbp_ctx;

/* Counters since dbp_ctx_create (host-side bookkeeping). */
typedef struct {
    int64_t allreduce_calls;   /* NCCL collectives issued (0 at world == 1)            */
    int64_t allreduce_bytes;   /* NCCL payload bytes per rank, sum over calls (P625)  */
    int64_t kernel_launches;   /* libdbp kernels enqueued                              */
    int64_t consensus_rounds;  /* algorithmic consensus rounds: ADMM-UL T, CG T+1,
                                  ADMM-DL T-1 per call (SPEC S389-390), any world     */
    int64_t graph_replays;     /* schedules replayed from a cached CUDA graph (DBP_OPT_GRAPHS) */
} dbp_stats;

/* Options for dbp_set_option(). */
typedef enum {
    /* 0 (default): at world == 1 use the fused single-GPU kernels; 1: always
     * use the per-iteration (multi-kernel + collective) path, as at world > 1. */
    DBP_OPT_FORCE_SPLIT = 1,
    /* 1: bracket every libdbp kernel launch with CUDA events on its stream and
     * accumulate per-kernel device time (read with dbp_get_kernel_times). */
    DBP_OPT_KERNEL_TIMING = 2,
    /* 0 (default): at world == 1, when UP <= 16, N_sym == 1, C <= 128/UP*4 and
     * U, S are even, each solver is ONE per-subcarrier kernel (local Gram,
     * inverse, every consensus round and the output on chip); 1: use the
     * preprocessing + iteration kernels instead (same results up to rounding). */
    DBP_OPT_NO_FUSED = 3,
    /* Device-side consensus (NEXT-1; ADMM-UL, CG-UL, ADMM-DL).  0 (default): world > 1 uses the split
     * path, one ncclAllReduce per round.  1: at world > 1 each rank runs the fused per-subcarrier
     * kernel on its own clusters and the rounds' partial sums cross GPUs inside that kernel, by
     * peer stores of round-tagged words into a symmetric buffer (CUDA IPC over NVLink, LL
     * protocol); no collective per round.  Needs peer access between all ranks' GPUs (creating the
     * buffer is collective: every rank must make the same call).  2: as 1, and also at world == 1
     * against the rank's own buffer (a self-peer exercise of the device protocol for testing).
     * Safety: the kernel is launched cooperatively on a persistent grid (all CTAs co-resident, or
     * the launch fails); when this mode selects the fused kernel, a rank-local failure (unaligned
     * H / y, launch error) returns an error instead of falling back to the NCCL path; every wait on
     * a peer's round is bounded (DBP_XC_TIMEOUT_NS, 4 s), after which dbp_sync returns
     * DBP_ERR_CUDA ("device consensus timed out") and the outputs are undefined -- a fault on one
     * rank never hangs the GPUs.  Shapes the fused kernel does not take (N_sym > 1, U > 16) use the
     * NCCL path on every rank (the decision depends only on the dims).  Round ids are consecutive
     * within and across calls (ADMM-UL T, CG-UL T + 1, ADMM-DL T - 1 rounds).
     * Unverified across GPUs (single-GPU environment). */
    DBP_OPT_DEVICE_CONSENSUS = 4,
    /* Per-cluster inverse of Alg. 1 / Alg. 3 (P275-280, P290, P482-488, P500).  0 (default): the
     * paper's choice made strict -- S < U uses the S x S form (A_c = H_c H_c^H + rho I_S uplink,
     * A_c = H_c^H H_c + rho^{-1} I_S downlink; three mat-vecs per round), S >= U the U x U form
     * (B_c; at S == U the two have equal size and U x U needs one mat-vec per round, Table I).
     * 1: always U x U.  2: always S x S (S <= 32).  The two forms give the same iterates up to
     * rounding (Woodbury).  The S x S form runs on one warp per cluster pair with one launch per
     * consensus round (and the NCCL allreduce in between at world > 1); it affects the workspace
     * size, so set it before dbp_workspace_bytes.  CG (Alg. 2) has a single form. */
    DBP_OPT_MODE = 5,
    /* 1 (default): the multi-launch schedules (per-pair preprocessing, the per-round kernels and
     * the NCCL allreduces between them -- the world > 1 path, or FORCE_SPLIT / NO_FUSED) are
     * captured into a CUDA graph on first use and replayed while the call's dims, scalars and
     * device pointers repeat (host-pointer calls and KERNEL_TIMING never use graphs).  0: plain
     * launches.  Results are identical either way. */
    DBP_OPT_GRAPHS = 6,
    /* 1 (default): the cluster-summed Gram sum_c H_c^H H_c and y^MRC = sum_c H_c^H y_c are formed on
     * the tensor cores (fp16 mma.sync on an exact power-of-two-scaled hi/lo split, FP32 accumulation;
     * error ~2^-22 relative to the Gram, within the 1e-4 parity bar):
     *   - dbp_detect_cg at world == 1, N_sym <= 8, 9 <= U <= 16, U and S even, S <= 64 (no FORCE_SPLIT /
     *     NO_FUSED / DEVICE_CONSENSUS): the whole solve in one kernel (k_cg_tc; k_cg_tcj for N_sym > 1, the
     *     J matched filters on the tensor cores too);
     *   - the split / two-kernel dbp_detect_cg path (world > 1, U up to 32) and the non-fused
     *     dbp_detect_mmse path, N_sym == 1, U even, S <= 64: the rank's G_loc and y^MRC_loc (k_cgg_tc).
     * 0: the FP32 kernels (k_fused; per-pair Grams + fixed-order sum).  The two agree to rounding,
     * not bitwise. */
    DBP_OPT_CG_TENSOR = 7,
    /* 0 (default): ordinary stream order.  1: the single-kernel solver paths (world == 1 fused
     * ADMM-UL / CG-UL / ADMM-DL) are launched with programmatic stream serialization: the solver's
     * CTAs may start while the kernel before it on the stream is finishing (its last wave), filling
     * the SMs that kernel's tail leaves idle.  The solver reads H / y / s WITHOUT waiting for that
     * kernel, so the caller must not have it produce them (e.g. ADMM-UL of one frame followed by
     * ADMM-DL of another); every global store waits for it (griddepcontrol.wait), so outputs stay in
     * stream order.  Ignored with device consensus, host pointers make it moot (the H2D copy sits in
     * between).  Our own fused kernels let the next kernel start once their last wave is running. */
    DBP_OPT_OVERLAP_PREV = 8
} dbp_option;

/* Per-kernel device time accumulated under DBP_OPT_KERNEL_TIMING. */
typedef struct {
    char name[40];
    int64_t launches;
    double total_ms;
} dbp_kernel_time;

/* NCCL bootstrap: fills 128 bytes (an ncclUniqueId) on rank 0; broadcast it to
 * the other ranks (e.g. over torch.distributed) before dbp_ctx_create. */
dbp_status dbp_get_unique_id(uint8_t id[128]);

/* Create a context bound to CUDA `device` for `rank` of `world`.  `id` is the
 * rank-0 unique id (ignored and may be NULL when world == 1).  Collective
 * over all ranks when world > 1 (ncclCommInitRank).  world > 1 with id == NULL
 * creates a context without an NCCL communicator whose consensus exchange is a
 * host hook (dbp_set_allreduce_hook, which must be set before any solver call). */
dbp_status dbp_ctx_create(dbp_ctx** ctx, int device, int rank, int world, const uint8_t* id);

/* Host-side consensus exchange for a context created without a communicator (world > 1,
 * id == NULL): instead of ncclAllReduce, each round's partial sums (n_floats fp32 values,
 * complex interleaved) are copied to a pinned host buffer, `fn(host_buf, n_floats, user)` must
 * replace them in place by their sum over all ranks (in the same rank order everywhere) and
 * return 0, and the result is copied back -- the same dataflow over any transport (e.g. gloo;
 * the test suite uses it to run two ranks of the real library on one GPU).  Slow by design;
 * never used by the NCCL path.  Graphs and device-side consensus are off for such a context.
 * A non-zero return from fn makes the solver call return DBP_ERR_NCCL. */
typedef int (*dbp_allreduce_fn)(float* host_buf, int64_t n_floats, void* user);
dbp_status dbp_set_allreduce_hook(dbp_ctx* ctx, dbp_allreduce_fn fn, void* user);
dbp_status dbp_ctx_destroy(dbp_ctx* ctx);
dbp_status dbp_set_option(dbp_ctx* ctx, int option, int64_t value);
dbp_status dbp_get_stats(const dbp_ctx* ctx, dbp_stats* out);

/* The context's communicator as NCCL sees it (ncclCommCount / ncclCommUserRank): the number of
 * ranks the consensus allreduce spans and this rank's position.  world == 1: 1 and 0 (no
 * communicator).  Errors: NULL arguments -> DBP_ERR_INVALID_ARG; NCCL failure -> DBP_ERR_NCCL. */
dbp_status dbp_get_comm_info(const dbp_ctx* ctx, int* nranks, int* rank);

/* Thread-local message describing the last non-OK status ("" if none). */
const char* dbp_last_error(void);

/* Device workspace needed by one call of `algo` with `dims` on this context
 * (depends on world and options).  Deterministic; 0 is a valid answer. */
dbp_status dbp_workspace_bytes(const dbp_ctx* ctx, const dbp_dims* dims, int algo, size_t* bytes);

/* Algorithm 1 (P282-318): decentralized ADMM uplink data detection.
 *   H      [C_loc][N][S][U]     uplink H_c (P151)                      (read)
 *   y      [C_loc][N][N_sym][S] receive vectors y_c (eq. (1), P152)    (read)
 *   rho > 0 ADMM penalty (P234); gamma > 0 step (P245, 1 = default);
 *   N0 >= 0 noise variance, Es > 0 symbol energy (MMSE regulariser, P212);
 *   reg    prox of step (E2) (P335-344); mod: constellation for BOX radius
 *          and for the hard decisions;
 *   T >= 1 iterations incl. the init t = 1 (Alg. 1 loop from t = 2; T
 *          consensus collectives per call);
 *   s_hat  [N][N_sym][U] soft output x_hat = s^(T) (P316), identical on
 *          every rank                                                   (write)
 *   hard   NULL or [N][N_sym][U] Gray bit labels of the nearest point,
 *          [I bits | Q bits], ties toward the negative level (P210)     (write)
 * The U x U form of step (E1), eq. (3) (P272), is used for every S (the S x S
 * form eq. (4) gives the same iterates; reading 7). */
dbp_status dbp_detect_admm(dbp_ctx* ctx, const dbp_dims* dims, const dbp_cf32* H,
                           const dbp_cf32* y, float rho, float gamma, float N0, float Es,
                           int reg, int mod, int32_t T, dbp_cf32* s_hat, uint8_t* hard,
                           void* ws, size_t ws_bytes, void* stream);

/* Algorithm 2 (P383-413): decentralized conjugate-gradient uplink detection.
 *   rho >= 0: N0/Es for MMSE, 0 for ZF (P376);  T >= 1 CG iterations
 *   (T + 1 consensus collectives: y^MRC and one per iteration);
 *   x_hat  [N][N_sym][U] soft output (P411), replicated;  hard as above.
 * Line 11 is read with e^(t) (reading 1); alpha uses Re(p^H e)
 * (reading 3); ||r||^2 == 0 freezes the iterate (reading 4). */
dbp_status dbp_detect_cg(dbp_ctx* ctx, const dbp_dims* dims, const dbp_cf32* H,
                         const dbp_cf32* y, float rho, int mod, int32_t T, dbp_cf32* x_hat,
                         uint8_t* hard, void* ws, size_t ws_bytes, void* stream);

/* Algorithm 3 (P491-527): decentralized ADMM downlink beamforming.
 *   eps >= 0: the constraint ||H x - s|| <= eps of (P0); eps = 0 is Alg. 3 as
 *   printed, eps > 0 applies Lemma 2 (P538) at line 14:
 *   z_c = w_c + max{0, 1 - eps/||s - w||} (s - w)/C (reading 8).
 *   Hd  [C_loc][N][U][S]     downlink H_c^d = (H_c^u)^T (P174, P181)   (read)
 *   s   [N][N_sym][U]        transmit symbols s^d, replicated (P172)   (read)
 *   rho > 0, gamma > 0 (P457);  T >= 1 (T - 1 consensus collectives: the
 *   first iteration is local, P811);
 *   x   [C_loc][N][N_sym][S] local beamforming vectors x_c^(T) (P525)  (write) */
dbp_status dbp_beamform_admm(dbp_ctx* ctx, const dbp_dims* dims, const dbp_cf32* Hd,
                             const dbp_cf32* s, float rho, float gamma, float eps, int32_t T,
                             dbp_cf32* x, void* ws, size_t ws_bytes, void* stream);

/* Centralized baselines (NEXT-3; Table I rows MMSE-UL / ZF-DL, P594-595,
 * the comparison of P622 / P789-792): the whole array H = [H_1; ...; H_C]
 * solved exactly per subcarrier.  Each rank forms its clusters' Gram and
 * matched-filter sums; world > 1 adds ONE allreduce of [sum_c G_c | sum_c
 * H_c^H y_c] (N (U(U+1)/2 + N_sym U) complex values; it is not a consensus
 * round), then every rank solves the U x U system (DBP_ERR_NOT_HPD on a
 * rank-deficient Gram).
 *
 * dbp_detect_mmse: x_hat = (H^H H + (N0/Es) I)^{-1} H^H y (P212-218);
 *   N0 = 0 gives ZF detection.  H, y, x_hat, hard as in dbp_detect_admm.
 * dbp_precode_zf:  x = H^H (H H^H)^{-1} s for H = [H_1^d, ..., H_C^d]
 *   (P431), i.e. x_c = H_c^H r with r = (sum_c H_c H_c^H)^{-1} s.
 *   Hd, s, x as in dbp_beamform_admm.
 * Workspace: dbp_workspace_bytes with DBP_ALGO_MMSE_UL / DBP_ALGO_ZF_DL. */
dbp_status dbp_detect_mmse(dbp_ctx* ctx, const dbp_dims* dims, const dbp_cf32* H, const dbp_cf32* y,
                           float N0, float Es, int mod, dbp_cf32* x_hat, uint8_t* hard, void* ws,
                           size_t ws_bytes, void* stream);
dbp_status dbp_precode_zf(dbp_ctx* ctx, const dbp_dims* dims, const dbp_cf32* Hd, const dbp_cf32* s,
                          dbp_cf32* x, void* ws, size_t ws_bytes, void* stream);

/* Hard slicer alone (P210): bits[i] = Gray label of the nearest point of `mod`
 * to x[i] (decided in fp32, same rule as the detectors' `hard`).  Device or
 * host pointers as above. */
dbp_status dbp_slice(dbp_ctx* ctx, int mod, int64_t count, const dbp_cf32* x, uint8_t* bits,
                     void* stream);

/* Resolve the recorded events (blocks until they complete) and return up to
 * `max_entries` per-kernel totals; `reset` != 0 clears the totals. */
dbp_status dbp_get_kernel_times(dbp_ctx* ctx, dbp_kernel_time* out, int max_entries, int* n_entries,
                                int reset);

/* ---- Table I (P566-595): real-multiplication counts of the decentralized and
 * centralized algorithms, the paper's complexity model (P616-622).  Host-only
 * arithmetic, no context or GPU needed.
 *   algo    DBP_CPLX_ADMM_DL, _ADMM_UL, _CG_UL (decentralized, with `mode`
 *           and `metric`), _ZF_DL, _MMSE_UL (centralized: mode and metric are
 *           ignored, the whole count is returned as `total` and `pre`)
 *   mode    DBP_CPLX_SxS or DBP_CPLX_UxU (ignored for CG-UL)
 *   metric  DBP_CPLX_TM (timing: one cluster's PE) or DBP_CPLX_AR (all PEs)
 *   out     [0] preprocessing, [1] first iteration, [2] each subsequent
 *           iteration, [3] total(T) = [0] + [1] + (T - 1) [2]
 * Every Table I expression is integral for integer U, S, C (the 1/3 terms
 * combine to multiples of 3), so the counts are exact.  Errors: U, S, C, T < 1
 * or an unknown algo / mode / metric -> DBP_ERR_INVALID_ARG. */
typedef enum { DBP_CPLX_ADMM_DL = 0, DBP_CPLX_ADMM_UL = 1, DBP_CPLX_CG_UL = 2, DBP_CPLX_ZF_DL = 3,
               DBP_CPLX_MMSE_UL = 4 } dbp_cplx_algo;
typedef enum { DBP_CPLX_SxS = 0, DBP_CPLX_UxU = 1 } dbp_cplx_mode;
typedef enum { DBP_CPLX_TM = 0, DBP_CPLX_AR = 1 } dbp_cplx_metric;
dbp_status dbp_complexity(int algo, int mode, int metric, int64_t U, int64_t S, int64_t C, int64_t T,
                          int64_t out[4]);

/* Synchronise `stream`; returns DBP_ERR_NOT_HPD if a Cholesky pivot failed in
 * any call since the previous dbp_sync (and clears the flag), DBP_ERR_CUDA if a
 * device-consensus wait timed out (DBP_OPT_DEVICE_CONSENSUS), or
 * DBP_ERR_CUDA / DBP_ERR_NCCL for deferred runtime errors. */
dbp_status dbp_sync(dbp_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DBP_H */
