// dbp_iter.cu -- consensus iterations of ADMM-UL (Alg. 1) and ADMM-DL
// (Alg. 3) on a per-pair inverse computed by the preprocessing kernel
// (k_prefold, or k_prelr for UP = 32), SURVEY 8(a) rows a4-a8 and c2-c4.
// Used by the two-kernel path (world == 1 outside k_fused's shapes, or
// DBP_OPT_NO_FUSED) and by the split path (world > 1, DBP_OPT_FORCE_SPLIT).
//
// Layout: one lane per row of the U x U operator ("lane = user"), UP lanes per
// (cluster, subcarrier) pair, all lanes of a pair inside one warp.
//  * Iterations: every local update is one row of a Hermitian mat-vec with
//    the vector broadcast through shared memory; the consensus sum over the
//    CTA's clusters is taken in fixed cluster order (deterministic).
//  * k_admm_gj / k_bf_gj (world == 1): all T iterations + outputs in one
//    launch, the rows of B^{-1} stay in registers.  k_admm_it / k_bf_it (any
//    world): one round per launch, leaving the partial consensus sum for the
//    NCCL allreduce.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_internal.h"
#include "dbp_lanerow.cuh"

// tuning knob (build.py -D...): bf_output keeps r in registers up to this UP, else it
// reads r_u by broadcast LDS per use (UP = 16: the split output pass 112 -> 99 us, and
// k_bf_gj fits 64 registers without spills)
#ifndef DBP_BFOUT_REG_MAX_UP
#define DBP_BFOUT_REG_MAX_UP 8
#endif
namespace dbp {

// The fused iteration kernels' B^{-1} rows (k_admm_gj / k_bf_gj).  At UP = 32 a warp is one pair: its packed
// triangle is staged through shared memory with coalesced 16-B cp.async (lane-row loads straight from HBM
// touch 32 sectors per warp instruction, see warp_tri_copy); below that the rows come straight from HBM.
#ifndef DBP_GJ_STAGED_MIN
#define DBP_GJ_STAGED_MIN 32
#endif
constexpr bool gj_staged(int UP) { return UP >= DBP_GJ_STAGED_MIN; }
template <int UP>
__device__ __forceinline__ void gj_load_rows(const float2* __restrict__ Gp, size_t pair, float2* stage, int q, int i,
                                             float2 (&R)[UP]) {
    if constexpr (gj_staged(UP)) {
        static_assert(UP == 32, "one pair per warp");
        float2* tb = stage + (size_t)q * tri(UP);
        const float2* src = Gp + pair * tri(UP);
        for (int e = i; e < tri(UP) / 2; e += 32) cp_async16(tb + 2 * e, src + 2 * e);
        cp_async_commit();
        cp_async_wait_all();
        DBP_SYNCWARP();
        load_herm_row_s<UP>(tb, i, R);
    } else {
        load_herm_row<UP>(Gp + pair * tri(UP), i, R);
    }
}


// ============================================================ ADMM-UL


// Fused (world == 1): G^{-1} in registers, all T iterations of Alg. 1 on chip.
// CTA = NT subcarriers x C clusters x UP lanes.
template <int UP>
__global__ void __launch_bounds__(512, UP <= 16 ? 2 : 1) k_admm_gj(UlArgs a) {   // 2 CTAs/SM at <= 64 registers (no spills)
    extern __shared__ __align__(16) float2 sm[];
    DBP_POISON_SMEM(sm);
    const int C = a.C_loc, NT = a.NT;
    float2* pbuf = sm;                                  // [NT*C][UP] per-pair line
    float2* W = pbuf + (size_t)NT * C * UP;             // [NT][C][UP]
    float2* Sv = W + (size_t)NT * C * UP;               // [NT][UP]
    const int tid = threadIdx.x;
    const int q = tid / UP, i = tid % UP;
    const int nl = q / C, c = q % C;
    const int n0 = blockIdx.x * NT;
    const int n = n0 + nl;
    const bool valid = n < a.N;
    const size_t pair = (size_t)c * a.N + (valid ? n : a.N - 1);
    float2* buf = pbuf + (size_t)q * UP;

    float2 R[UP];
    gj_load_rows<UP>(a.Ginv, pair, sm + (size_t)2 * NT * C * UP + (size_t)NT * UP, q, i, R);   // row i of B_c^{-1}
#pragma unroll
    for (int j = 0; j < UP; ++j) R[j] = c_scale(R[j], a.rho);   // rho B_c^{-1} (eq. (3))

    for (int jj = 0; jj < a.J; ++jj) {
        const float2 yreg = a.yreg[(pair * a.J + jj) * UP + i];  // B^{-1} H^H y (Alg. 1 line 8)
        float2 lam = make_float2(0.f, 0.f), z = yreg, w = yreg;   // line 10
        for (int t = 1; t <= a.T; ++t) {
            if (t > 1) {
                const float2 s = Sv[nl * UP + i];
                lam = c_add(lam, c_scale(c_sub(z, s), a.gamma));     // line 12
                const float2 v = c_sub(s, lam);
                z = c_add(yreg, row_apply<UP>(R, buf, i, v));       // line 15, eq. (3)
                w = c_add(z, lam);                                   // line 17
            }
            W[((size_t)nl * C + c) * UP + i] = valid ? w : make_float2(0.f, 0.f);
            DBP_SYNCTHREADS();
            if (tid < NT * UP) {                                     // line 18 (consensus) + 19 (prox)
                const int el = tid / UP, uu = tid % UP;
                Sv[el * UP + uu] = prox(cluster_sum(W, C, UP, el, uu), a.px);
            }
            DBP_SYNCTHREADS();
        }
        if (tid < NT * UP) {
            const int el = tid / UP, uu = tid % UP;
            const int nn = n0 + el;
            if (nn < a.N && uu < a.U) {
                const float2 s = Sv[el * UP + uu];
                a.s_hat[((size_t)nn * a.J + jj) * a.U + uu] = s;
                if (a.hard) a.hard[((size_t)nn * a.J + jj) * a.U + uu] = slice_bits(s, a.md);
            }
        }
        DBP_SYNCTHREADS();
    }
}

// Per-warp staging of the packed triangles for the split kernels.  A warp
// holds the 32/UP consecutive pair slots q0.. of one subcarrier row; it copies
// their chunk-c0 triangles into its own shared buffer with coalesced 16-B
// cp.async (tri(UP) * 8 B is a multiple of 16 for every UP), so lane-row reads
// come from shared memory: read straight from HBM, lane i's row (a contiguous
// piece plus a strided column) makes every warp load touch 32 sectors, and the
// L1 wavefront rate, not HBM, set the time.  Double-buffered per warp: chunk
// k+1's copies are in flight while chunk k computes; no CTA barrier.  Used at
// UP = 32 (E: 705 vs 942 us per ADMM-UL round); at UP <= 16 half-warp rows
// gather fewer sectors and the direct loads measured faster (C split: 22.6 vs
// 25.3 us), so there the rows come straight from HBM.
constexpr int split_staged(int UP) { return UP >= 32; }
// staging depth (chunks per warp in flight + the one being read): a CTA walks only C_loc / CCH chunks
// (4 at the E share), so a 2-deep ring leaves the first chunk's load latency exposed per CTA
#ifndef DBP_SPLIT_NBUF
#define DBP_SPLIT_NBUF 2
#endif
constexpr int SPLIT_NBUF = DBP_SPLIT_NBUF;
__device__ __forceinline__ void cp_async_wait_nbuf() {
    asm volatile("cp.async.wait_group %0;" ::"n"(SPLIT_NBUF - 1) : "memory");
}
template <int UP>
__device__ __forceinline__ void warp_tri_copy(float2* dst, const float2* __restrict__ Gp, int C, int N, int c0,
                                              int n0, int q0, int CCH, int lane) {
    constexpr int TV = tri(UP) / 2, PWQ = 32 / UP;
    // the last warp may be partial when UP < 32 (UP = 32: every warp is one full pair)
    const int nlanes = UP == 32 ? 32 : min(32, (int)blockDim.x - (int)(threadIdx.x & ~31u));
    for (int e = lane; e < PWQ * TV; e += nlanes) {
        const int pj = e / TV, k = e - pj * TV;
        const int qq = q0 + pj, nl = qq / CCH, c = c0 + qq % CCH, n = n0 + nl;
        if (c < C && n < N) cp_async16(dst + pj * tri(UP) + 2 * k, Gp + ((size_t)c * N + n) * tri(UP) + 2 * k);
    }
    cp_async_commit();
}

// Chunks 0 .. NBUF-2 of the warp's triangles into buffers 0 .. NBUF-2 (one commit group each, empty
// past the last chunk, so the group count stays uniform).
template <int UP>
__device__ __forceinline__ void warp_tri_prologue(float2* tb, const float2* __restrict__ Gp, int C, int N, int n0,
                                                  int q0, int CCH, int lane) {
    constexpr int WB = 32 / UP * tri(UP);
#pragma unroll
    for (int j = 0; j < SPLIT_NBUF - 1; ++j) {
        if (j * CCH < C) warp_tri_copy<UP>(tb + j * WB, Gp, C, N, j * CCH, n0, q0, CCH, lane);
        else cp_async_commit();
    }
}

// Row i of this lane's pair for chunk c0 (buffers tb[NBUF] of 32/UP triangles each): chunk k + NBUF - 1
// is issued into the buffer chunk k - 1 was read from, then chunk k's group is waited for.
template <int UP>
__device__ __forceinline__ void warp_tri_row(float2* tb, const float2* __restrict__ Gp, int C, int N, int c0, int n0,
                                             int q0, int CCH, int lane, int qi, int i, float2 (&R)[UP]) {
    constexpr int WB = 32 / UP * tri(UP);
    const int k = c0 / CCH;
    DBP_SYNCWARP();                                        // the buffer about to be refilled was read a chunk ago
    const int kn = k + SPLIT_NBUF - 1;
    if (kn * CCH < C) warp_tri_copy<UP>(tb + (kn % SPLIT_NBUF) * WB, Gp, C, N, kn * CCH, n0, q0, CCH, lane);
    else cp_async_commit();
    cp_async_wait_nbuf();                                  // chunk k's group is complete
    DBP_SYNCWARP();
    load_herm_row_s<UP>(tb + (k % SPLIT_NBUF) * WB + qi * tri(UP), i, R);
}

// Split path: one iteration (or the init t = 1) for all local clusters of NT
// subcarriers, clusters visited in chunks of CCH (any C_loc); writes the
// local partial consensus sum into wbuf.  No barrier inside the chunk loop:
// every (subcarrier, cluster-slot) pair accumulates its clusters' w_c in its
// own shared-memory slot (chunk order), and one fixed-order sum over the slots
// at the end forms the partial sum (deterministic).  Each warp therefore
// streams its pairs' G^{-1} rows independently, and the load latency of one
// chunk is hidden by the other warps instead of serialising the CTA.
// INIT: the instantiation launched for the init round (t = 1, no B^{-1}); INIT = false, rounds 2..T
// (compile-time: the round kernel carries no init branches)
template <int UP, bool INIT>
__global__ void __launch_bounds__(256) k_admm_it(UlArgs a, int CCH) {   // split_cfg: <= 256 threads
    constexpr bool init = INIT;                            // a.init (measured: E share 73.3 -> 69.7 us per launch)
    extern __shared__ __align__(16) float2 sm[];
    DBP_POISON_SMEM(sm);
    const int C = a.C_loc, NT = a.NT, J = a.J;
    float2* pbuf = sm;                                  // [NT*CCH][UP]
    float2* Wp = pbuf + (size_t)NT * CCH * UP;          // [NT][J][CCH][UP] per-slot partial sums
    float2* Sv = Wp + (size_t)NT * J * CCH * UP;        // [NT][J][UP]
    float2* Tb = Sv + (size_t)NT * J * UP;              // [warps][NBUF][32/UP][tri(UP)] staged G^{-1}
    const int tid = threadIdx.x;
    const int q = tid / UP, i = tid % UP;
    const int nl = q / CCH, cl = q % CCH;
    const int n0 = blockIdx.x * NT;
    const int n = n0 + nl;
    const int nn = n < a.N ? n : a.N - 1;
    float2* buf = pbuf + (size_t)q * UP;
    const int lane = tid & 31, q0 = (tid >> 5) * (32 / UP);
    float2* tb = Tb + (size_t)(tid >> 5) * SPLIT_NBUF * (32 / UP) * tri(UP);
    if (split_staged(UP) && !init) warp_tri_prologue<UP>(tb, a.Ginv, C, a.N, n0, q0, CCH, lane);
    for (int e = tid; e < NT * J * UP; e += blockDim.x) {
        const int el = e / (J * UP);
        const bool ok = n0 + el < a.N && !init;
        Sv[e] = prox(ok ? a.wbuf[(size_t)n0 * J * UP + e] : make_float2(0.f, 0.f), a.px);
    }
    float2* wp = Wp + ((size_t)nl * J * CCH + cl) * UP + i;   // this lane's slot, symbol stride CCH * UP
    for (int jj = 0; jj < J; ++jj) wp[(size_t)jj * CCH * UP] = make_float2(0.f, 0.f);
    DBP_SYNCTHREADS();
    for (int c0 = 0; c0 < C; c0 += CCH) {
        const int c = c0 + cl;
        const bool valid = n < a.N && c < C;
        const size_t pair = (size_t)(c < C ? c : C - 1) * a.N + nn;
        // symbol 0's y^reg and w_c are loaded before the wait for the staged rows (their latency overlaps it)
        const float2 yreg0 = a.yreg[pair * J * UP + i];
        const float2 w00 = (!init && a.wonly) ? a.z[pair * J * UP + i] : make_float2(0.f, 0.f);
        float2 R[UP];
        if (!init) {
            if (split_staged(UP)) warp_tri_row<UP>(tb, a.Ginv, C, a.N, c0, n0, q0, CCH, lane, q - q0, i, R);
            else load_herm_row<UP>(a.Ginv + pair * tri(UP), i, R);
#pragma unroll
            for (int j = 0; j < UP; ++j) R[j] = c_scale(R[j], a.rho);
        }
        for (int jj = 0; jj < J; ++jj) {
            const size_t o = (pair * J + jj) * UP + i;
            const float2 yreg = jj == 0 ? yreg0 : a.yreg[o];
            float2 lam, z, w;
            if (init) {                                                // line 10
                lam = make_float2(0.f, 0.f);
                z = yreg;
                w = yreg;
            } else if (a.wonly) {
                // gamma = 1: lambda' = w - s, so z' + lambda' = y^reg + rho B^{-1} (2 s - w) + w - s
                // (lines 12, 15, 17 with lambda and z eliminated): only w_c is carried between rounds
                const float2 s = Sv[((size_t)nl * J + jj) * UP + i];
                const float2 w0 = jj == 0 ? w00 : a.z[o];
                w = c_add(c_add(yreg, row_apply<UP>(R, buf, i, c_sub(c_scale(s, 2.f), w0))), c_sub(w0, s));
            } else {
                const float2 s = Sv[((size_t)nl * J + jj) * UP + i];
                lam = c_add(a.lam[o], c_scale(c_sub(a.z[o], s), a.gamma));   // line 12
                z = c_add(yreg, row_apply<UP>(R, buf, i, c_sub(s, lam)));    // line 15
                w = c_add(z, lam);                                           // line 17
            }
            if (valid) {
                if (a.wonly) {
                    a.z[o] = w;                                              // the z buffer holds w_c
                } else {
                    a.lam[o] = lam;
                    a.z[o] = z;
                }
                wp[(size_t)jj * CCH * UP] = c_add(wp[(size_t)jj * CCH * UP], w);
            }
        }
    }
    DBP_SYNCTHREADS();
    for (int e = tid; e < NT * J * UP; e += blockDim.x)      // e = (el J + jj) UP + u
        if (n0 + e / (J * UP) < a.N) a.wbuf[(size_t)n0 * J * UP + e] = cluster_sum(Wp, CCH, UP, e / UP, e % UP);
}

// ============================================================ ADMM-DL


// x_c = H_c^H r (r = B^{-1} q published in buf): lanes own antennas s = i, i+UP, ...
template <int UP>
__device__ __forceinline__ void bf_output(const float2* __restrict__ Hd, float2* buf, int i, float2 ri, int U, int S,
                                          float2* __restrict__ xo, bool valid) {
    buf[i] = ri;
    DBP_SYNCWARP();
    // UP = 32: r_u by broadcast LDS (a register copy of r next to the caller's row spills)
    constexpr bool RR = UP <= DBP_BFOUT_REG_MAX_UP;
    float2 r[RR ? UP : 1];
    if constexpr (RR) read_vec<UP>(buf, r);
    for (int s = i; s < S; s += UP) {
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < UP; ++u)
            if (u < U) c_fmac(acc, __ldg(Hd + (size_t)u * S + s), RR ? r[RR ? u : 0] : buf[u]);
        if (valid) xo[s] = acc;
    }
    DBP_SYNCWARP();
}

// Fused (world == 1): B^{-1} in registers; init, T-1 consensus iterations of
// Alg. 3 in the exact m-form (m_c = q - rho^{-1} B^{-1} q, q = z + lambda;
// DESIGN.md section 5) and the output pass x_c = H_c^H B^{-1} q.
// MINB = 2 (<= 64 registers, 2 CTAs/SM) pays when N_sym > 1 (N_sym = 7: 277 -> 243 us) but not at
// N_sym = 1 (89 vs 117 us): launch_bf_gj picks per call.
template <int UP, int MINB>
__global__ void __launch_bounds__(512, MINB) k_bf_gj(DlArgs a) {
    extern __shared__ __align__(16) float2 sm[];
    DBP_POISON_SMEM(sm);
    const int C = a.C_loc, NT = a.NT;
    float2* pbuf = sm;
    float2* W = pbuf + (size_t)NT * C * UP;
    float2* Ws = W + (size_t)NT * C * UP;
    const int tid = threadIdx.x;
    const int q = tid / UP, i = tid % UP;
    const int nl = q / C, c = q % C;
    const int n0 = blockIdx.x * NT;
    const int n = n0 + nl;
    const bool valid = n < a.N;
    const int nn = valid ? n : a.N - 1;
    const size_t pair = (size_t)c * a.N + nn;
    float2* buf = pbuf + (size_t)q * UP;

    // the output pass re-reads H_c: start pulling this pair's tile into L2 now
    if (i == 0) {
        const size_t bytes = (size_t)a.U * a.S * 8;
        if ((bytes & 15) == 0 && bytes < (1u << 20))
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.Hd + pair * (size_t)a.U * a.S),
                         "r"((uint32_t)bytes) : "memory");
    }
    float2 R[UP];
    gj_load_rows<UP>(a.Binv, pair, sm + (size_t)2 * NT * C * UP + (size_t)NT * UP, q, i, R);   // row i of B_c^{-1}

    for (int jj = 0; jj < a.J; ++jj) {
        const float2 sv = i < a.U ? a.s[((size_t)nn * a.J + jj) * a.U + i] : make_float2(0.f, 0.f);
        float2 lam = make_float2(0.f, 0.f);
        float2 qv = c_scale(sv, a.a0);                                   // line 8: z = a0 s
        for (int t = 2; t <= a.T; ++t) {
            const float2 bq = row_apply<UP>(R, buf, i, qv);
            const float2 m = c_sub(qv, c_scale(bq, a.rho_inv));          // line 11 (m-form)
            const float2 w = c_sub(m, lam);                              // line 12
            W[((size_t)nl * C + c) * UP + i] = valid ? w : make_float2(0.f, 0.f);
            DBP_SYNCTHREADS();
            if (tid < NT * UP) Ws[tid] = cluster_sum(W, C, UP, tid / UP, tid % UP);   // line 13
            DBP_SYNCTHREADS();
            const float2 d = c_sub(sv, Ws[nl * UP + i]);
            const float f = lemma2_scale(group_sum<UP>(c_norm2(d)), a.eps, a.inv_c);
            const float2 z = c_add(w, c_scale(d, f));                                // line 14 (Lemma 2)
            lam = c_sub(lam, c_scale(c_sub(m, z), a.gamma));                         // line 15
            qv = c_add(z, lam);
            // (no third barrier: the next round's W / Ws writes come after its first barrier, which
            // every thread reaches only once it has read this round's Ws)
        }
        const float2 r = row_apply<UP>(R, buf, i, qv);                  // B^{-1} q
        if (a.J == 1) {
            bf_output<UP>(a.Hd + pair * (size_t)a.U * a.S, buf, i, r, a.U, a.S,
                          a.x + (pair * a.J + jj) * a.S, valid);        // line 20 / output
        } else {
            if (valid) a.m[(pair * a.J + jj) * UP + i] = r;             // all symbols' r, then one H_c pass
                                                                        // (padding lanes alias pair N - 1)
        }
    }
    if (a.J > 1) {
        // x_c[j] = H_c^H r_j for every symbol j from ONE pass over H_c: lane i takes antennas
        // i, i+UP, ..., loads the antenna's column of H_c once and reuses it for all J symbols
        DBP_SYNCWARP();
        const float2* Hp = a.Hd + pair * (size_t)a.U * a.S;
        const float2* rp = a.m + pair * a.J * UP;
        for (int s = i; s < a.S; s += UP) {
            float2 h[UP];
#pragma unroll
            for (int u = 0; u < UP; ++u) h[u] = u < a.U ? __ldg(Hp + (size_t)u * a.S + s) : make_float2(0.f, 0.f);
            for (int jj = 0; jj < a.J; ++jj) {
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int u = 0; u < UP; ++u) c_fmac(acc, h[u], rp[jj * UP + u]);
                if (valid) a.x[(pair * a.J + jj) * a.S + s] = acc;
            }
        }
    }
}

// Split path step t (2..T): complete iteration t-1 (or the init when t == 2),
// then m, w_c and the local partial sum.  step == T+1: complete, write x_c.
// Clusters in chunks of CCH.
// FIN: the instantiation launched for the output pass (a.step > a.T); FIN = false, the rounds
template <int UP, bool FIN>
__global__ void __launch_bounds__(256, UP >= 32 ? 2 : 3) k_bf_it(DlArgs a, int CCH) {   // split_cfg: <= 256 threads
    extern __shared__ __align__(16) float2 sm[];
    DBP_POISON_SMEM(sm);
    const int C = a.C_loc, NT = a.NT, J = a.J;
    float2* pbuf = sm;                                  // [NT*CCH][UP]
    float2* Wp = pbuf + (size_t)NT * CCH * UP;          // [NT][J][CCH][UP] per-slot partial sums
    float2* Wv = Wp + (size_t)NT * J * CCH * UP;        // [NT][J][UP]  allreduced w^(t-1)
    float2* Tb = Wv + (size_t)NT * J * UP;              // [warps][NBUF][32/UP][tri(UP)] staged B^{-1}
    const int tid = threadIdx.x;
    const int q = tid / UP, i = tid % UP;
    const int nl = q / CCH, cl = q % CCH;
    const int n0 = blockIdx.x * NT;
    const int n = n0 + nl;
    const int nn = n < a.N ? n : a.N - 1;
    float2* buf = pbuf + (size_t)q * UP;
    const int lane = tid & 31, q0 = (tid >> 5) * (32 / UP);
    float2* tb = Tb + (size_t)(tid >> 5) * SPLIT_NBUF * (32 / UP) * tri(UP);
    if (split_staged(UP)) warp_tri_prologue<UP>(tb, a.Binv, C, a.N, n0, q0, CCH, lane);
    // the step kernels know they are not the output pass (compile time: measured faster, 24.5 -> 21.2 us at
    // config D); the output pass keeps the runtime test (its compile-time twin measured slower, 107.7 -> 119.7)
    const bool fin = FIN && a.step > a.T;
    const bool first = a.step == 2;
    // the output pass reads H_c of every pair: pull the pair's tile into L2 one
    // chunk ahead (all chunks up front overflows L2 at C_loc = 128: 8x slower)
    const size_t hbytes = (size_t)a.U * a.S * 8;
    const bool pf = fin && i == 0 && n < a.N && (hbytes & 15) == 0 && hbytes < (1u << 20);
    auto prefetch_h = [&](int c) {
        if (pf && c < C)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                         ::"l"(a.Hd + ((size_t)c * a.N + n) * a.U * a.S), "r"((uint32_t)hbytes) : "memory");
    };
    prefetch_h(cl);
    for (int e = tid; e < NT * J * UP; e += blockDim.x) {
        const int el = e / (J * UP);
        Wv[e] = (n0 + el < a.N && !first) ? a.wbuf[(size_t)n0 * J * UP + e] : make_float2(0.f, 0.f);
    }
    float2* wp = Wp + ((size_t)nl * J * CCH + cl) * UP + i;   // this lane's slot, symbol stride CCH * UP
    for (int jj = 0; jj < J; ++jj) wp[(size_t)jj * CCH * UP] = make_float2(0.f, 0.f);
    DBP_SYNCTHREADS();
    for (int c0 = 0; c0 < C; c0 += CCH) {
        const int c = c0 + cl;
        const bool valid = n < a.N && c < C;
        const size_t pair = (size_t)(c < C ? c : C - 1) * a.N + nn;
        float2 R[UP];
        prefetch_h(c0 + CCH + cl);
        if (split_staged(UP)) warp_tri_row<UP>(tb, a.Binv, C, a.N, c0, n0, q0, CCH, lane, q - q0, i, R);
        else load_herm_row<UP>(a.Binv + pair * tri(UP), i, R);
        for (int jj = 0; jj < J; ++jj) {
            const size_t o = (pair * J + jj) * UP + i;
            const float2 sv = i < a.U ? a.s[((size_t)nn * J + jj) * a.U + i] : make_float2(0.f, 0.f);
            float2 lam, qv;
            if (first) {                                                 // line 8
                lam = make_float2(0.f, 0.f);
                qv = c_scale(sv, a.a0);
            } else {                                                     // lines 14-15 of t-1
                const float2 mo = a.m[o], lo = a.lam[o];   // (preloading them before the wait measured slower here)
                const float2 w = c_sub(mo, lo);
                const float2 d = c_sub(sv, Wv[((size_t)nl * J + jj) * UP + i]);
                const float f = lemma2_scale(group_sum<UP>(c_norm2(d)), a.eps, a.inv_c);
                const float2 z = c_add(w, c_scale(d, f));                    // line 14 (Lemma 2)
                lam = c_sub(lo, c_scale(c_sub(mo, z), a.gamma));
                qv = c_add(z, lam);
            }
            const float2 bq = row_apply<UP>(R, buf, i, qv);
            if (fin) {
                bf_output<UP>(a.Hd + pair * (size_t)a.U * a.S, buf, i, bq, a.U, a.S, a.x + (pair * J + jj) * a.S, valid);
                continue;
            }
            const float2 m = c_sub(qv, c_scale(bq, a.rho_inv));          // line 11
            if (valid) {
                a.m[o] = m;
                a.lam[o] = lam;
                wp[(size_t)jj * CCH * UP] = c_add(wp[(size_t)jj * CCH * UP], c_sub(m, lam));   // line 12
            }
        }
    }
    if (fin) return;
    DBP_SYNCTHREADS();
    for (int e = tid; e < NT * J * UP; e += blockDim.x)      // e = (el J + jj) UP + u
        if (n0 + e / (J * UP) < a.N) a.wbuf[(size_t)n0 * J * UP + e] = cluster_sum(Wp, CCH, UP, e / UP, e % UP);
}

// ============================================================ centralized baselines

// Per subcarrier n: (G_n + delta I) v = rhs_nj for every symbol j by a lane-row
// Gauss-Jordan inverse (UP lanes per subcarrier).  UL (MMSE/ZF detection):
// rhs = wbuf [N][J][UP] (allreduced y^MRC), writes x_hat/hard [N][J][U].
// DL (ZF precoding): rhs = s [N][J][U], writes r [N][J][UP] for k_zf_out.
template <int UP, bool DL>
__global__ void __launch_bounds__(256) k_central_solve(const float2* __restrict__ Gloc, const float2* __restrict__ rhs,
                                                       float delta, int N, int J, int U, float2* __restrict__ out,
                                                       uint8_t* __restrict__ hard, Modem md, int* flag) {
    __shared__ __align__(16) float2 sbuf[256 / UP][UP];
    const int g = threadIdx.x / UP, i = threadIdx.x % UP;
    const long n = (long)blockIdx.x * (256 / UP) + g;
    const bool valid = n < N;
    const long nn = valid ? n : N - 1;
    float2 R[UP];
    load_herm_row<UP>(Gloc + (size_t)nn * tri(UP), i, R);
#pragma unroll
    for (int jc = 0; jc < UP; ++jc)              // + delta I, + 1 on padded users (exact, decoupled)
        R[jc].x += ((1u << jc) >> i) & 1u ? delta + (i >= U ? 1.f : 0.f) : 0.f;
    const bool ok = gj_invert<UP>(R, sbuf[g], i);
    if (!ok && valid) atomicOr(flag, 1);
    for (int jj = 0; jj < J; ++jj) {
        float2 b;
        if (DL) b = i < U ? rhs[((size_t)nn * J + jj) * U + i] : make_float2(0.f, 0.f);
        else b = rhs[((size_t)nn * J + jj) * UP + i];
        const float2 v = row_apply<UP>(R, sbuf[g], i, b);
        if (!valid) continue;
        if (DL) {
            out[((size_t)n * J + jj) * UP + i] = v;
        } else if (i < U) {
            out[((size_t)n * J + jj) * U + i] = v;
            if (hard) hard[((size_t)n * J + jj) * U + i] = slice_bits(v, md);
        }
    }
}

// ZF-DL output per pair: x_c = H_c^H r_n (P431), r from k_central_solve.
template <int UP>
__global__ void __launch_bounds__(256) k_zf_out(const float2* __restrict__ Hd, const float2* __restrict__ r, int N,
                                                int J, int U, int S, long npairs, float2* __restrict__ x) {
    __shared__ __align__(16) float2 sbuf[256 / UP][UP];
    const int g = threadIdx.x / UP, i = threadIdx.x % UP;
    const long p = (long)blockIdx.x * (256 / UP) + g;
    const bool valid = p < npairs;
    const long pp = valid ? p : npairs - 1;
    const long n = pp % N;
    for (int jj = 0; jj < J; ++jj)
        bf_output<UP>(Hd + (size_t)pp * U * S, sbuf[g], i, r[((size_t)n * J + jj) * UP + i], U, S,
                      x + ((size_t)pp * J + jj) * S, valid);
}

// ============================================================ launchers
static int cdiv_i(long x, long y) { return (int)((x + y - 1) / y); }

size_t iter_smem(int UP, int NT, int C) { return ((size_t)2 * NT * C * UP + (size_t)NT * UP) * 8; }
// + the staged triangles of gj_load_rows (UP = 32: one per pair)
static size_t gj_smem(int UP, int NT, int C) {
    return iter_smem(UP, NT, C) + (gj_staged(UP) ? (size_t)NT * C * tri(UP) * 8 : 0);
}

// CTA shape: NT subcarriers x C_loc clusters x UP lanes (<= 1024 threads).
bool iter_cfg(int UP, int C_loc, int N, int max_smem, int* NT) {
    const int per_n = C_loc * UP;
    if (per_n > 512) return false;
    int nt = std::max(1, 512 / per_n);
    nt = std::min(nt, N);
    while (nt > 1 && iter_smem(UP, nt, C_loc) > (size_t)max_smem) --nt;
    if (iter_smem(UP, nt, C_loc) > (size_t)max_smem) return false;
    *NT = nt;
    return true;
}

template <typename K>
static void big_smem(K k, size_t smem) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_admm_gj(const LaunchCtx& L, int UP, UlArgs a) {
    const size_t smem = gj_smem(UP, a.NT, a.C_loc);
    DBP_DISPATCH_UP(UP, big_smem(k_admm_gj<UPc>, smem);
                    k_admm_gj<UPc><<<cdiv_i(a.N, a.NT), a.NT * a.C_loc * UPc, smem, L.stream>>>(a));
    L.count(1);
    return cudaGetLastError();
}

// pbuf [NT*CCH][UP], per-slot partial sums [NT][J][CCH][UP], [NT][J][UP] consensus vector,
size_t split_smem(int UP, int NT, int CCH, int J) {
    // + per-warp staged triangles: NBUF x tri(UP) per pair slot of every (possibly partial) warp
    const size_t slots = split_staged(UP) ? (size_t)(NT * CCH * UP + 31) / 32 * (32 / UP) : 0;
    return ((size_t)NT * CCH * UP * (1 + J) + (size_t)NT * J * UP + SPLIT_NBUF * slots * tri(UP)) * 8;
}

// Split CTA shape: CCH clusters per chunk, NT subcarriers, ~TH threads: small CTAs, so
// several per SM hide each other's load latency (split_scaling_proxy.py, world-8 shares:
// E ADMM-UL 1725 / 1500 / 1421 us and C ADMM-DL at world 2 195 / 185 / 183 us at
// TH = 512 / 256 / 128).
#ifndef DBP_SPLIT_THREADS
#define DBP_SPLIT_THREADS 0
#endif
void split_cfg(int UP, int C_loc, int N, int J, int* NT, int* CCH) {
    const int TH = DBP_SPLIT_THREADS ? std::min(DBP_SPLIT_THREADS, 256) : (UP >= 32 ? 128 : 256);
    int cch = std::max(1, std::min(C_loc, TH / UP));
    int nt = std::max(1, std::min(N, TH / (cch * UP)));
    *NT = nt;
    *CCH = cch;
}

cudaError_t launch_admm_it(const LaunchCtx& L, int UP, UlArgs a, int CCH) {
    const size_t smem = split_smem(UP, a.NT, CCH, a.J);
    if (a.init) {
        DBP_DISPATCH_UP(UP, big_smem(k_admm_it<UPc, true>, smem);
                        k_admm_it<UPc, true><<<cdiv_i(a.N, a.NT), a.NT * CCH * UPc, smem, L.stream>>>(a, CCH));
    } else {
        DBP_DISPATCH_UP(UP, big_smem(k_admm_it<UPc, false>, smem);
                        k_admm_it<UPc, false><<<cdiv_i(a.N, a.NT), a.NT * CCH * UPc, smem, L.stream>>>(a, CCH));
    }
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_bf_gj(const LaunchCtx& L, int UP, DlArgs a) {
    const size_t smem = gj_smem(UP, a.NT, a.C_loc);
    const int grid = cdiv_i(a.N, a.NT), nthr = a.NT * a.C_loc * UP;
    DBP_DISPATCH_UP(UP,
        if constexpr (UPc <= 16) {
            if (a.J > 1) {
                big_smem(k_bf_gj<UPc, 2>, smem);
                k_bf_gj<UPc, 2><<<grid, nthr, smem, L.stream>>>(a);
            } else {
                big_smem(k_bf_gj<UPc, 1>, smem);
                k_bf_gj<UPc, 1><<<grid, nthr, smem, L.stream>>>(a);
            }
        } else {
            big_smem(k_bf_gj<UPc, 1>, smem);
            k_bf_gj<UPc, 1><<<grid, nthr, smem, L.stream>>>(a);
        });
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_central_solve(const LaunchCtx& L, int UP, bool dl, const float2* Gloc, const float2* rhs, float delta,
                                 int N, int J, int U, float2* out, uint8_t* hard, Modem md) {
    DBP_DISPATCH_UP(UP,
        if (dl) k_central_solve<UPc, true><<<cdiv_i(N, 256 / UPc), 256, 0, L.stream>>>(Gloc, rhs, delta, N, J, U, out,
                                                                                    hard, md, L.flag);
        else k_central_solve<UPc, false><<<cdiv_i(N, 256 / UPc), 256, 0, L.stream>>>(Gloc, rhs, delta, N, J, U, out,
                                                                                   hard, md, L.flag));
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_zf_out(const LaunchCtx& L, int UP, const float2* Hd, const float2* r, int N, int J, int U, int S,
                          long npairs, float2* x) {
    DBP_DISPATCH_UP(UP, k_zf_out<UPc><<<cdiv_i(npairs, 256 / UPc), 256, 0, L.stream>>>(Hd, r, N, J, U, S, npairs, x));
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_bf_it(const LaunchCtx& L, int UP, DlArgs a, int CCH) {
    const size_t smem = split_smem(UP, a.NT, CCH, a.J);
    if (a.step > a.T) {
        DBP_DISPATCH_UP(UP, big_smem(k_bf_it<UPc, true>, smem);
                        k_bf_it<UPc, true><<<cdiv_i(a.N, a.NT), a.NT * CCH * UPc, smem, L.stream>>>(a, CCH));
    } else {
        DBP_DISPATCH_UP(UP, big_smem(k_bf_it<UPc, false>, smem);
                        k_bf_it<UPc, false><<<cdiv_i(a.N, a.NT), a.NT * CCH * UPc, smem, L.stream>>>(a, CCH));
    }
    L.count(1);
    return cudaGetLastError();
}

}  // namespace dbp
