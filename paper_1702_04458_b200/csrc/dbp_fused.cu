// dbp_fused.cu -- k_fused: one launch per solver on one GPU (world == 1),
// SURVEY 8(a) rows a1-a8 (Alg. 1), b1-b5 (Alg. 2), c1-c4 (Alg. 3).
//
// A CTA owns NPC subcarriers with all C clusters of each (WPS = C/PW warps
// per subcarrier, NPC * WPS = 4 warps), so the whole per-subcarrier method --
// local preprocessing, every consensus round, the output -- runs on chip:
//
//   SOLVER 1 (ADMM-UL, Alg. 1): Gram + matched filter (folded rows, per-warp
//     TMA ring, dbp_fold.cuh), Hermitian sweep with the bordered matched
//     filter -> rho B_c^{-1} and y^reg_c in registers; T consensus rounds:
//     z_c = y^reg_c + rho B_c^{-1}(s - lambda_c) (folded Hermitian mat-vec),
//     w = sum_c (z_c + lambda_c) in fixed cluster order through shared
//     memory (the consensus "allreduce" of P744 over the CTA), prox (E2),
//     lambda update (E3); s_hat + hard bits.
//   SOLVER 2 (ADMM-DL, Alg. 3): B_c = H_c H_c^H + rho^{-1} I, sweep -> B_c^{-1};
//     exact m-form iterations (reading 12); output x_c = H_c^H B_c^{-1} q_c
//     re-streams H_c through the same ring (second pass, L2-resident: it was
//     read microseconds earlier by the same CTA).
//   SOLVER 0 (CG-UL, Alg. 2): Gram + matched filter, the cluster sums
//     G = sum_c G_c and y^MRC = sum_c H_c^H y_c (P416 footnote; the per-round
//     allreduce of w_c = G_c p degenerates to this sum at world == 1), then T
//     CG iterations on UP lanes per subcarrier (shuffle dot products, P715).
//
// Versus the split path (k_prefold -> B^{-1} in HBM -> iteration kernels):
// no per-pair inverse is written or re-read (2 x 42 MB for config C/D), the
// DL output's second H read hits L2, and each solver is a single launch.
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_fold.cuh"
#include "dbp_internal.h"
#include "dbp_tc.cuh"

#pragma nv_diag_suppress 128   // SOLVER 0 continues before the inverse: "loop is not reachable"

namespace dbp {

template <int UP, int SOLVER>
struct FZ {
    using F = Fold<UP>;
    static constexpr bool DL = SOLVER == 2 || SOLVER == 4;
    static constexpr bool SUMS = SOLVER == 0 || SOLVER == 3 || SOLVER == 4;   // cluster-summed Gram
    static constexpr bool MF = !DL;
    using G = FoldStage<UP, DL, MF>;
    static constexpr int WARPS = 4;
#ifndef DBP_FZ_NST
#define DBP_FZ_NST 2
#endif
    static constexpr int NST = DBP_FZ_NST;
#ifndef DBP_FZ_TC
#define DBP_FZ_TC 0
#endif
    // UP = 16: the per-pair Gram (+ matched filter) runs on the tensor cores (dbp_tc.cuh); a
    // TMA stage is then one whole pair (runtime size, 128B-swizzled), the warp's 8 pairs are
    // computed one after another and handed to the folded layout through shared memory in two
    // halves of 4 pairs (gtri / mfl, aliasing the mat-vec partials ybuf).
    static constexpr bool TC = UP == 16 && DBP_FZ_TC;
    static constexpr int PWL = F::PW * F::PLP;            // pivot / vector lines (float2)
    static constexpr int DLN = F::PW * UP;                // Jacobi scales (float)
    static constexpr int YB = F::PW * fold_ybuf_pair<UP>(); // mat-vec partials (float2), padded
    static constexpr int TCB = TC ? 4 * F::TRI + 4 * UP : 0;  // TC hand-off: 4 packed Grams + 4 H^H y
    static constexpr int UNI = (YB > TCB ? YB : TCB);      // float2
    // per-warp region after the ring: pivot lines, Jacobi scales, ybuf / TC hand-off
    static constexpr int LOC = (PWL * 8 + DLN * 4 + UNI * 8 + 127) / 128 * 128;
    static constexpr int WREG = (NST * G::STG + LOC + 127) / 128 * 128;   // non-TC (stage size static)
    // CTA-shared: per-warp consensus partials [WARPS][UP] + per-subcarrier sums [4][UP];
    // CG: per-warp Gram partials [WARPS][TRI] + per-subcarrier Gram [4][TRI]
    static constexpr int CBUF = WARPS * UP * 8 + WARPS * UP * 8;       // Wp + Sv
    static constexpr int GBUF = SUMS ? 2 * WARPS * F::TRI * 8 : 0;
    // + 1024: the base is rounded up to 1024 B in the kernel (128B-swizzled TMA destinations)
    static size_t smem(int wreg) { return 1024 + (size_t)WARPS * wreg + 128 + CBUF + GBUF; }
};

struct FuArgs {
    XArgs xc;
    int S, U, N, C, T, WPS, NPC;
    int stg, wreg, nkk, nsb, stage_bytes, yoff;   // ring stage pitch, per-warp region pitch; TC: K steps, DL boxes, y offset
    float rho, gamma, delta;
    // UL outputs (SOLVER 0, 1)
    float2* s_hat;        // [N][U]
    uint8_t* hard;        // [N][U] or null
    Prox px;
    Modem md;
    // DL (SOLVER 2)
    const float2* s;      // [N][U]
    float2* x;            // [C][N][S]
    float rho_inv, a0, inv_c, eps;
    int* flag;
};

template <int UP, int SOLVER>
#ifndef DBP_FZ_MINB
#define DBP_FZ_MINB 3
#endif
__global__ void __launch_bounds__(128, DBP_FZ_MINB)
k_fused(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmY, FuArgs a) {
    using Z = FZ<UP, SOLVER>;
    using F = Fold<UP>;
    using G = typename Z::G;
    constexpr int L = F::L, PW = F::PW, SC = F::SC, NST = Z::NST, R = F::R, TRI = F::TRI;
    constexpr bool DL = Z::DL, MF = Z::MF;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DBP_POISON_SMEM(smem_raw);
    griddep_launch();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // 1024-aligned base: [4 warp regions][mbarriers + CG queue (128 B)][Wp, Sv, Gp, Gs]
    unsigned char* const base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* const cta = base + (size_t)Z::WARPS * a.wreg;
    uint64_t* bar = reinterpret_cast<uint64_t*>(cta) + warp * NST;
    unsigned char* wbase = base + (size_t)warp * a.wreg;
    unsigned char* const wloc = wbase + NST * a.stg;
    const int q = lane / L, l = lane % L;
    float2* pl = reinterpret_cast<float2*>(wloc) + q * F::PLP;                             // pivots / vectors
    float* dline = reinterpret_cast<float*>(wloc + Z::PWL * 8) + q * UP;
    float2* const uni = reinterpret_cast<float2*>(wloc + Z::PWL * 8 + Z::DLN * 4);
    float2* ybuf = uni + q * fold_ybuf_pair<UP>();
    float2* Wp = reinterpret_cast<float2*>(cta + 128);                                     // [4 warps][UP]
    float2* Sv = Wp + Z::WARPS * UP;                                                       // [4 subc.][UP]
    float2* Gp = Sv + Z::WARPS * UP;                                                       // CG: [4 warps][TRI]
    float2* Gs = Gp + (Z::SUMS ? Z::WARPS * TRI : 0);                                      // queue: [4][TRI]

    int row[R];
#pragma unroll
    for (int m = 0; m < R; ++m) row[m] = F::row(m, l);

    const int WPS = a.WPS, NPC = a.NPC;
    const int j = warp / WPS;                          // subcarrier slot of this warp
    const int cb = warp - j * WPS;                     // cluster block
    const int c = cb * PW + q;                         // this pair's cluster
    const int ngroups = (a.N + NPC - 1) / NPC;
    const int nitems = blockIdx.x < ngroups ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int nch = Z::TC ? PW : (a.S + SC - 1) / SC;  // stages per pass: TC one per pair, else SC antennas
#ifndef DBP_EXP_NO_DLOUT
#define DBP_EXP_NO_DLOUT 0      // experiment only: drop the DL output pass (wrong results; timing the pass)
#endif
    const int per_item = DL && !DBP_EXP_NO_DLOUT ? 2 * nch : nch;   // DL: Gram pass + output pass
    const int nseq = nitems * per_item;

    // TMA issue cursor (lane 0): the (item, chunk) of the next stage to load, advanced by one
    // per issue -- no division on the per-stage path
    int is_item = 0, is_ch = 0;
    auto issue = [&](int st) {
        const int ch = is_ch >= nch ? is_ch - nch : is_ch;
        const int n = (blockIdx.x + is_item * gridDim.x) * NPC + j;
        unsigned char* dst = wbase + st * a.stg;
        mbar_arrive_expect_tx(&bar[st], (uint32_t)a.stage_bytes);
        if (Z::TC) {
            // one whole pair (cluster cb * PW + ch): UL H [S8][16] + y [S8]; DL nsb boxes [16][16]
            if (DL) {
                for (int sb = 0; sb < a.nsb; ++sb) tma_load4(dst + sb * 2048, &tmH, 16 * sb, 0, n, cb * PW + ch, &bar[st]);
            } else {
                tma_load4(dst, &tmH, 0, 0, n, cb * PW + ch, &bar[st]);
                tma_load4(dst + a.yoff, &tmY, 0, 0, n, cb * PW + ch, &bar[st]);
            }
        } else if (DL) {
            tma_load4(dst, &tmH, ch * SC, 0, n, cb * PW, &bar[st]);
        } else {
            tma_load4(dst, &tmH, 0, ch * SC, n, cb * PW, &bar[st]);
            tma_load4(dst + G::HSZ * 8, &tmY, ch * SC, 0, n, cb * PW, &bar[st]);
        }
        if (++is_ch == per_item) { is_ch = 0; ++is_item; }
    };
    if (lane == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    DBP_SYNCWARP();
    if (lane == 0)
        for (int s = 0; s < NST && s < nseq; ++s) issue(s);

    int sq = 0, st = 0, qn = 0;
    uint32_t phase = 0;
    static_assert(Z::WARPS * NST * 8 <= 96, "mbarriers overlap the CG queue indices");
    int* qsub = reinterpret_cast<int*>(cta + 96);          // CG queue: subcarrier of each slot
    auto next_stage = [&]() {
        DBP_SYNCWARP();
        if (lane == 0 && sq + NST < nseq) {
            fence_proxy_async();
            issue(st);
        }
        ++sq;
        if (++st == NST) { st = 0; phase ^= 1u; }
    };

    // DL output pass: x_c[s] = sum_u conj(H_us) r_u, re-streaming H_c through the ring (its second
    // pass, L2-resident); lane l takes antennas l, l+L, ... of each stage.  (Reading H_c directly
    // from L2 with LDG instead measured 30% slower for the whole kernel.)
    // TC: the warp's PW pairs one after another, pair p's H^d re-streamed as one stage; lane s
    // takes antennas s, s + 32 (128B-swizzled [16 users][16 antennas] boxes); r of pair p is the
    // UP-line rl + p * rstride (ADMM-DL: the pair's pivot line; ZF-DL: the subcarrier's solution).
    auto dl_output_tc = [&](const float2* rl, int rstride, int n) {
        griddep_wait();
        for (int p = 0; p < PW; ++p) {
            mbar_wait(&bar[st], phase);
            const unsigned char* hs = wbase + st * a.stg;
            float2 r[UP];
            read_vec<UP>(rl + p * rstride, r);
            const int cl = cb * PW + p;
            for (int s = lane; s < a.S; s += 32) {
                const int sb = s >> 4, sl = s & 15;
                f2x acc = 0ull;
#pragma unroll
                for (int u = 0; u < UP; ++u) {
                    const float2 h = *reinterpret_cast<const float2*>(hs + sb * 2048 + u * 128 +
                                                                     (((sl >> 1) ^ (u & 7)) << 4) + ((sl & 1) << 3));
                    x2_cmac(acc, r[u], h.x, h.y);
                }
                if (n < a.N && cl < a.C) a.x[((size_t)cl * a.N + n) * a.S + s] = c_conj(upk2(acc));
            }
            next_stage();
        }
    };
    auto dl_output = [&](const float2 (&r)[UP], int n, bool valid) {
        using GD = FoldStage<UP, true, false>;
        float2* xo = a.x + ((size_t)c * a.N + n) * a.S;
        griddep_wait();
        for (int ch = 0; ch < nch; ++ch) {
            mbar_wait(&bar[st], phase);
            const float2* hq = reinterpret_cast<const float2*>(wbase + st * a.stg) + q * GD::NL * GD::HL;
#pragma unroll
            for (int sl = l; sl < SC; sl += L) {
                // conj(x_s) = sum_u conj(r_u) H_us: r_u is the reused FFMA2 pair operand
                f2x acc = 0ull;
#pragma unroll
                for (int u = 0; u < UP; ++u) {
                    const float2 h = hq[u * GD::HL + sl];
                    x2_cmac(acc, r[u], h.x, h.y);
                }
                const int s = ch * SC + sl;
                if (valid && s < a.S) xo[s] = c_conj(upk2(acc));
            }
            next_stage();
        }
    };

    for (int it = 0; it < nitems; ++it) {
        const int n = (blockIdx.x + it * gridDim.x) * NPC + j;
        const bool valid = n < a.N && c < a.C;

        // ------------------------------------------------ local Gram (+ matched filter)
        f2x A[F::NSLOT];
#pragma unroll
        for (int e = 0; e < F::NSLOT; ++e) A[e] = 0ull;
        f2x E[R];
#pragma unroll
        for (int m = 0; m < R; ++m) E[m] = 0ull;
        if constexpr (Z::TC) {
            // tensor-core Gram (+ H^H y), one pair per stage, handed to the folded slots 4 pairs at a time
            const int g = lane >> 2, t4 = lane & 3;
            float2* gtri = uni;
            float2* mfl = uni + 4 * TRI;
            for (int h = 0; h < 2; ++h) {
                for (int p4 = 0; p4 < 4; ++p4) {
                    mbar_wait(&bar[st], phase);
                    if constexpr (DBP_FZ_TC == 2) {
                        // fp16 Z + Z^H Gram; the consumed stage doubles as the transpose scratch
                        unsigned char* sb = wbase + st * a.stg;
                        tc16_gram_pair<DL, MF>(sb, a.nkk, gtri + p4 * TRI, mfl + p4 * UP,
                                               reinterpret_cast<float2*>(sb), g, t4, lane);
                    } else {
                        float acc[5][4];
                        tc_gram<DL, MF>(acc, wbase + st * a.stg, a.nkk, g, t4);
                        tc_store<DL, MF>(acc, gtri + p4 * TRI, mfl + p4 * UP, g, t4);
                    }
                    next_stage();
                }
                DBP_SYNCWARP();
                if ((q >> 2) == h) {
                    const float2* gq = gtri + (q & 3) * TRI;
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        const int rb = (row[m] * (row[m] + 1)) / 2;
#pragma unroll
                        for (int tt = 0; tt < (m + 1) * L; ++tt)
                            A[F::off(m) + tt] = tt <= row[m] ? pk2(gq[rb + tt]) : 0ull;
                        if (MF) E[m] = pk2(mfl[(q & 3) * UP + row[m]]);
                    }
                }
                DBP_SYNCWARP();
            }
        } else {
            for (int ch = 0; ch < nch; ++ch) {
                mbar_wait(&bar[st], phase);
                const float2* stage = reinterpret_cast<const float2*>(wbase + st * a.stg);
                if (DL) fold_gram_dl<UP>(A, stage, q, row);
                else fold_gram_ul<UP, true>(A, E, stage, q, row);
                next_stage();
            }
        }
        float dg[R];
        fold_diag<UP>(A, row, a.delta, dg);

        if constexpr (Z::SUMS) {
            // ---------------------------------------------- cluster sums (CG, MMSE-UL, ZF-DL)
            // sum over the warp's pairs (xor butterfly over the pair bits of the lane), then
            // over the subcarrier's WPS warps in fixed order: G = sum_c G_c, y^MRC = sum_c H_c^H y_c
#pragma unroll
            for (int e = 0; e < F::NSLOT; ++e) {
                float2 v = valid ? upk2(A[e]) : make_float2(0.f, 0.f);
#pragma unroll
                for (int o = L; o < 32; o <<= 1) {
                    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
                    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
                }
                A[e] = pk2(v);
            }
#pragma unroll
            for (int m = 0; m < R; ++m) {
                float2 v = valid ? upk2(E[m]) : make_float2(0.f, 0.f);
#pragma unroll
                for (int o = L; o < 32; o <<= 1) {
                    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
                    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
                }
                E[m] = pk2(v);
            }
            if (lane < L) {
                fold_store<UP>(Gp + warp * TRI, A, row);
#pragma unroll
                for (int m = 0; m < R; ++m) Wp[warp * UP + row[m]] = upk2(E[m]);
            }
            DBP_SYNCTHREADS();
            // the subcarrier sums go to CG queue slots qn..qn+NPC-1 (4 slots, one per warp)
            for (int e = tid; e < NPC * (TRI + UP); e += Z::WARPS * 32) {
                const int jj = e / (TRI + UP), f = e - jj * (TRI + UP);
                float2 acc = make_float2(0.f, 0.f);
                if (f < TRI) {
                    for (int w2 = 0; w2 < WPS; ++w2) acc = c_add(acc, Gp[(jj * WPS + w2) * TRI + f]);
                    Gs[(qn + jj) * TRI + f] = acc;
                } else {
                    for (int w2 = 0; w2 < WPS; ++w2) acc = c_add(acc, Wp[(jj * WPS + w2) * UP + f - TRI]);
                    Sv[(qn + jj) * UP + f - TRI] = acc;
                }
            }
            if (tid < NPC) qsub[qn + tid] = (blockIdx.x + it * gridDim.x) * NPC + tid;
            qn += NPC;
            DBP_SYNCTHREADS();
            // exact solve of queue slot w on the warp's UP-lane groups (lane-row Gauss-Jordan,
            // dbp_lanerow.cuh): returns ((G_w + delta I)^{-1} rhs)_u for u = lane % UP
            auto solve = [&](int w, float delta, float2 rhs_u, bool live) {
                const int u = lane % UP;
                const float2* Gj = Gs + w * TRI;
                float2 grow[UP];
#pragma unroll
                for (int jc = 0; jc < UP; ++jc) {
                    grow[jc] = jc <= u ? Gj[(u * (u + 1)) / 2 + jc] : c_conj(Gj[(jc * (jc + 1)) / 2 + u]);
                    // + delta on the diagonal, + 1 for padded users (u >= U): the padding stays decoupled
                    // and exact at delta = 0 (ZF); (jc == u) as a bit test, without local memory
                    grow[jc].x += ((1u << jc) >> u) & 1u ? delta + (u >= a.U ? 1.f : 0.f) : 0.f;
                }
                float2* P = pl - q * F::PLP + (lane / UP) * F::PLP;          // a per-group line
                const bool ok = gj_invert<UP>(grow, P, u);
                if (!ok && live) atomicOr(a.flag, 1);        // padding subcarriers (n >= N) have G = 0
                return row_apply<UP>(grow, P, u, rhs_u);
            };
            if constexpr (SOLVER == 4) {
                // ZF-DL: r = (sum_c H_c H_c^H)^{-1} s per subcarrier, then x_c = H_c^H r (P431)
                if (warp < NPC) {
                    const int nn = (blockIdx.x + it * gridDim.x) * NPC + warp;
                    const int u = lane % UP;
                    const float2 sv = (u < a.U && nn < a.N) ? a.s[(size_t)nn * a.U + u] : make_float2(0.f, 0.f);
                    const float2 r = solve(warp, 0.f, sv, nn < a.N);
                    DBP_SYNCWARP();
                    if (lane < UP) Sv[warp * UP + u] = r;
                }
                qn = 0;
                DBP_SYNCTHREADS();
                if constexpr (Z::TC) {
                    dl_output_tc(Sv + j * UP, 0, n);
                } else {
                    float2 r[UP];
                    read_vec<UP>(Sv + j * UP, r);
                    dl_output(r, n, valid);
                }
                DBP_SYNCTHREADS();                        // Sv / Gs reused by the next item
                continue;
            } else {
                if (qn < Z::WARPS && it + 1 < nitems) continue;
                // up to 4 queued subcarriers, one per warp (all warps busy)
                if (warp < qn) {
                    const int nn = qsub[warp];
                    const int u = lane % UP;
                    float2 x;
                    if constexpr (SOLVER == 3) {
                        x = solve(warp, a.rho, Sv[warp * UP + u], nn < a.N); // (G + N0/Es I)^{-1} y^MRC
                    } else {
                        const float2* Gj = Gs + warp * TRI;
                        float2 grow[UP];                        // row u of G in registers
#pragma unroll
                        for (int jc = 0; jc < UP; ++jc)
                            grow[jc] = jc <= u ? Gj[(u * (u + 1)) / 2 + jc] : c_conj(Gj[(jc * (jc + 1)) / 2 + u]);
                        float2* P = pl - q * F::PLP + (lane / UP) * F::PLP;          // a per-group line
                        // device-side consensus (NEXT-1): sum of v over ranks for round t (LL words)
                        auto xsum = [&](int t, float2 v) {
                            if (!a.xc.on || nn >= a.N) return v;
                            const unsigned rid = a.xc.base + (unsigned)t;
                            const int par = rid & 1u;
                            const size_t o = ((size_t)(par * 8 + a.xc.rank) * a.xc.cap + nn) * UP + u;
                            for (int rk = 0; rk < a.xc.world; ++rk) st_ll_sys(a.xc.part[rk] + o, v, rid);
                            float2 sum = make_float2(0.f, 0.f);
                            for (int pk = 0; pk < a.xc.world; ++pk)
                                sum = c_add(sum, ld_ll_sys(a.xc.part[a.xc.rank] +
                                                           ((size_t)(par * 8 + pk) * a.xc.cap + nn) * UP + u, rid,
                                                           a.flag));
                            return sum;
                        };
                        float2 r = xsum(1, Sv[warp * UP + u]);  // line 6: r = y^MRC (consensus), p = r, x = 0
                        float2 p = r;
                        x = make_float2(0.f, 0.f);
                        float rr = group_sum<UP>(c_norm2(r));
                        for (int t = 0; t < a.T; ++t) {
                            DBP_SYNCWARP();
                            P[u] = p;
                            DBP_SYNCWARP();
                            float2 pv[UP];
                            read_vec<UP>(P, pv);
                            float2 w = make_float2(0.f, 0.f);                            // lines 9-11: w = G p
#pragma unroll
                            for (int jc = 0; jc < UP; ++jc) c_fma(w, grow[jc], pv[jc]);
                            w = xsum(2 + t, w);                                          // line 11 consensus
                            cg_update<UP>(x, r, p, rr, w, a.rho);                        // lines 13-18
                        }
                    }
                    griddep_wait();
                    if (lane < UP && u < a.U && nn < a.N) {
                        a.s_hat[(size_t)nn * a.U + u] = x;
                        if (a.hard) a.hard[(size_t)nn * a.U + u] = slice_bits(x, a.md);
                    }
                }
                qn = 0;
                DBP_SYNCTHREADS();                        // queue slots reused
                continue;
            }
        }

        // ------------------------------------------------ B^{-1} (+ y^reg) by the Hermitian sweep
        float dr[R];
        fold_jacobi<UP, !DL>(A, E, dg, dr, dline, row);
        const bool ok = fold_sweep<UP, !DL>(A, E, pl, row, l);
        if (!ok && valid) atomicOr(a.flag, 1);
        fold_unscale_mv<UP, !DL>(A, E, dr, dline, DL ? 1.f : a.rho, row);   // UL: rho B^{-1} (eq. (3))

        // consensus over the subcarrier's clusters, Sv[j] <- f(sum_c w_c): xor butterfly over the
        // warp's pairs, then the WPS warp partials in fixed order (deterministic)
        // consensus over the subcarrier's clusters: xor butterfly over the warp's pairs, the WPS
        // warp partials summed in fixed order by UP threads per subcarrier (deterministic) into
        // Sv; returns f(sum_c w_c) for the lane's rows, f = prox (UL) or identity (DL).  (A
        // one-barrier variant, every lane summing its own rows, measured slower.)
        auto consensus = [&](int t, const float2 (&w)[R], bool do_prox, float2 (&out)[R]) {
            float2 ps[R];
#pragma unroll
            for (int m = 0; m < R; ++m) {
                ps[m] = valid ? w[m] : make_float2(0.f, 0.f);
#pragma unroll
                for (int o = L; o < 32; o <<= 1) {
                    ps[m].x += __shfl_xor_sync(0xffffffffu, ps[m].x, o);
                    ps[m].y += __shfl_xor_sync(0xffffffffu, ps[m].y, o);
                }
            }
            if (lane < L) {
#pragma unroll
                for (int m = 0; m < R; ++m) Wp[warp * UP + row[m]] = ps[m];
            }
            DBP_SYNCTHREADS();
            if (!a.xc.on) {
                if (tid < NPC * UP) {
                    const int jj = tid / UP, u = tid - jj * UP;
                    float2 acc = make_float2(0.f, 0.f);
                    for (int w2 = 0; w2 < WPS; ++w2) acc = c_add(acc, Wp[(jj * WPS + w2) * UP + u]);
                    Sv[tid] = do_prox ? prox(acc, a.px) : acc;
                }
            } else {
                // rank-local partial -> every rank's buffer, then the sum over ranks (NEXT-1).
                // LL protocol: each 8-byte word carries its own round id ({re, rid}, {im, rid}), so
                // a reader polls its entry until both ids match -- no fence, no separate flag.
                const unsigned rid = a.xc.base + (unsigned)t;
                const int par = rid & 1u;
                const int n0 = (blockIdx.x + it * gridDim.x) * NPC;
                if (tid < NPC * UP) {
                    const int jj = tid / UP, u = tid - jj * UP;
                    float2 acc = make_float2(0.f, 0.f);
                    for (int w2 = 0; w2 < WPS; ++w2) acc = c_add(acc, Wp[(jj * WPS + w2) * UP + u]);
                    float2 sum = make_float2(0.f, 0.f);
                    if (n0 + jj < a.N) {
                        const size_t o = ((size_t)(par * 8 + a.xc.rank) * a.xc.cap + n0 + jj) * UP + u;
                        for (int r = 0; r < a.xc.world; ++r) st_ll_sys(a.xc.part[r] + o, acc, rid);
                        for (int p = 0; p < a.xc.world; ++p)        // rank order: identical sums everywhere
                            sum = c_add(sum, ld_ll_sys(a.xc.part[a.xc.rank] +
                                                       ((size_t)(par * 8 + p) * a.xc.cap + n0 + jj) * UP + u, rid,
                                                       a.flag));
                    }
                    Sv[tid] = do_prox ? prox(sum, a.px) : sum;
                }
            }
            DBP_SYNCTHREADS();
#pragma unroll
            for (int m = 0; m < R; ++m) out[m] = Sv[j * UP + row[m]];
        };
        auto last_out = [&](int u) { return Sv[j * UP + u]; };   // entry u of the last round (output lanes)

        if constexpr (SOLVER == 1) {
            // ---------------------------------------------- ADMM-UL iterations (Alg. 1 lines 10-19)
            float2 yreg[R], lam[R], z[R], w[R];
#pragma unroll
            for (int m = 0; m < R; ++m) {
                yreg[m] = upk2(E[m]);
                lam[m] = make_float2(0.f, 0.f);
                z[m] = yreg[m];
                w[m] = yreg[m];
            }
            float2 sc[R];
            consensus(1, w, true, sc);
            for (int t = 2; t <= a.T; ++t) {
                float2 v[R], bv[R];
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    lam[m] = c_add(lam[m], c_scale(c_sub(z[m], sc[m]), a.gamma));  // line 12
                    v[m] = c_sub(sc[m], lam[m]);
                }
                fold_mv<UP>(A, v, bv, pl, ybuf, row, l);                          // rho B^{-1} (s - lambda)
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    z[m] = c_add(yreg[m], bv[m]);                                 // line 15
                    w[m] = c_add(z[m], lam[m]);                                   // line 17
                }
                consensus(t, w, true, sc);                                        // lines 18-19
            }
            griddep_wait();
            if (warp == j * WPS && lane < UP) {
                const int u = lane;
                if (u < a.U && n < a.N) {
                    const float2 s = last_out(u);
                    a.s_hat[(size_t)n * a.U + u] = s;
                    if (a.hard) a.hard[(size_t)n * a.U + u] = slice_bits(s, a.md);
                }
            }
        } else {
            // ---------------------------------------------- ADMM-DL iterations (Alg. 3, m-form)
            float2 sv[R], lam[R], qv[R];
#pragma unroll
            for (int m = 0; m < R; ++m) {
                sv[m] = (row[m] < a.U && n < a.N) ? a.s[(size_t)n * a.U + row[m]] : make_float2(0.f, 0.f);
                lam[m] = make_float2(0.f, 0.f);
                qv[m] = c_scale(sv[m], a.a0);                                     // line 8
            }
            for (int t = 2; t <= a.T; ++t) {
                float2 bq[R], mm[R], w[R];
                fold_mv<UP>(A, qv, bq, pl, ybuf, row, l);
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    mm[m] = c_sub(qv[m], c_scale(bq[m], a.rho_inv));               // line 11
                    w[m] = c_sub(mm[m], lam[m]);                                   // line 12
                }
                float2 W[R];
                consensus(t - 1, w, false, W);                                     // line 13 (round ids base+1..)
                float2 dv[R];
                float nrm2 = 0.f;
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    dv[m] = c_sub(sv[m], W[m]);
                    nrm2 += c_norm2(dv[m]);
                }
#pragma unroll
                for (int o = 1; o < L; o <<= 1) nrm2 += __shfl_xor_sync(0xffffffffu, nrm2, o);   // ||s - w|| of the pair
                const float f = lemma2_scale(nrm2, a.eps, a.inv_c);
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    const float2 z = c_add(w[m], c_scale(dv[m], f));                                    // line 14
                    lam[m] = c_sub(lam[m], c_scale(c_sub(mm[m], z), a.gamma));                          // line 15
                    qv[m] = c_add(z, lam[m]);
                }
            }
            float2 rv[R];
            fold_mv<UP>(A, qv, rv, pl, ybuf, row, l);                             // r = B^{-1} q
            // publish r for the pair; every lane takes all UP entries
            DBP_SYNCWARP();
#pragma unroll
            for (int m = 0; m < R; ++m) pl[row[m]] = rv[m];
            DBP_SYNCWARP();
            if constexpr (Z::TC) {
                dl_output_tc(pl - q * F::PLP, F::PLP, n);
            } else if (!DBP_EXP_NO_DLOUT) {
                float2 r[UP];
                read_vec<UP>(pl, r);
                dl_output(r, n, valid);
            }
        }
    }
}

static int g_sms_fz = 0;

template <int UP, int SOLVER>
constexpr int NST_of() { return FZ<UP, SOLVER>::NST; }

template <int UP, int SOLVER>
static bool launch_fz_t(const LaunchCtx& L, const float2* H, const float2* y, FuArgs a) {
    using Z = FZ<UP, SOLVER>;
    using F = Fold<UP>;
    CUtensorMap tmH{}, tmY{};
    // H: UL [C][N][S][U] -> dims (U, S, N, C); DL [C][N][U][S] -> dims (S, U, N, C); y [C][N][1][S]
    if constexpr (Z::TC) {
        // TF32 path: K8 steps (S rounded to 8); FP16 path: K16 steps (S rounded to 16)
        const int S8 = DBP_FZ_TC == 2 ? (a.S + 15) / 16 * 16 : (a.S + 7) / 8 * 8;
        a.nsb = (a.S + 15) / 16;
        if (!Z::DL) {
            if (!make_map4(&tmH, H, a.U, a.S, a.N, a.C, 16, S8, 1, 1, true)) return false;
            if (!make_map4(&tmY, y, a.S, 1, a.N, a.C, S8, 1, 1, 1)) return false;
            a.nkk = DBP_FZ_TC == 2 ? S8 / 16 : S8 / 8;
            a.stage_bytes = S8 * 128 + S8 * 8;
            a.yoff = S8 * 128;
        } else {
            if (!make_map4(&tmH, H, a.S, a.U, a.N, a.C, 16, 16, 1, 1, true)) return false;
            a.nkk = DBP_FZ_TC == 2 ? a.nsb : 2 * a.nsb;
            a.stage_bytes = a.nsb * 2048;
        }
        // TC == 2 reuses the consumed stage as the [16][17] float2 transpose scratch (2176 B)
        a.stg = (std::max(a.stage_bytes, DBP_FZ_TC == 2 ? 16 * 17 * 8 : 0) + 1023) / 1024 * 1024;
        a.wreg = (NST_of<UP, SOLVER>() * a.stg + Z::LOC + 1023) / 1024 * 1024;
    } else {
        if (!Z::DL) {
            if (!make_map4(&tmH, H, a.U, a.S, a.N, a.C, UP + 2, F::SC, 1, F::PW)) return false;
            if (!make_map4(&tmY, y, a.S, 1, a.N, a.C, F::SC, 1, 1, F::PW)) return false;
        } else {
            if (!make_map4(&tmH, H, a.S, a.U, a.N, a.C, F::SC, UP + 1, 1, F::PW)) return false;
        }
        a.stg = Z::G::STG;
        a.stage_bytes = Z::G::BYTES;
        a.wreg = Z::WREG;
    }
    const size_t SMEM = Z::smem(a.wreg);
    if (!g_sms_fz) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms_fz, cudaDevAttrMultiProcessorCount, dev);
    }
    auto k = k_fused<UP, SOLVER>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, Z::WARPS * 32, SMEM);
    const int ngroups = (a.N + a.NPC - 1) / a.NPC;
    // Grid per solver (bit SOLVER of the mask set: persistent, one wave of resident CTAs striding over the
    // subcarrier groups; clear: one CTA per group, the hardware scheduler balancing the tail).  Measured
    // on config C/D: one CTA per group is faster for ADMM-UL / ADMM-DL (99.5 -> 95.7,
    // 111.5 -> 107.7 us) and ZF-DL (83 -> 80 us), persistent for CG-UL (two-stream step) and MMSE-UL
    // (66.5 vs 69 us).  DBP_FZ_PERSIST overrides the mask.
    static const int persist = [] { const char* e = getenv("DBP_FZ_PERSIST"); return e ? (int)strtol(e, nullptr, 0) : 0x09; }();
    if (a.xc.on) {
        // Device-side consensus: CTAs spin on peers' rounds, so every CTA of the grid must be resident
        // at once on every rank.  Persistent grid (identical on every rank: same
        // N, same device model) launched cooperatively -- the launch fails instead of deadlocking if
        // the grid cannot be co-resident.
        if (per_sm < 1) return false;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)std::min(ngroups, g_sms_fz * per_sm));
        cfg.blockDim = dim3(Z::WARPS * 32);
        cfg.dynamicSmemBytes = SMEM;
        cfg.stream = L.stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, k, tmH, tmY, a) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        L.count(1);
        return true;
    }
    const int grid = (persist >> SOLVER) & 1 ? std::min(ngroups, g_sms_fz * std::max(per_sm, 1)) : ngroups;
    if (!launch_pdl(k, grid, Z::WARPS * 32, SMEM, L, tmH, tmY, a)) return false;
    L.count(1);
    return true;
}

// Shape gate of the fused path (the caller falls back to the split kernels).
bool fused_ok(int UP, int C, int N, int J, int S, int U) {
    if (UP > 16 || J != 1 || N <= 0 || C <= 0 || N > (1 << 30)) return false;
    const int PW = 32 / (UP / 4);
    if (C > 4 * PW) return false;
    return (U % 2 == 0) && (S % 2 == 0);
}

static void fz_shape(int UP, int C, FuArgs& a) {
    const int PW = 32 / (UP / 4);
    const int need = (C + PW - 1) / PW;
    a.WPS = need <= 1 ? 1 : need <= 2 ? 2 : 4;
    a.NPC = 4 / a.WPS;
}

bool launch_fused_ul(const LaunchCtx& L, int UP, bool cg, const float2* H, const float2* y, int C, int N, int S, int U,
                     int T, float rho, float gamma, Prox px, Modem md, float2* s_hat, uint8_t* hard, const XArgs* xc) {
    if (!fused_ok(UP, C, N, 1, S, U)) return false;
    FuArgs a{};
    if (xc) a.xc = *xc;
    a.S = S; a.U = U; a.N = N; a.C = C; a.T = T;
    a.rho = rho; a.gamma = gamma; a.delta = cg ? 0.f : rho;
    a.s_hat = s_hat; a.hard = hard; a.px = px; a.md = md; a.flag = L.flag;
    fz_shape(UP, C, a);
    switch (UP) {
        case 4: return cg ? launch_fz_t<4, 0>(L, H, y, a) : launch_fz_t<4, 1>(L, H, y, a);
        case 8: return cg ? launch_fz_t<8, 0>(L, H, y, a) : launch_fz_t<8, 1>(L, H, y, a);
        case 16: return cg ? launch_fz_t<16, 0>(L, H, y, a) : launch_fz_t<16, 1>(L, H, y, a);
        default: return false;
    }
}

bool launch_fused_dl(const LaunchCtx& L, int UP, const float2* Hd, const float2* s, int C, int C_glob, int N, int S,
                     int U, int T, float rho, float gamma, float a0, float eps, float2* x, const XArgs* xc) {
    if (!fused_ok(UP, C, N, 1, S, U)) return false;
    FuArgs a{};
    if (xc) a.xc = *xc;
    a.S = S; a.U = U; a.N = N; a.C = C; a.T = T;
    a.rho = rho; a.gamma = gamma; a.delta = 1.f / rho;
    a.s = s; a.x = x; a.rho_inv = 1.f / rho; a.a0 = a0; a.inv_c = 1.f / (float)C_glob; a.eps = eps; a.flag = L.flag;
    fz_shape(UP, C, a);
    switch (UP) {
        case 4: return launch_fz_t<4, 2>(L, Hd, nullptr, a);
        case 8: return launch_fz_t<8, 2>(L, Hd, nullptr, a);
        case 16: return launch_fz_t<16, 2>(L, Hd, nullptr, a);
        default: return false;
    }
}

// Centralized baselines (Table I rows MMSE-UL / ZF-DL): cluster-summed Gram + exact solve.
bool launch_fused_central(const LaunchCtx& L, int UP, bool dl, const float2* H, const float2* ys, int C, int N, int S,
                          int U, float reg, Modem md, float2* out, uint8_t* hard) {
    if (!fused_ok(UP, C, N, 1, S, U)) return false;
    FuArgs a{};
    a.S = S; a.U = U; a.N = N; a.C = C; a.T = 1;
    a.rho = reg; a.gamma = 1.f; a.delta = 0.f;
    a.md = md; a.flag = L.flag;
    if (dl) { a.s = ys; a.x = out; } else { a.s_hat = out; a.hard = hard; }
    fz_shape(UP, C, a);
    switch (UP) {
        case 4: return dl ? launch_fz_t<4, 4>(L, H, nullptr, a) : launch_fz_t<4, 3>(L, H, ys, a);
        case 8: return dl ? launch_fz_t<8, 4>(L, H, nullptr, a) : launch_fz_t<8, 3>(L, H, ys, a);
        case 16: return dl ? launch_fz_t<16, 4>(L, H, nullptr, a) : launch_fz_t<16, 3>(L, H, ys, a);
        default: return false;
    }
}

}  // namespace dbp
