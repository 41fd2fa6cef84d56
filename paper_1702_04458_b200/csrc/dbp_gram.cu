// dbp_gram.cu -- k_gram: batched per-pair Hermitian Gram matrices and matched
// filters.
//
//   UL (Alg. 1 line 7 / Alg. 2 footnote P416):  G_c = H_c^H H_c + delta I,
//        H_c = S x U block of the uplink channel, plus mf_c = H_c^H y_c.
//   DL (Alg. 3 line 5):                         B_c = H_c H_c^H + delta I,
//        H_c = U x S downlink block H^d_c.
// Output: packed lower triangle (row-major, (i, j) at i(i+1)/2 + j) per pair.
//
// B200 design:
//  * One persistent CTA per SM (8 warps).  A CTA owns groups of PPC pairs and
//    streams each group's antenna rows in chunks of SC rows through a
//    4-stage shared-memory ring filled by 3-D TMA tensor loads
//    (cp.async.bulk.tensor.3d, SASS UTMALDG): box = {UP+2 users, SC rows,
//    PPC pairs}.  The box is wider than the tensor, so the two extra user
//    columns come back zero-filled: that pads every smem row by 16 B, which
//    makes the tile reads bank-conflict-free, and it also zero-pads U up to
//    the kernel's UP for free (the padding users then contribute nothing).
//  * Each thread owns one 8x8 tile job of one pair for the whole group:
//    either the off-diagonal block (a > b) or a pair of diagonal blocks
//    (lower halves, real diagonals) -- both 256 FFMA per antenna row with 8
//    LDS.128, so the job type is warp-uniform and the FMA pipe, not the LSU,
//    is the limit.  Rows are visited in a per-pair rotated order so that the
//    32 lanes of a warp spread evenly over the 8 bank groups.
//  * Warps never meet at a CTA barrier: each waits on the stage's mbarrier;
//    the last warp done with a stage re-arms it NST items ahead.
//  * For N_sym = 1 the matched filter H_c^H y_c rides along (8 extra CMACs
//    per row); otherwise a separate pass computes it.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_internal.h"

namespace dbp {

template <int UP, bool DL>
struct G8 {
    static constexpr int TB = 4;                                 // 4x4 tile jobs
    static constexpr int NBK = UP / TB;                          // blocks: 1, 2, 4, 8
    static constexpr int NOFF = NBK * (NBK - 1) / 2;             // 0, 1, 6, 28
    static constexpr int NDIAG = NBK >= 2 ? NBK / 2 : 1;         // 1, 1, 2, 4
    static constexpr int JOBS = NOFF + NDIAG;                    // 1, 2, 8, 32
    static constexpr int THREADS = 256;
    static constexpr int PPC = THREADS / JOBS;                   // 256, 128, 32, 8 pairs per group
    // antenna rows per chunk: UL keeps one stage near 25-41 KB; DL loads 2
    // adjacent antennas of a user with one LDS.128
    static constexpr int SC = DL ? 2 : (UP == 4 ? 2 : UP == 8 ? 2 : UP == 16 ? 4 : 8);
    static constexpr int OFF_T = PPC * NOFF;
    static constexpr int ROWF = DL ? SC : UP + 2;                // smem row length (float2)
    static constexpr int PAIRF = DL ? (UP + 1) * SC : SC * (UP + 2);
    // ring depth: ~100 KB of chunks in flight per CTA (2 CTAs per SM)
    static constexpr int STAGE_B = PPC * PAIRF * 8;
    static constexpr int NST = STAGE_B * 3 > 100000 ? 3 : (100000 / STAGE_B > 16 ? 16 : 100000 / STAGE_B);
    // row rotation per pair so a warp's lanes spread over the 8 bank groups
    static constexpr int ROTSH = UP == 4 ? 2 : UP == 8 ? 2 : UP == 16 ? 1 : 0;
    static_assert(OFF_T % 32 == 0, "job type is warp-uniform");
    static_assert(PPC <= 256, "TMA box dim");
};

template <int UP, bool DL>
static size_t gram8_smem(int J, bool mf) {
    using C = G8<UP, DL>;
    const size_t stage = (size_t)C::PPC * C::PAIRF * 8 + (mf ? (size_t)C::PPC * J * C::SC * 8 : 0);
    return 128 + C::NST * ((stage + 127) & ~(size_t)127);
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_cta() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct GramArgs {
    const float2* H;      // fallback path (no tensor map)
    const float2* y;
    int S, U, J;
    long npairs;
    float delta;
    float2* Gout;
    float2* mfout;        // [pairs][J][UP] or null
    int use_tma;
};

// One row of a block of TB users from the smem chunk.  UL: row-major
// [pair][row][UP+2]; DL: [pair][user][SC] (so a user's SC values are adjacent).
template <int TB, bool DL, int ROWF, int SC>
__device__ __forceinline__ void ld_block(const float2* base, int r, int u0, float2 (&v)[TB]) {
    if (!DL) {
        const float4* p = reinterpret_cast<const float4*>(base + r * ROWF + u0);
#pragma unroll
        for (int k = 0; k < TB / 2; ++k) {
            const float4 q = p[k];
            v[2 * k] = make_float2(q.x, q.y);
            v[2 * k + 1] = make_float2(q.z, q.w);
        }
    } else {
#pragma unroll
        for (int k = 0; k < TB; ++k) v[k] = base[(u0 + k) * SC + r];
    }
}

template <int UP, bool DL, bool MF, bool TMA>
__global__ void __launch_bounds__(256, 2)
k_gram8(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmY, GramArgs a) {
    using C = G8<UP, DL>;
    constexpr int TB = C::TB, SC = C::SC, PPC = C::PPC, NST = C::NST, TRI = tri(UP);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    int* done = reinterpret_cast<int*>(smem_raw + 64);
    const int J = a.J, S = a.S;
    const size_t hbytes = (size_t)PPC * C::PAIRF * 8;
    const size_t ybytes = MF ? (size_t)PPC * J * SC * 8 : 0;
    const size_t stage_bytes = (hbytes + ybytes + 127) & ~(size_t)127;
    unsigned char* stage0 = smem_raw + 128;

    const int tid = threadIdx.x, lane = tid & 31;
    const long ngroups = (a.npairs + PPC - 1) / PPC;
    const int nch = (S + SC - 1) / SC;
    const long my_groups = blockIdx.x < ngroups ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long nitems = my_groups * nch;

    auto issue = [&](long item, int st) {
        const long g = blockIdx.x + (item / nch) * (long)gridDim.x;
        const int c = (int)(item % nch);
        unsigned char* dst = stage0 + st * stage_bytes;
        mbar_arrive_expect_tx(&full[st], (uint32_t)(hbytes + ybytes));
        if (!DL) tma_load_3d(dst, &tmH, 0, c * SC, (int)(g * PPC), &full[st]);
        else tma_load_3d(dst, &tmH, c * SC, 0, (int)(g * PPC), &full[st]);
        if (MF) tma_load_3d(dst + hbytes, &tmY, c * SC, 0, (int)(g * PPC), &full[st]);
    };
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); done[s] = 0; }
        fence_mbar_init();
    }
    __syncthreads();
    if (TMA && tid == 0)
        for (int s = 0; s < NST && s < nitems; ++s) issue(s, s);

    // ---- this thread's job
    const bool offj = tid < C::OFF_T;
    const int tj = offj ? tid : tid - C::OFF_T;
    const int njob = offj ? C::NOFF : C::NDIAG;
    const int pi = tj / njob, jq = tj % njob;
    int ba = 0, bb = 0;
    if (offj) {
        off_tile_coords(jq, ba, bb);
    } else {
        ba = C::NBK >= 2 ? 2 * jq : 0;
        bb = C::NBK >= 2 ? 2 * jq + 1 : -1;
    }
    const bool mf_writer = offj ? (bb == 0) : (jq == 0);
    const int rot = (pi >> C::ROTSH) & (SC - 1);

    // Off-diagonal job: 16 complex entries; diagonal job: strict lower halves
    // of blocks ba, bb (6 + 6 complex) and their 8 real diagonals (4 float2).
    constexpr int TS = TB * (TB - 1) / 2;
    float2 acc[TB * TB];
    float2 mf[TB];
    auto zero = [&]() {
#pragma unroll
        for (int k = 0; k < TB * TB; ++k) acc[k] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < TB; ++k) mf[k] = make_float2(0.f, 0.f);
    };
#define DACC(q, i) (((i) & 1) ? acc[2 * TS + (q) * (TB / 2) + (i) / 2].y : acc[2 * TS + (q) * (TB / 2) + (i) / 2].x)
    zero();

    for (long it = 0; it < nitems; ++it) {
        const int st = (int)(it % NST);
        const long g = blockIdx.x + (it / nch) * (long)gridDim.x;
        const int c = (int)(it % nch);
        const float2* hs = reinterpret_cast<const float2*>(stage0 + st * stage_bytes);
        const float2* ysm = reinterpret_cast<const float2*>(stage0 + st * stage_bytes + hbytes);
        if (TMA) {
            mbar_wait(&full[st], (uint32_t)((it / NST) & 1));
        } else {
            // fallback: synchronous copy into the same padded layout (zeros outside)
            __syncthreads();
            float2* hw = const_cast<float2*>(hs);
            float2* yw = const_cast<float2*>(ysm);
            for (int e = tid; e < PPC * C::PAIRF; e += C::THREADS) {
                const int p = e / C::PAIRF, q = e % C::PAIRF;
                const long gp = g * PPC + p;
                float2 v = make_float2(0.f, 0.f);
                if (!DL) {
                    const int r = q / (UP + 2), u = q % (UP + 2), s = c * SC + r;
                    if (gp < a.npairs && u < a.U && s < S) v = a.H[((size_t)gp * S + s) * a.U + u];
                } else {
                    const int u = q / SC, r = q % SC, s = c * SC + r;
                    if (gp < a.npairs && u < a.U && s < S) v = a.H[((size_t)gp * a.U + u) * S + s];
                }
                hw[e] = v;
            }
            if (MF)
                for (int e = tid; e < PPC * J * SC; e += C::THREADS) {
                    const int p = e / (J * SC), j = (e / SC) % J, r = e % SC, s = c * SC + r;
                    const long gp = g * PPC + p;
                    yw[e] = (gp < a.npairs && s < S) ? a.y[((size_t)gp * J + j) * S + s] : make_float2(0.f, 0.f);
                }
            __syncthreads();
        }
        const float2* hb = hs + (size_t)pi * C::PAIRF;
        const float2* yb = ysm + (size_t)pi * J * SC;

        if (!DL) {
            // uplink: G = H^H H, rows of the chunk in a rotated order
#pragma unroll 4
            for (int t = 0; t < SC; ++t) {
                const int r = (t + rot) & (SC - 1);
                const float4* rowp = reinterpret_cast<const float4*>(hb + r * (UP + 2));
                float2 A[TB], B[TB];
                {
                    const float4 q0 = rowp[2 * ba], q1 = rowp[2 * ba + 1];
                    A[0] = make_float2(q0.x, q0.y); A[1] = make_float2(q0.z, q0.w);
                    A[2] = make_float2(q1.x, q1.y); A[3] = make_float2(q1.z, q1.w);
                }
                if (offj || C::NBK >= 2) {
                    const float4 q0 = rowp[2 * bb], q1 = rowp[2 * bb + 1];
                    B[0] = make_float2(q0.x, q0.y); B[1] = make_float2(q0.z, q0.w);
                    B[2] = make_float2(q1.x, q1.y); B[3] = make_float2(q1.z, q1.w);
                } else {
                    B[0] = B[1] = B[2] = B[3] = make_float2(0.f, 0.f);
                }
                if (offj) {
#pragma unroll
                    for (int i = 0; i < TB; ++i)
#pragma unroll
                        for (int j = 0; j < TB; ++j) c_fmac(acc[i * TB + j], A[i], B[j]);
                } else {
#pragma unroll
                    for (int i = 0; i < TB; ++i) {
#pragma unroll
                        for (int j = 0; j < i; ++j) {
                            c_fmac(acc[i * (i - 1) / 2 + j], A[i], A[j]);
                            c_fmac(acc[TS + i * (i - 1) / 2 + j], B[i], B[j]);
                        }
                        DACC(0, i) = fmaf(A[i].x, A[i].x, fmaf(A[i].y, A[i].y, DACC(0, i)));
                        DACC(1, i) = fmaf(B[i].x, B[i].x, fmaf(B[i].y, B[i].y, DACC(1, i)));
                    }
                }
                if (MF && J == 1) {
                    const float2 ys = yb[r];
#pragma unroll
                    for (int k = 0; k < TB; ++k) c_fmac(mf[k], A[k], ys);
                }
            }
        } else {
            // downlink: B = H H^H, each LDS.128 brings antennas (s, s+1) of one user
            float2 A[TB][2], B[TB][2];
#pragma unroll
            for (int k = 0; k < TB; ++k) {
                const float4 qa = reinterpret_cast<const float4*>(hb)[TB * ba + k];
                A[k][0] = make_float2(qa.x, qa.y); A[k][1] = make_float2(qa.z, qa.w);
                if (offj || C::NBK >= 2) {
                    const float4 qb = reinterpret_cast<const float4*>(hb)[TB * bb + k];
                    B[k][0] = make_float2(qb.x, qb.y); B[k][1] = make_float2(qb.z, qb.w);
                } else {
                    B[k][0] = B[k][1] = make_float2(0.f, 0.f);
                }
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (offj) {
#pragma unroll
                    for (int i = 0; i < TB; ++i)
#pragma unroll
                        for (int j = 0; j < TB; ++j) c_fmacb(acc[i * TB + j], A[i][r], B[j][r]);
                } else {
#pragma unroll
                    for (int i = 0; i < TB; ++i) {
#pragma unroll
                        for (int j = 0; j < i; ++j) {
                            c_fmacb(acc[i * (i - 1) / 2 + j], A[i][r], A[j][r]);
                            c_fmacb(acc[TS + i * (i - 1) / 2 + j], B[i][r], B[j][r]);
                        }
                        DACC(0, i) = fmaf(A[i][r].x, A[i][r].x, fmaf(A[i][r].y, A[i][r].y, DACC(0, i)));
                        DACC(1, i) = fmaf(B[i][r].x, B[i][r].x, fmaf(B[i][r].y, B[i][r].y, DACC(1, i)));
                    }
                }
            }
        }
        // release the stage; the last warp re-arms it NST items ahead
        if (TMA) {
            __syncwarp();
            if (lane == 0 && atomicAdd(&done[st], 1) == C::THREADS / 32 - 1) {
                done[st] = 0;
                if (it + NST < nitems) {
                    fence_proxy_async_cta();
                    issue(it + NST, st);
                }
            }
        }
        if (c == nch - 1) {                                      // group finished: write out
            const long p = g * PPC + pi;
            if (p < a.npairs) {
                float2* G = a.Gout + (size_t)p * TRI;
                int ba_ = ba, bb_ = bb;
                asm volatile("" : "+r"(ba_), "+r"(bb_));        // keep the 64 output offsets out of the loop
                const int ba = ba_, bb = bb_;
                if (offj) {
#pragma unroll
                    for (int i = 0; i < TB; ++i)
#pragma unroll
                        for (int j = 0; j < TB; ++j) G[pidx(TB * ba + i, TB * bb + j)] = acc[i * TB + j];
                } else {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int d = q ? bb : ba;
                        if (d < 0) continue;
#pragma unroll
                        for (int i = 0; i < TB; ++i) {
#pragma unroll
                            for (int j = 0; j < i; ++j) G[pidx(TB * d + i, TB * d + j)] = acc[q * TS + i * (i - 1) / 2 + j];
                            G[pidx(TB * d + i, TB * d + i)] = make_float2((q ? DACC(1, i) : DACC(0, i)) + a.delta, 0.f);
                        }
                    }
                }
                if (MF && J == 1 && mf_writer) {
                    float2* m = a.mfout + (size_t)p * UP + TB * ba;
#pragma unroll
                    for (int k = 0; k < TB; ++k) m[k] = mf[k];
                }
            }
            zero();
        }
    }
}

#undef DACC

// Matched filter for N_sym > 1 (separate pass): mf[p][j][u] = sum_s conj(H[p][s][u]) y[p][j][s].
__global__ void k_mf(const float2* __restrict__ H, const float2* __restrict__ y, int S, int U, int UP, int J,
                     long npairs, float2* __restrict__ mf) {
    const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= npairs * J * UP) return;
    const int u = (int)(e % UP);
    const long pj = e / UP;
    const long p = pj / J;
    float2 acc = make_float2(0.f, 0.f);
    if (u < U)
        for (int s = 0; s < S; ++s) c_fmac(acc, H[((size_t)p * S + s) * U + u], y[(size_t)pj * S + s]);
    mf[e] = acc;
}

// ------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

static bool make_map3(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
                      uint32_t b1, uint32_t b2) {
    auto fn = encode_fn();
    if (!fn) return false;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((d0 * 8) & 15)) return false;
    if (d2 > (1ull << 32) || b0 > 256 || b1 > 256 || b2 > 256 || ((b0 * 8) & 15)) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {d0 * 8, d0 * d1 * 8};
    cuuint32_t box[3] = {b0, b1, b2};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static int g_sms = 0;

template <int UP, bool DL>
static cudaError_t launch_gram8_t(const LaunchCtx& L, const float2* H, const float2* y, int S, int U, int J,
                                  long npairs, float delta, float2* Gout, float2* mfout) {
    using C = G8<UP, DL>;
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const bool mf_in = !DL && mfout && J == 1;
    CUtensorMap tmH{}, tmY{};
    bool tma = true;
    if (!DL) tma = make_map3(&tmH, H, U, S, npairs, UP + 2, C::SC, C::PPC);
    else tma = make_map3(&tmH, H, S, U, npairs, C::SC, UP + 1, C::PPC);
    if (tma && mf_in) tma = make_map3(&tmY, y, S, J, npairs, C::SC, J, C::PPC);
    GramArgs a{H, y, S, U, J, npairs, delta, Gout, mf_in ? mfout : nullptr, tma ? 1 : 0};
    const size_t smem = gram8_smem<UP, DL>(J, mf_in);
    const long ngroups = (npairs + C::PPC - 1) / C::PPC;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mf_in ? (tma ? (const void*)k_gram8<UP, DL, true, true> : (const void*)k_gram8<UP, DL, true, false>)
                                                                  : (tma ? (const void*)k_gram8<UP, DL, false, true> : (const void*)k_gram8<UP, DL, false, false>),
                                                  C::THREADS, smem);
    const int grid = (int)std::min<long>(ngroups, (long)g_sms * std::max(per_sm, 1));
    auto go = [&](auto k) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, C::THREADS, smem, L.stream>>>(tmH, tmY, a);
    };
    if (tma) {
        if (mf_in) go(k_gram8<UP, DL, true, true>);
        else go(k_gram8<UP, DL, false, true>);
    } else {
        if (mf_in) go(k_gram8<UP, DL, true, false>);
        else go(k_gram8<UP, DL, false, false>);
    }
    L.count(1);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && !DL && mfout && J > 1) {
        const long tot = npairs * J * UP;
        k_mf<<<(int)((tot + 255) / 256), 256, 0, L.stream>>>(H, y, S, U, UP, J, npairs, mfout);
        L.count(1);
        e = cudaGetLastError();
    }
    return e;
}

size_t pre_smem(int UP, int S, int U, int J, int mode) {
    (void)S; (void)U;
    size_t r = 0;
    DBP_DISPATCH_UP(UP, r = (mode == PRE_BF_ ? gram8_smem<UPc, true>(J, false) : gram8_smem<UPc, false>(J, J == 1)));
    return r;
}

cudaError_t launch_gram(const LaunchCtx& L, int UP, int mode, const float2* H, const float2* y, int S, int U, int J,
                        long npairs, float delta, float2* Gout, float2* mfout) {
    if (npairs <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    DBP_DISPATCH_UP(UP,
        if (mode == PRE_BF_) e = (launch_gram8_t<UPc, true>(L, H, y, S, U, J, npairs, delta, Gout, nullptr));
        else e = (launch_gram8_t<UPc, false>(L, H, y, S, U, J, npairs, delta, Gout, mfout)));
    return e;
}

}  // namespace dbp
