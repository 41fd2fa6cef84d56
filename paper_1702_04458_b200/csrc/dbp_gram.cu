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
//  * Persistent CTAs (256 threads, 2 per SM).  A stage is PPS whole pairs:
//    one 3-D TMA tensor load (cp.async.bulk.tensor.3d, SASS UTMALDG) of the
//    box {UP+2 users, S antennas, PPS pairs} (UL) or {S+2, UP+1, PPS} (DL).
//    Every pair's 4 KB channel block is read contiguously (DRAM-page
//    friendly).  The box is wider than the tensor: the out-of-bounds lanes
//    come back zero-filled, which pads every smem row by 16 B (bank-conflict
//    free reads) and zero-pads U up to UP for free.
//  * Stages form a ring (>= 2 deep) guarded by mbarriers; warps never meet at
//    a CTA barrier -- the last warp done with a stage re-arms it for the
//    group NST steps ahead.
//  * Each thread owns one 4x4 tile job of one pair and a 1/KS share of its
//    antenna rows (off-diagonal tiles and pairs of diagonal tiles cost the
//    same 64 FFMA per row; job types are warp-uniform).  The KS partial sums
//    meet by warp shuffles; results go straight to global memory.
//  * For N_sym = 1 the matched filter H_c^H y_c rides along; otherwise a
//    separate pass computes it.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_internal.h"

namespace dbp {

template <int UP, bool DL>
struct GW {
    static constexpr int TB = 4;                                 // 4x4 tile jobs
    static constexpr int NBK = UP / TB;                          // blocks: 1, 2, 4, 8
    static constexpr int NOFF = NBK * (NBK - 1) / 2;             // 0, 1, 6, 28
    static constexpr int NDIAG = NBK >= 2 ? NBK / 2 : 1;         // 1, 1, 2, 4
    static constexpr int JOBS = NOFF + NDIAG;                    // 1, 2, 8, 32
    static constexpr int THREADS = 256;
    static constexpr int KS = UP <= 8 ? 8 : UP == 16 ? 4 : 2;    // antenna (K) split
    static constexpr int PPS = THREADS / (JOBS * KS);            // pairs per stage: 32, 16, 8, 4
    static constexpr int OFF_T = PPS * NOFF * KS;
    static constexpr int UPJ = UP / JOBS;                        // matched-filter users per job
    static constexpr int ROWF = UP + 2;                          // UL smem row (float2), padded
    static_assert(PPS * JOBS * KS == THREADS, "one thread per (pair, job, k-part)");
    static_assert(OFF_T % 32 == 0, "job type is warp-uniform");
};

// smem floats2 per pair: UL [S][UP+2]; DL [UP+1][dlrow(S)]
__host__ __device__ inline int gw_dlrow(int S) { return ((S + 1) & ~1) + 2; }   // even: float4-aligned rows
template <int UP, bool DL>
__host__ __device__ inline int gw_pairf(int S) { return DL ? (UP + 1) * gw_dlrow(S) : S * (UP + 2); }

template <int UP, bool DL>
static void gw_stage(int S, int J, bool mf, size_t* hbytes, size_t* stage, int* nst) {
    using C = GW<UP, DL>;
    *hbytes = (size_t)C::PPS * gw_pairf<UP, DL>(S) * 8;
    const size_t yb = mf ? (size_t)C::PPS * J * S * 8 : 0;
    *stage = (*hbytes + yb + 127) & ~(size_t)127;
    int n = (int)std::min<size_t>(4, (110 * 1024) / *stage);
    *nst = std::max(n, 2);
}

template <int UP, bool DL>
static size_t gw_smem(int S, int J, bool mf) {
    size_t hb, st;
    int n;
    gw_stage<UP, DL>(S, J, mf, &hb, &st, &n);
    return 128 + n * st;
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
    float2* mfout;        // [pairs][J][UP] or null (N_sym == 1 only)
    int nst;
    uint32_t hbytes, ybytes, stage_bytes;
};

template <int KS, int N>
__device__ __forceinline__ void ksum(float2 (&acc)[N]) {
#pragma unroll
    for (int o = 1; o < KS; o <<= 1)
#pragma unroll
        for (int k = 0; k < N; ++k) {
            acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, o);
            acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, o);
        }
}

template <int UP, bool DL, bool MF, bool TMA, int SS>
__global__ void __launch_bounds__(256, 2)
k_gram(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmY, GramArgs a) {
    using C = GW<UP, DL>;
    constexpr int TB = C::TB, KS = C::KS, PPS = C::PPS, TRI = tri(UP), TS = TB * (TB - 1) / 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    int* done = reinterpret_cast<int*>(smem_raw + 64);
    unsigned char* stage0 = smem_raw + 128;
    const int J = a.J, S = SS > 0 ? SS : a.S, NST = a.nst;
    const int pairf = gw_pairf<UP, DL>(S);

    const int tid = threadIdx.x, lane = tid & 31;
    const long ngroups = (a.npairs + PPS - 1) / PPS;
    const long nitems = blockIdx.x < ngroups ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    auto issue = [&](long item, int st) {
        const long g = blockIdx.x + item * (long)gridDim.x;
        unsigned char* dst = stage0 + (size_t)st * a.stage_bytes;
        mbar_arrive_expect_tx(&full[st], a.hbytes + a.ybytes);
        tma_load_3d(dst, &tmH, 0, 0, (int)(g * PPS), &full[st]);
        if (MF) tma_load_3d(dst + a.hbytes, &tmY, 0, 0, (int)(g * PPS), &full[st]);
    };
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); done[s] = 0; }
        fence_mbar_init();
    }
    __syncthreads();
    if (TMA && tid == 0)
        for (int s = 0; s < NST && s < nitems; ++s) issue(s, s);

    // ---- this thread's job: (pair pi of the stage, tile, k-part h)
    const bool offj = tid < C::OFF_T;
    const int tj = offj ? tid : tid - C::OFF_T;
    const int slot = tj / KS, h = tj % KS;
    const int njob = offj ? C::NOFF : C::NDIAG;
    const int pi = slot / njob, jq = slot % njob;
    int ba = 0, bb = -1;
    if (offj) off_tile_coords(jq, ba, bb);
    else if (C::NBK >= 2) { ba = 2 * jq; bb = 2 * jq + 1; }
    const int u0 = (offj ? jq : C::NOFF + jq) * C::UPJ;     // matched-filter users of this job

    for (long it = 0; it < nitems; ++it) {
        const int st = (int)(it % NST);
        const long g = blockIdx.x + it * (long)gridDim.x;
        const float2* hs = reinterpret_cast<const float2*>(stage0 + (size_t)st * a.stage_bytes);
        const float2* ysm = reinterpret_cast<const float2*>(stage0 + (size_t)st * a.stage_bytes + a.hbytes);
        if (TMA) {
            mbar_wait(&full[st], (uint32_t)((it / NST) & 1));
        } else {
            __syncthreads();
            float2* hw = const_cast<float2*>(hs);
            float2* yw = const_cast<float2*>(ysm);
            for (int e = tid; e < PPS * pairf; e += C::THREADS) {
                const int p = e / pairf, q = e % pairf;
                const long gp = g * PPS + p;
                float2 v = make_float2(0.f, 0.f);
                if (!DL) {
                    const int s = q / (UP + 2), u = q % (UP + 2);
                    if (gp < a.npairs && u < a.U) v = a.H[((size_t)gp * S + s) * a.U + u];
                } else {
                    const int u = q / gw_dlrow(S), s = q % gw_dlrow(S);
                    if (gp < a.npairs && u < a.U && s < S) v = a.H[((size_t)gp * a.U + u) * S + s];
                }
                hw[e] = v;
            }
            if (MF)
                for (int e = tid; e < PPS * J * S; e += C::THREADS) {
                    const long gp = g * PPS + e / (J * S);
                    yw[e] = gp < a.npairs ? a.y[(size_t)g * PPS * J * S + e] : make_float2(0.f, 0.f);
                }
            __syncthreads();
        }
        const float2* hb = hs + (size_t)pi * pairf;
        const float2* yb = ysm + (size_t)pi * J * S;

        float2 acc[TB * TB];
#pragma unroll
        for (int k = 0; k < TB * TB; ++k) acc[k] = make_float2(0.f, 0.f);
        float2 mf[C::UPJ];
#pragma unroll
        for (int k = 0; k < C::UPJ; ++k) mf[k] = make_float2(0.f, 0.f);
#define DACC(q, i) (((i) & 1) ? acc[2 * TS + (q) * (TB / 2) + (i) / 2].y : acc[2 * TS + (q) * (TB / 2) + (i) / 2].x)

        if (!DL) {
            // G = H^H H over rows s = KS*t + h, visited in a per-pair rotated order
            const int RT = (S + KS - 1) / KS;
            const int rot = SS > 0 ? (pi & (RT - 1)) : (pi % RT);
#pragma unroll (SS > 0 ? 8 : 2)
            for (int t = 0; t < RT; ++t) {
                int tt = t + rot;
                tt = tt >= RT ? tt - RT : tt;
                const int s = KS * tt + h;
                if (SS == 0 && s >= S) continue;
                const float4* rowp = reinterpret_cast<const float4*>(hb + s * (UP + 2));
                float2 A[TB], B[TB];
                {
                    const float4 q0 = rowp[2 * ba], q1 = rowp[2 * ba + 1];
                    A[0] = make_float2(q0.x, q0.y); A[1] = make_float2(q0.z, q0.w);
                    A[2] = make_float2(q1.x, q1.y); A[3] = make_float2(q1.z, q1.w);
                }
                if (bb >= 0) {
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
                if (MF) {
                    const float2 ys = yb[s];
                    const float2* hu = hb + s * (UP + 2) + u0;
#pragma unroll
                    for (int k = 0; k < C::UPJ; ++k) c_fmac(mf[k], hu[k], ys);
                }
            }
        } else {
            // B = H H^H (H = U x S downlink block): s-pairs sp = KS*t + h, LDS.128 per user
            const int RT = (S + 2 * KS - 1) / (2 * KS);
#pragma unroll 2
            for (int t = 0; t < RT; ++t) {
                const int sp = KS * t + h;
                if (2 * sp >= S) continue;
                float2 A[TB][2], B[TB][2];
#pragma unroll
                for (int k = 0; k < TB; ++k) {
                    const float4 qa = *reinterpret_cast<const float4*>(hb + (TB * ba + k) * gw_dlrow(S) + 2 * sp);
                    A[k][0] = make_float2(qa.x, qa.y); A[k][1] = make_float2(qa.z, qa.w);
                    if (bb >= 0) {
                        const float4 qb = *reinterpret_cast<const float4*>(hb + (TB * bb + k) * gw_dlrow(S) + 2 * sp);
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
        }
        // release the stage (data is in registers now); the last warp re-arms it NST groups ahead
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
        ksum<KS>(acc);
        if (MF) ksum<KS>(mf);
        const long p = g * PPS + pi;
        if (p < a.npairs) {
            float2* G = a.Gout + (size_t)p * TRI;
            if (offj) {
#pragma unroll
                for (int k = 0; k < TB * TB; ++k)
                    if (k % KS == h) G[pidx(TB * ba + k / TB, TB * bb + k % TB)] = acc[k];
            } else {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int d = q ? bb : ba;
                    if (d < 0) continue;
#pragma unroll
                    for (int i = 0; i < TB; ++i) {
#pragma unroll
                        for (int j = 0; j < i; ++j)
                            if ((i * TB + j) % KS == h) G[pidx(TB * d + i, TB * d + j)] = acc[q * TS + i * (i - 1) / 2 + j];
                        if ((i * TB + i) % KS == h)
                            G[pidx(TB * d + i, TB * d + i)] = make_float2((q ? DACC(1, i) : DACC(0, i)) + a.delta, 0.f);
                    }
                }
            }
            if (MF && h == 0) {
#pragma unroll
                for (int k = 0; k < C::UPJ; ++k) a.mfout[(size_t)p * UP + u0 + k] = mf[k];
            }
        }
#undef DACC
    }
}

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

bool make_map3(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
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

bool make_map4(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint32_t b0,
               uint32_t b1, uint32_t b2, uint32_t b3) {
    auto fn = encode_fn();
    if (!fn) return false;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((d0 * 8) & 15)) return false;
    if (d2 > (1ull << 32) || d3 > (1ull << 32) || b0 > 256 || b1 > 256 || b2 > 256 || b3 > 256 || ((b0 * 8) & 15))
        return false;
    cuuint64_t dims[4] = {d0, d1, d2, d3};
    cuuint64_t strides[3] = {d0 * 8, d0 * d1 * 8, d0 * d1 * d2 * 8};
    cuuint32_t box[4] = {b0, b1, b2, b3};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static int g_sms = 0;

template <int UP, bool DL>
static cudaError_t launch_gram_t(const LaunchCtx& L, const float2* H, const float2* y, int S, int U, int J,
                                 long npairs, float delta, float2* Gout, float2* mfout) {
    using C = GW<UP, DL>;
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const bool mf_in = !DL && mfout && J == 1;
    CUtensorMap tmH{}, tmY{};
    bool tma;
    // UL box {UP+2 users, S rows, PPS pairs}: the 2 extra (out-of-bounds, zero-filled) users pad each smem row
    // DL box {S+2 antennas, UP+1 users, PPS pairs}: pads each user row and each pair
    if (!DL) tma = make_map3(&tmH, H, U, S, npairs, UP + 2, S, C::PPS);
    else tma = make_map3(&tmH, H, S, U, npairs, gw_dlrow(S), UP + 1, C::PPS);
    if (tma && mf_in) tma = make_map3(&tmY, y, S, J, npairs, S, J, C::PPS);
    size_t hb, stb;
    int nst;
    gw_stage<UP, DL>(S, J, mf_in, &hb, &stb, &nst);
    GramArgs a{H, y, S, U, J, npairs, delta, Gout, mf_in ? mfout : nullptr, nst, (uint32_t)hb,
               (uint32_t)(mf_in ? (size_t)C::PPS * J * S * 8 : 0), (uint32_t)stb};
    const size_t smem = 128 + nst * stb;
    const long ngroups = (npairs + C::PPS - 1) / C::PPS;
    auto go = [&](auto k) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, C::THREADS, smem);
        const int grid = (int)std::min<long>(ngroups, (long)g_sms * std::max(per_sm, 1));
        k<<<grid, C::THREADS, smem, L.stream>>>(tmH, tmY, a);
    };
    if (tma && S == 32) {
        if (mf_in) go(k_gram<UP, DL, true, true, 32>);
        else go(k_gram<UP, DL, false, true, 32>);
    } else if (tma) {
        if (mf_in) go(k_gram<UP, DL, true, true, 0>);
        else go(k_gram<UP, DL, false, true, 0>);
    } else {
        if (mf_in) go(k_gram<UP, DL, true, false, 0>);
        else go(k_gram<UP, DL, false, false, 0>);
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
    (void)U;
    size_t r = 0;
    DBP_DISPATCH_UP(UP, r = (mode == PRE_BF_ ? gw_smem<UPc, true>(S, J, false) : gw_smem<UPc, false>(S, J, J == 1)));
    return r;
}

cudaError_t launch_gram(const LaunchCtx& L, int UP, int mode, const float2* H, const float2* y, int S, int U, int J,
                        long npairs, float delta, float2* Gout, float2* mfout) {
    if (npairs <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    DBP_DISPATCH_UP(UP,
        if (mode == PRE_BF_) e = (launch_gram_t<UPc, true>(L, H, y, S, U, J, npairs, delta, Gout, nullptr));
        else e = (launch_gram_t<UPc, false>(L, H, y, S, U, J, npairs, delta, Gout, mfout)));
    return e;
}

}  // namespace dbp
