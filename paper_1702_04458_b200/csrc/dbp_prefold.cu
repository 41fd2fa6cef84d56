// dbp_prefold.cu -- k_prefold: per-pair preprocessing in the "folded rows"
// layout for UP <= 16 and N_sym = 1.
//
//   UL Gram   G_c = H_c^H H_c + delta I  (Alg. 1 line 7, delta = rho; Alg. 2
//             footnote P416, delta = 0), matched filter b = H_c^H y_c (line 8 /
//             Alg. 2 line 3).
//   DL Gram   B_c = H_c H_c^H + delta I  (Alg. 3 line 5, H_c = H^d_c, delta = 1/rho).
//   MODE 0    write G (packed lower) and b                 -> CG (k_cg_gsum)
//   MODE 1    write G^{-1} and y^reg = G^{-1} b            -> ADMM-UL iterations
//   MODE 2    write B^{-1}                                 -> ADMM-DL iterations
//
// B200 design.  The work is FP32-FMA bound (a pair's
// 16 x 32 operand is too small for tensor-core tiles without 4-8x waste), so
// the layout minimises FMA-pipe work per pair:
//  * L = UP/4 lanes own one pair; lane l holds R = 4 rows of the Hermitian
//    matrix, r_m = l, 2L-1-l, 2L+l, 4L-1-l (m = 0..3), and for row r_m the
//    static columns t < (m+1)L (slot valid iff t <= r_m).  The four row
//    lengths of every lane sum to 2(UP+1): the lower triangle is covered with
//    85% slot efficiency (full rows: 50%), and every slot has a compile-time
//    column, so antenna row h_s reaches the FMAs by UP/2 broadcast LDS.128.
//  * The inverse is the Hermitian sweep operator (Goodnight 1979 form):
//    sweeping pivot k maps a_kk -> -1/a_kk, a_ik -> a_ik/a_kk,
//    a_ij -> a_ij - a_ik a_kj / a_kk, keeps the matrix Hermitian, so only the
//    lower slots are updated; after all UP pivots the block is -G^{-1}.  The
//    matched filter rides along as a border column (sweeping the bordered
//    matrix [[G, b], [b^H, 0]] leaves G^{-1} b in the border), so y^reg costs
//    R complex FMAs per pivot.  The matrix is Jacobi-scaled to unit diagonal
//    first: pivots are then Schur complements <= 1, which lets the pivot row
//    use the same update a - f conj(c_t) (f = 1 - 1/a_kk) without cancellation.
//  * Every warp is an independent persistent worker with its own 3-stage
//    mbarrier ring of 3-D TMA boxes (4 antennas x PW pairs per stage); there
//    is no CTA-level barrier.  Bank conflicts (UP = 16, 8 pairs per warp):
//    UL rows are padded to UP+2 users (zero-filled out-of-bounds box elements,
//    line pitch = 1 mod 8 16-B units) and pair q reads antenna (s + q/2) mod 4;
//    DL boxes are {4 antennas, UP+1 users} (pair pitch = 2 mod 8 units) and
//    pair q reads antenna pair (s/2 + q/4) mod 2.  Either way the 8 pairs'
//    LDS.128 addresses fall on 8 distinct bank groups.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_internal.h"
#include "dbp_lanerow.cuh"

// tuning knobs (build.py -D...): TMA ring depth, UL antenna-loop unroll
#ifndef DBP_PF_NST
#define DBP_PF_NST 3
#endif
#ifndef DBP_PF_UNROLL
#define DBP_PF_UNROLL 2
#endif
#ifndef DBP_PF_RCPRN
#define DBP_PF_RCPRN 1
#endif
#ifndef DBP_PF_PUB_BRANCH
#define DBP_PF_PUB_BRANCH 1
#endif
#pragma nv_diag_suppress 128   // MODE 0 returns before the inverse: "loop is not reachable"

namespace dbp {

constexpr int PF_UNROLL = DBP_PF_UNROLL;

template <int UP>
struct PF {
    static constexpr int R = 4;
    static constexpr int L = UP / R;                 // lanes per pair: 1, 2, 4
    static constexpr int PW = 32 / L;                // pairs per warp: 32, 16, 8
    static constexpr int SC = 4;                     // antennas per stage
    static constexpr int WARPS = 4;
    static constexpr int NST = DBP_PF_NST;
    static constexpr int NSLOT = 10 * L;             // L * R(R+1)/2
};

__host__ __device__ constexpr int pf_off(int m, int L) { return L * m * (m + 1) / 2; }

template <int UP, bool DL, int MODE>
struct PFL {
    using P = PF<UP>;
    static constexpr bool MF = !DL && MODE != 2;
    static constexpr int HL = DL ? P::SC : UP + 2;              // smem line (float2)
    static constexpr int NL = DL ? UP + 1 : P::SC;              // lines per pair
    static constexpr int HSZ = P::PW * NL * HL;                 // float2
    static constexpr int YSZ = MF ? P::PW * P::SC : 0;
    static constexpr int STG = ((HSZ + YSZ) * 8 + 127) / 128 * 128;   // bytes
    static constexpr int PLN = P::PW * (UP + 2);                // pivot lines (float2)
    static constexpr int WREG = (P::NST * STG + PLN * 8 + P::PW * UP * 4 + 127) / 128 * 128;
    static constexpr size_t SMEM = 128 + (size_t)P::WARPS * WREG;
};

struct PfArgs {
    int S, U;
    long npairs;
    float delta;
    float2* Gout;     // [pairs][tri(UP)]
    float2* vout;     // [pairs][UP] (MODE 0: b, MODE 1: y^reg)
    int* flag;
};

template <int UP, bool DL, int MODE>
__global__ void __launch_bounds__(128, 3)
k_prefold(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmY, PfArgs a) {
    using P = PF<UP>;
    using Q = PFL<UP, DL, MODE>;
    constexpr int L = P::L, PW = P::PW, SC = P::SC, NST = P::NST, R = P::R;
    constexpr int HL = Q::HL, NL = Q::NL, TRI = tri(UP);
    constexpr bool MF = Q::MF, INV = MODE != 0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw) + warp * NST;
    unsigned char* wbase = smem_raw + 128 + (size_t)warp * Q::WREG;
    const int q = lane / L, l = lane % L;
    float2* pl = reinterpret_cast<float2*>(wbase + NST * Q::STG) + q * (UP + 2);    // pivot column + E_k
    float* dline = reinterpret_cast<float*>(wbase + NST * Q::STG + Q::PLN * 8) + q * UP;   // Jacobi scales

    int row[R];
#pragma unroll
    for (int m = 0; m < R; ++m) row[m] = (m & 1) ? (m + 1) * L - 1 - l : m * L + l;

    // (pair counts fit in int: launch_prefold takes npairs <= 2^30)
    const int ngroups = (int)((a.npairs + PW - 1) / PW);
    const int gw = blockIdx.x * P::WARPS + warp, W = gridDim.x * P::WARPS;
    const int nitems = gw < ngroups ? (ngroups - 1 - gw) / W + 1 : 0;
    const int nch = (a.S + SC - 1) / SC;
    const int nseq = nitems * nch;

    // sequence number sq -> (item, chunk, stage); issued NST ahead of consumption
    auto issue = [&](int sq, int st) {
        const int item = sq / nch, ch = sq - item * nch;
        const int p0 = (gw + item * W) * PW;
        unsigned char* dst = wbase + st * Q::STG;
        mbar_arrive_expect_tx(&bar[st], (uint32_t)((Q::HSZ + Q::YSZ) * 8));
        if (DL) {
            tma_load3(dst, &tmH, ch * SC, 0, p0, &bar[st]);
        } else {
            tma_load3(dst, &tmH, 0, ch * SC, p0, &bar[st]);
            if (MF) tma_load3(dst + Q::HSZ * 8, &tmY, ch * SC, 0, p0, &bar[st]);
        }
    };
    if (lane == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0)
        for (int s = 0; s < NST && s < nseq; ++s) issue(s, s);

    int sq = 0, st = 0;
    uint32_t phase = 0;
    for (int it = 0; it < nitems; ++it) {
        const long p = (long)(gw + it * W) * PW + q;
        const bool valid = p < a.npairs;

        // ------------------------------------------------ Gram slots (+ matched filter)
        float2 A[P::NSLOT];
#pragma unroll
        for (int e = 0; e < P::NSLOT; ++e) A[e] = make_float2(0.f, 0.f);
        float2 E[R];
#pragma unroll
        for (int m = 0; m < R; ++m) E[m] = make_float2(0.f, 0.f);

        for (int ch = 0; ch < nch; ++ch) {
            mbar_wait(&bar[st], phase);
            const float2* hs = reinterpret_cast<const float2*>(wbase + st * Q::STG);
            if (!DL) {
                const float2* hq = hs + q * NL * HL;
                const float2* yq = hs + Q::HSZ + q * SC;
#pragma unroll PF_UNROLL
                for (int s = 0; s < SC; ++s) {
                    const int sr = (s + (q >> 1)) & (SC - 1);     // pair-rotated antenna: conflict-free LDS.128
                    const float2* hrow = hq + sr * HL;
                    float2 h[UP];
                    read_vec<UP>(hrow, h);
                    float2 o[R];
#pragma unroll
                    for (int m = 0; m < R; ++m) o[m] = hrow[row[m]];
#pragma unroll
                    for (int m = 0; m < R; ++m)
#pragma unroll
                        for (int t = 0; t < (m + 1) * L; ++t) c_fmac(A[pf_off(m, L) + t], o[m], h[t]);  // conj(h_sr) h_st
                    if (MF) {
                        const float2 yv = yq[sr];
#pragma unroll
                        for (int m = 0; m < R; ++m) c_fmac(E[m], o[m], yv);
                    }
                }
            } else {
                const float2* hq = hs + q * NL * HL;
#pragma unroll 1
                for (int s0 = 0; s0 < SC; s0 += 2) {
                    const int s = (s0 + 2 * (q >> 2)) & (SC - 1);       // pair-rotated antenna pair
                    float4 o[R];
#pragma unroll
                    for (int m = 0; m < R; ++m) o[m] = *reinterpret_cast<const float4*>(hq + row[m] * HL + s);
#pragma unroll
                    for (int t = 0; t < UP; ++t) {
                        const float4 v = *reinterpret_cast<const float4*>(hq + t * HL + s);
#pragma unroll
                        for (int m = 0; m < R; ++m) {
                            if (t < (m + 1) * L) {     // B_rt += H_rs conj(H_ts)
                                c_fmacb(A[pf_off(m, L) + t], make_float2(o[m].x, o[m].y), make_float2(v.x, v.y));
                                c_fmacb(A[pf_off(m, L) + t], make_float2(o[m].z, o[m].w), make_float2(v.z, v.w));
                            }
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0 && sq + NST < nseq) {
                fence_proxy_async();
                issue(sq + NST, st);
            }
            ++sq;
            if (++st == NST) { st = 0; phase ^= 1u; }
        }

        // diagonal: real, + delta
        // (bit-mask predicates: a "t == row" compare chain gets folded into a
        // dynamically indexed local-memory access by the compiler)
        float dg[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {
            dg[m] = 0.f;
            const unsigned dmask = 1u << row[m];
#pragma unroll
            for (int t = 0; t < (m + 1) * L; ++t) {
                const bool d = (dmask >> t) & 1u;
                float2& x = A[pf_off(m, L) + t];
                x.x = d ? x.x + a.delta : x.x;
                x.y = d ? 0.f : x.y;
                dg[m] += d ? x.x : 0.f;
            }
        }
        if constexpr (!INV) {
            if (valid) {
                float2* G = a.Gout + (size_t)p * TRI;
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    float2* Gr = G + (row[m] * (row[m] + 1)) / 2;
#pragma unroll
                    for (int t = 0; t < (m + 1) * L; ++t)
                        if (t <= row[m]) Gr[t] = A[pf_off(m, L) + t];
                    a.vout[(size_t)p * UP + row[m]] = E[m];
                }
            }
            continue;
        }

        // ------------------------------------------------ Jacobi scaling to unit diagonal
        float dr[R];
#pragma unroll
        for (int m = 0; m < R; ++m) dr[m] = dg[m] > 0.f ? rsqrtf(dg[m]) : 1.f;
        __syncwarp();
#pragma unroll
        for (int m = 0; m < R; ++m) dline[row[m]] = dr[m];
        __syncwarp();
#pragma unroll
        for (int m = 0; m < R; ++m) {
#pragma unroll
            for (int t = 0; t < (m + 1) * L; ++t)
                A[pf_off(m, L) + t] = c_scale(A[pf_off(m, L) + t], dr[m] * dline[t]);
            E[m] = c_scale(E[m], dr[m]);
        }

        // ------------------------------------------------ Hermitian sweep, pivots k = 0..UP-1
        bool ok = true;
#pragma unroll
        for (int k = 0; k < UP; ++k) {
            const int mk = k / L;
            const int lk = (mk & 1) ? (mk + 1) * L - 1 - k : k - mk * L;   // owner lane of row k
            __syncwarp();
            // publish column k of the current matrix: c_j = a_jk.  Stores are
            // unconditional with the address selected (pl[UP+1] is a dump slot),
            // so the sweep has no divergent branch and ptxas emits no
            // divergent-path copy of it around __syncwarp.
            float2* const dump = pl + UP + 1;
#pragma unroll
            for (int m = 0; m < R; ++m)
                if (k < (m + 1) * L) *(row[m] >= k ? pl + row[m] : dump) = A[pf_off(m, L) + k];
#if DBP_PF_PUB_BRANCH
            if (l == lk) {
#pragma unroll
                for (int t = 0; t < k && t < (mk + 1) * L; ++t) pl[t] = c_conj(A[pf_off(mk, L) + t]);
                if (MODE == 1) pl[UP] = E[mk];
            }
#else
            {
                const bool own = l == lk;
#pragma unroll
                for (int t = 0; t < k && t < (mk + 1) * L; ++t) *(own ? pl + t : dump) = c_conj(A[pf_off(mk, L) + t]);
                if (MODE == 1) *(own ? pl + UP : dump) = E[mk];
            }
#endif
            __syncwarp();
            float2 cr[R];
#pragma unroll
            for (int m = 0; m < R; ++m) cr[m] = pl[row[m]];
            const float2 Ek = MODE == 1 ? pl[UP] : make_float2(0.f, 0.f);
            const float piv = pl[k].x;
            const bool good = (piv > 0.f) && (piv < INFINITY);
            ok = ok && good;
            const float ip = good ? (DBP_PF_RCPRN ? __frcp_rn(piv) : rcp_approx(piv)) : 0.f;
            float2 f[R];
            bool me[R];
#pragma unroll
            for (int m = 0; m < R; ++m) {
                me[m] = row[m] == k;
                f[m] = me[m] ? make_float2(1.f - ip, 0.f) : c_scale(cr[m], ip);
                if (MODE == 1) {    // border: E -= f E_k
                    E[m].x = fmaf(-f[m].x, Ek.x, fmaf(f[m].y, Ek.y, E[m].x));
                    E[m].y = fmaf(-f[m].x, Ek.y, fmaf(-f[m].y, Ek.x, E[m].y));
                }
            }
            // t-outer so each broadcast c_t (two per LDS.128) is live only across its R slots
#pragma unroll
            for (int t2 = 0; t2 < UP; t2 += 2) {
                const float4 cc = *reinterpret_cast<const float4*>(pl + t2);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int t = t2 + h;
                    const float2 ct = h ? make_float2(cc.z, cc.w) : make_float2(cc.x, cc.y);
#pragma unroll
                    for (int m = 0; m < R; ++m) {
                        if (t >= (m + 1) * L) continue;
                        float2& x = A[pf_off(m, L) + t];
                        if (t == k) {
                            x = me[m] ? make_float2(-ip, 0.f) : c_scale(x, ip);
                        } else {    // x -= f conj(c_t)
                            x.x = fmaf(-f[m].x, ct.x, fmaf(-f[m].y, ct.y, x.x));
                            x.y = fmaf(-f[m].y, ct.x, fmaf(f[m].x, ct.y, x.y));
                        }
                    }
                }
            }
        }
        if (!ok && valid) atomicOr(a.flag, 1);

        // ------------------------------------------------ G^{-1} = -D (swept) D, y^reg = D (border)
        if (valid) {
            float2* G = a.Gout + (size_t)p * TRI;
#pragma unroll
            for (int m = 0; m < R; ++m) {
                float2* Gr = G + (row[m] * (row[m] + 1)) / 2;
#pragma unroll
                for (int t = 0; t < (m + 1) * L; ++t)
                    if (t <= row[m]) Gr[t] = c_scale(A[pf_off(m, L) + t], -dr[m] * dline[t]);
                if (MODE == 1) a.vout[(size_t)p * UP + row[m]] = c_scale(E[m], dr[m]);
            }
        }
    }
}

static int g_sms_pf = 0;

template <int UP, bool DL, int MODE>
static bool launch_pf_t(const LaunchCtx& L, const float2* H, const float2* y, PfArgs a) {
    using P = PF<UP>;
    using Q = PFL<UP, DL, MODE>;
    CUtensorMap tmH{}, tmY{};
    if (!DL) {
        if (!make_map3(&tmH, H, a.U, a.S, a.npairs, UP + 2, P::SC, P::PW)) return false;
        if (Q::MF && !make_map3(&tmY, y, a.S, 1, a.npairs, P::SC, 1, P::PW)) return false;
    } else {
        if (!make_map3(&tmH, H, a.S, a.U, a.npairs, P::SC, UP + 1, P::PW)) return false;
    }
    if (!g_sms_pf) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms_pf, cudaDevAttrMultiProcessorCount, dev);
    }
    auto k = k_prefold<UP, DL, MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Q::SMEM);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, P::WARPS * 32, Q::SMEM);
    const long ngroups = (a.npairs + P::PW - 1) / P::PW;
    const long nblk = (ngroups + P::WARPS - 1) / P::WARPS;
    const int grid = (int)std::min<long>(nblk, (long)g_sms_pf * std::max(per_sm, 1));
    k<<<grid, P::WARPS * 32, Q::SMEM, L.stream>>>(tmH, tmY, a);
    L.count(1);
    return true;
}

size_t prefold_smem(int UP, bool dl, int mode) {
    size_t r = 0;
    switch (UP) {
        case 4: r = dl ? PFL<4, true, 2>::SMEM : PFL<4, false, 1>::SMEM; break;
        case 8: r = dl ? PFL<8, true, 2>::SMEM : PFL<8, false, 1>::SMEM; break;
        case 16: r = dl ? PFL<16, true, 2>::SMEM : PFL<16, false, 1>::SMEM; break;
        default: r = 0;
    }
    (void)mode;
    return r;
}

// Returns true when launched; false when the shape is outside this kernel's
// domain (UP = 32, N_sym > 1, odd U / S for the TMA maps) -- the caller then
// uses the lane-row kernel (dbp_prelr.cu).
bool launch_prefold(const LaunchCtx& L, int UP, int mode, const float2* H, const float2* y, int S, int U, int J,
                    long npairs, float delta, float2* Gout, float2* vout) {
    if (UP > 16 || (mode != 2 && J != 1) || npairs <= 0 || npairs > (1L << 30)) return false;
    PfArgs a{S, U, npairs, delta, Gout, vout, L.flag};
    switch (UP) {
#define DBP_PF_CASE(UPc)                                                  \
    case UPc:                                                             \
        if (mode == 0) return launch_pf_t<UPc, false, 0>(L, H, y, a);     \
        if (mode == 1) return launch_pf_t<UPc, false, 1>(L, H, y, a);     \
        return launch_pf_t<UPc, true, 2>(L, H, y, a);
        DBP_PF_CASE(4)
        DBP_PF_CASE(8)
        DBP_PF_CASE(16)
#undef DBP_PF_CASE
        default: return false;
    }
}

}  // namespace dbp
