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
#include "dbp_fold.cuh"
#include "dbp_internal.h"

#pragma nv_diag_suppress 128   // MODE 0 returns before the inverse: "loop is not reachable"

namespace dbp {

template <int UP>
struct PF : Fold<UP> {
    static constexpr int WARPS = 4;
};

template <int UP, bool DL, int MODE>
struct PFL {
    using P = PF<UP>;
    using G = FoldStage<UP, DL, !DL && (MODE == 0 || MODE == 1)>;
    static constexpr int PLN = P::PW * P::PLP;                  // pivot lines (float2)
    static constexpr int WREG = (P::NST * G::STG + PLN * 8 + P::PW * UP * 4 + 127) / 128 * 128;
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
__global__ void __launch_bounds__(128, UP >= 32 ? 2 : 3)
k_prefold(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmY, PfArgs a) {
    using P = PF<UP>;
    using Q = PFL<UP, DL, MODE>;
    using G = typename Q::G;
    constexpr int L = P::L, PW = P::PW, SC = P::SC, NST = P::NST, R = P::R;
    // MODE 0 Gram + b, 1 inverse + y^reg, 2 inverse (DL), 4 Gram only (UL, N_sym > 1), 5 inverse only (UL)
    constexpr bool MF = !DL && (MODE == 0 || MODE == 1), INV = MODE == 1 || MODE == 2 || MODE == 5;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DBP_POISON_SMEM(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw) + warp * NST;
    unsigned char* wbase = smem_raw + 128 + (size_t)warp * Q::WREG;
    const int q = lane / L, l = lane % L;
    float2* pl = reinterpret_cast<float2*>(wbase + NST * G::STG) + q * P::PLP;      // pivot column + E_k
    float* dline = reinterpret_cast<float*>(wbase + NST * G::STG + Q::PLN * 8) + q * UP;   // Jacobi scales

    int row[R];
#pragma unroll
    for (int m = 0; m < R; ++m) row[m] = P::row(m, l);

    // (pair counts fit in int: launch_prefold takes npairs <= 2^30)
    const int ngroups = (int)((a.npairs + PW - 1) / PW);
    const int gw = blockIdx.x * P::WARPS + warp, W = gridDim.x * P::WARPS;
    const int nitems = gw < ngroups ? (ngroups - 1 - gw) / W + 1 : 0;
    const int nch = (a.S + SC - 1) / SC;
    const int nseq = nitems * nch;

    // TMA issue cursor (lane 0): the (item, chunk) of the next stage to load, advanced by one
    // per issue (stages are issued in sequence order, NST ahead of consumption)
    int is_item = 0, is_ch = 0;
    auto issue = [&](int st) {
        const int p0 = (gw + is_item * W) * PW;
        const int ch = is_ch;
        unsigned char* dst = wbase + st * G::STG;
        mbar_arrive_expect_tx(&bar[st], (uint32_t)G::BYTES);
        if (DL) {
            tma_load3(dst, &tmH, ch * SC, 0, p0, &bar[st]);
        } else {
            tma_load3(dst, &tmH, 0, ch * SC, p0, &bar[st]);
            if (MF) tma_load3(dst + G::HSZ * 8, &tmY, ch * SC, 0, p0, &bar[st]);
        }
        if (++is_ch == nch) { is_ch = 0; ++is_item; }
    };
    if (lane == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    DBP_SYNCWARP();
    if (lane == 0)
        for (int s = 0; s < NST && s < nseq; ++s) issue(s);

    int sq = 0, st = 0;
    uint32_t phase = 0;
    for (int it = 0; it < nitems; ++it) {
        const long p = (long)(gw + it * W) * PW + q;
        const bool valid = p < a.npairs;

        f2x A[P::NSLOT];
#pragma unroll
        for (int e = 0; e < P::NSLOT; ++e) A[e] = 0ull;
        f2x E[R];
#pragma unroll
        for (int m = 0; m < R; ++m) E[m] = 0ull;

        for (int ch = 0; ch < nch; ++ch) {
            mbar_wait(&bar[st], phase);
            const float2* stage = reinterpret_cast<const float2*>(wbase + st * G::STG);
#ifndef DBP_EXP_PF_NOGRAM
#define DBP_EXP_PF_NOGRAM 0     // experiment only: stream the stages without the Gram (wrong results)
#endif
            if (!DBP_EXP_PF_NOGRAM) {
                if (DL) fold_gram_dl<UP>(A, stage, q, row);
                else fold_gram_ul<UP, MF>(A, E, stage, q, row);
            }
            DBP_SYNCWARP();
            if (lane == 0 && sq + NST < nseq) {
                fence_proxy_async();
                issue(st);
            }
            ++sq;
            if (++st == NST) { st = 0; phase ^= 1u; }
        }
        float dg[R];
        fold_diag<UP>(A, row, a.delta, dg);
        if constexpr (!INV) {
            if (valid) {
                fold_store<UP>(a.Gout + (size_t)p * P::TRI, A, row);
                if (MF) {
#pragma unroll
                    for (int m = 0; m < R; ++m) a.vout[(size_t)p * UP + row[m]] = upk2(E[m]);
                }
            }
            continue;
        }
        float dr[R];
        fold_jacobi<UP, MODE == 1>(A, E, dg, dr, dline, row);
        const bool ok = fold_sweep<UP, MODE == 1>(A, E, pl, row, l);
        if (!ok && valid) atomicOr(a.flag, 1);
        fold_unscale<UP, MODE == 1>(A, E, dr, dline, 1.f);
        if (valid) {
            fold_store<UP>(a.Gout + (size_t)p * P::TRI, A, row);
            if (MODE == 1) {
#pragma unroll
                for (int m = 0; m < R; ++m) a.vout[(size_t)p * UP + row[m]] = upk2(E[m]);
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
        if ((MODE == 0 || MODE == 1) && !make_map3(&tmY, y, a.S, 1, a.npairs, P::SC, 1, P::PW)) return false;
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
        case 32: r = dl ? PFL<32, true, 2>::SMEM : PFL<32, false, 1>::SMEM; break;
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
    if (UP > 32 || (mode <= 1 && J != 1) || npairs <= 0 || npairs > (1L << 30)) return false;
    PfArgs a{S, U, npairs, delta, Gout, vout, L.flag};
    switch (UP) {
#define DBP_PF_CASE(UPc)                                                  \
    case UPc:                                                             \
        if (mode == 0) return launch_pf_t<UPc, false, 0>(L, H, y, a);     \
        if (mode == 1) return launch_pf_t<UPc, false, 1>(L, H, y, a);     \
        if (mode == 3) return launch_pf_t<UPc, true, 0>(L, H, y, a);      \
        if (mode == 4) return launch_pf_t<UPc, false, 4>(L, H, y, a);     \
        if (mode == 5) return launch_pf_t<UPc, false, 5>(L, H, y, a);     \
        return launch_pf_t<UPc, true, 2>(L, H, y, a);
        DBP_PF_CASE(4)
        DBP_PF_CASE(8)
        DBP_PF_CASE(16)
        DBP_PF_CASE(32)
#undef DBP_PF_CASE
        default: return false;
    }
}

}  // namespace dbp
