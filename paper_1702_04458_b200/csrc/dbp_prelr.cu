// dbp_prelr.cu -- k_prelr: per-pair preprocessing in the "lane = row" layout
// (SURVEY 8(a) rows a1-a3, b1, c1), fused with the inverse.
//
//   UL Gram   G_c = H_c^H H_c + delta I  (Alg. 1 line 7, delta = rho; Alg. 2
//             footnote P416, delta = 0), matched filter H_c^H y_c (line 8 /
//             Alg. 2 line 3).
//   DL Gram   B_c = H_c H_c^H + delta I  (Alg. 3 line 5, H_c = H^d_c, delta = 1/rho).
//   MODE 0    write G (packed lower) and H^H y          -> CG (k_cg_gsum)
//   MODE 1    Gauss-Jordan G^{-1}, y^reg = G^{-1} H^H y -> ADMM-UL iterations
//   MODE 2    Gauss-Jordan B^{-1}                        -> ADMM-DL iterations
//
// B200 design:
//  * UP lanes of one warp own one pair; lane i accumulates row i of the Gram,
//    G[i][j] = sum_s conj(h_si) h_sj for all j, from the antenna row h_s read
//    with UP/2 broadcast LDS.128 (all lanes of a pair read the same row).  No
//    split-K reduction, no per-job addressing: ~88% of the loop is FFMA, and
//    row i of G lands in lane i's registers -- exactly the layout the
//    Gauss-Jordan inverse (dbp_lanerow.cuh) and the iterations consume, so G
//    never round-trips through memory.
//  * Persistent CTAs of 128 threads; a stage is PPC = 128/UP consecutive pairs
//    brought in by one 1-D TMA bulk copy per pair (cp.async.bulk, SASS UBLKCP)
//    into slots padded by 16 B (the two pairs of a warp hit different banks),
//    in a 2-stage mbarrier ring.  A stage is released as soon as the Gram loop
//    has consumed it, so the next group's load overlaps the inverse.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dbp_device.cuh"
#include "dbp_internal.h"
#include "dbp_lanerow.cuh"

namespace dbp {

template <int UP>
struct LR {
    static constexpr int THREADS = 128;
    static constexpr int PPC = THREADS / UP;      // pairs per stage: 32, 16, 8, 4
    static constexpr int NST = 2;
};

__host__ __device__ inline int lr_ds(int S) { return ((S + 1) & ~1) + 2; }                 // DL padded row (even)
// per-pair H slot (float2): UL [S][U] + 16 B pad; DL [UP+1][ds(S)] (3-D TMA box, zero-filled padding)
__host__ __device__ inline int lr_hslot(int S, int U, int UP, bool dl) {
    return dl ? (UP + 1) * lr_ds(S) : ((S * U + 1) & ~1) + 2;
}
__host__ __device__ inline int lr_yslot(int S, int J) { return ((S * J + 1) & ~1) + 2; }

template <int UP>
static size_t lr_smem(int S, int U, int J, bool ul) {
    using C = LR<UP>;
    const size_t stage = ((size_t)C::PPC * (lr_hslot(S, U, UP, !ul) + (ul ? lr_yslot(S, J) : 0)) * 8 + 127) & ~(size_t)127;
    return 128 + C::NST * stage + (size_t)C::PPC * UP * 8;
}

struct LrArgs {
    const float2* H;      // UL [pairs][S][U], DL [pairs][U][S]
    const float2* y;      // UL [pairs][J][S]
    int S, U, J, tma;     // tma: DL tile by 3-D tensor map (else plain copy)
    long npairs;
    float delta;
    float2* Gout;         // [pairs][tri(UP)]: G (MODE 0) or G^{-1} (MODE 1, 2)
    float2* vout;         // MODE 0: H^H y [pairs][J][UP]; MODE 1: y^reg [pairs][J][UP]
    int* flag;
};

template <int UP, bool DL, int MODE, bool FULL>
__global__ void __launch_bounds__(128)
k_prelr(const __grid_constant__ CUtensorMap tmH, LrArgs a) {
    using C = LR<UP>;
    constexpr int PPC = C::PPC, NST = C::NST, TRI = tri(UP);
    constexpr bool UL = !DL;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    DBP_POISON_SMEM(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    int* done = reinterpret_cast<int*>(smem_raw + 32);
    const int S = a.S, U = a.U, J = a.J;
    const int hs = lr_hslot(S, U, UP, DL), ysl = UL ? lr_yslot(S, J) : 0;
    const int DS = lr_ds(S);
    const size_t stage_f2 = (((size_t)PPC * (hs + ysl) * 8 + 127) & ~(size_t)127) / 8;
    float2* stage0 = reinterpret_cast<float2*>(smem_raw + 128);   // TMA destinations: 128 B aligned
    float2* pline = stage0 + NST * stage_f2;                       // [PPC][UP] pivot / vector lines

    const int tid = threadIdx.x, lane = tid & 31;
    const int q = tid / UP, i = tid % UP;
    const long ngroups = (a.npairs + PPC - 1) / PPC;
    const long nitems = blockIdx.x < ngroups ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t hbytes = (uint32_t)(S * U * 8), ybytes = UL ? (uint32_t)(S * J * 8) : 0u;
    const bool bulk = DL ? (a.tma != 0) : (((hbytes | ybytes) & 15u) == 0);

    auto issue = [&](long item, int st) {
        const long p0 = (blockIdx.x + item * (long)gridDim.x) * PPC;
        const int nv = (int)min((long)PPC, a.npairs - p0);
        float2* hsl = stage0 + st * stage_f2;
        float2* ysm = hsl + (size_t)PPC * hs;
        if (DL) {                                   // one 3-D box {DS, UP+1, PPC}
            mbar_arrive_expect_tx(&full[st], (uint32_t)(PPC * hs * 8));
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                ::"r"(smem_u32(hsl)), "l"(reinterpret_cast<uint64_t>(&tmH)), "r"(0), "r"(0), "r"((int)p0),
                  "r"(smem_u32(&full[st])) : "memory");
            return;
        }
        mbar_arrive_expect_tx(&full[st], nv * (hbytes + ybytes));
        for (int k = 0; k < nv; ++k) {
            bulk_g2s(hsl + (size_t)k * hs, a.H + (size_t)(p0 + k) * S * U, hbytes, &full[st]);
            bulk_g2s(ysm + (size_t)k * ysl, a.y + (size_t)(p0 + k) * S * J, ybytes, &full[st]);
        }
    };
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); done[s] = 0; }
        fence_mbar_init();
    }
    DBP_SYNCTHREADS();
    if (bulk && tid == 0)
        for (int s = 0; s < NST && s < nitems; ++s) issue(s, s);

    for (long it = 0; it < nitems; ++it) {
        const int st = (int)(it % NST);
        const long p0 = (blockIdx.x + it * (long)gridDim.x) * PPC;
        const int nv = (int)min((long)PPC, a.npairs - p0);
        const float2* hsl = stage0 + st * stage_f2;
        const float2* ysm = hsl + (size_t)PPC * hs;
        if (bulk) {
            mbar_wait(&full[st], (uint32_t)((it / NST) & 1));
        } else {
            DBP_SYNCTHREADS();
            float2* hw = const_cast<float2*>(hsl);
            float2* yw = const_cast<float2*>(ysm);
            for (int k = 0; k < nv; ++k) {
                if (UL) {
                    for (int e = tid; e < S * U; e += C::THREADS) hw[(size_t)k * hs + e] = a.H[(size_t)(p0 + k) * S * U + e];
                    for (int e = tid; e < S * J; e += C::THREADS) yw[(size_t)k * ysl + e] = a.y[(size_t)(p0 + k) * S * J + e];
                } else {
                    for (int e = tid; e < hs; e += C::THREADS) {
                        const int u = e / DS, s = e % DS;
                        hw[(size_t)k * hs + e] = (u < U && s < S) ? a.H[((size_t)(p0 + k) * U + u) * S + s]
                                                                  : make_float2(0.f, 0.f);
                    }
                }
            }
            DBP_SYNCTHREADS();
        }
        const bool valid = q < nv;
        const long p = p0 + (valid ? q : 0);
        const float2* hb = hsl + (size_t)q * hs;
        const float2* yb = ysm + (size_t)q * ysl;

        // ---------------- Gram row i (and matched filter for N_sym = 1)
        float2 g[UP];
#pragma unroll
        for (int j = 0; j < UP; ++j) g[j] = make_float2(0.f, 0.f);
        float2 mf = make_float2(0.f, 0.f);
        if (UL) {
#pragma unroll 4
            for (int s = 0; s < S; ++s) {
                const float2* row = hb + s * U;
                float2 h[UP];
                if (FULL) {
                    read_vec<UP>(row, h);
                } else {
#pragma unroll
                    for (int j = 0; j < UP; ++j) h[j] = j < U ? row[j] : make_float2(0.f, 0.f);
                }
                const float2 own = (FULL || i < U) ? row[i] : make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < UP; ++j) c_fmac(g[j], own, h[j]);     // conj(h_si) h_sj
                if (MODE != 2 && J == 1) c_fmac(mf, own, yb[s]);
            }
        } else {
            // B[i][j] = sum_s H[i][s] conj(H[j][s]); rows of H^d are users, padded to DS
            // (even) antennas and UP+1 rows, zero-filled: LDS.128 = antennas (s, s+1)
#pragma unroll 2
            for (int s = 0; s < S; s += 2) {
                const float4 o = *reinterpret_cast<const float4*>(hb + i * DS + s);
                const float2 o0 = make_float2(o.x, o.y), o1 = make_float2(o.z, o.w);
#pragma unroll
                for (int j = 0; j < UP; ++j) {
                    const float4 v = *reinterpret_cast<const float4*>(hb + j * DS + s);
                    c_fmacb(g[j], o0, make_float2(v.x, v.y));
                    c_fmacb(g[j], o1, make_float2(v.z, v.w));
                }
            }
        }
        // N_sym > 1: the matched filters of all symbols, before the stage is released
        if (UL && MODE != 2 && J > 1) {
            for (int jj = 0; jj < J; ++jj) {
                float2 m = make_float2(0.f, 0.f);
                if (FULL || i < U)
                    for (int s = 0; s < S; ++s) c_fmac(m, hb[s * U + i], yb[jj * S + s]);
                if (valid) a.vout[((size_t)p * J + jj) * UP + i] = m;
            }
        }
        // stage consumed: release it (the last warp re-arms it for the group NST ahead)
        if (bulk) {
            DBP_SYNCWARP();
            if (lane == 0 && atomicAdd(&done[st], 1) == C::THREADS / 32 - 1) {
                done[st] = 0;
                if (it + NST < nitems) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(it + NST, st);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < UP; ++j)
            if (j == i) g[j] = make_float2(g[j].x + a.delta, 0.f);       // real diagonal + delta

        float2* line = pline + q * UP;
        if (MODE == 0) {
            if (valid) {
                store_herm_row<UP>(a.Gout + (size_t)p * TRI, i, g);
                if (UL && J == 1) a.vout[(size_t)p * UP + i] = mf;
            }
            continue;
        }
        const bool ok = gj_invert<UP>(g, line, i);
        if (!ok && valid) atomicOr(a.flag, 1);
        if (valid) store_herm_row<UP>(a.Gout + (size_t)p * TRI, i, g);
        if (MODE == 1) {
            for (int jj = 0; jj < J; ++jj) {
                const float2 m = J == 1 ? mf : a.vout[((size_t)p * J + jj) * UP + i];
                const float2 yr = row_apply<UP>(g, line, i, m);
                if (valid) a.vout[((size_t)p * J + jj) * UP + i] = yr;
            }
        }
    }
}

static int g_sms_lr = 0;

template <int UP, bool DL, int MODE>
static cudaError_t launch_lr_t(const LaunchCtx& L, LrArgs a) {
    using C = LR<UP>;
    if (!g_sms_lr) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms_lr, cudaDevAttrMultiProcessorCount, dev);
    }
    const size_t smem = lr_smem<UP>(a.S, a.U, a.J, !DL);
    const long ngroups = (a.npairs + C::PPC - 1) / C::PPC;
    CUtensorMap tm{};
    a.tma = 0;
    if (DL) a.tma = make_map3(&tm, a.H, a.S, a.U, a.npairs, lr_ds(a.S), UP + 1, C::PPC) ? 1 : 0;
    auto go = [&](auto k) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, C::THREADS, smem);
        const int grid = (int)std::min<long>(ngroups, (long)g_sms_lr * std::max(per_sm, 1));
        k<<<grid, C::THREADS, smem, L.stream>>>(tm, a);
    };
    if (a.U == UP) go(k_prelr<UP, DL, MODE, true>);
    else go(k_prelr<UP, DL, MODE, false>);
    L.count(1);
    return cudaGetLastError();
}

size_t prelr_smem(int UP, int S, int U, int J, bool ul) {
    size_t r = 0;
    DBP_DISPATCH_UP(UP, r = lr_smem<UPc>(S, U, J, ul));
    return r;
}

// N_sym > 1 companion of k_prefold modes 4 / 5: b_j = H_c^H y_cj for every symbol j (lane u of a
// UP-lane group takes column u of H_c), and with YREG y^reg_j = G^{-1} b_j (Alg. 1 line 8) by a
// lane-row mat-vec with row u of the packed inverse k_prefold wrote.
template <int UP, bool YREG>
__global__ void __launch_bounds__(256) k_mf_yreg(const float2* __restrict__ H, const float2* __restrict__ y,
                                                 const float2* __restrict__ Ginv, int S, int U, int J, long npairs,
                                                 float2* __restrict__ out) {
    __shared__ __align__(16) float2 sbuf[256 / UP][UP];
    const int g = threadIdx.x / UP, i = threadIdx.x % UP;
    const long p = (long)blockIdx.x * (256 / UP) + g;
    const bool valid = p < npairs;
    const long pp = valid ? p : npairs - 1;
    float2 R[UP];
    if (YREG) load_herm_row<UP>(Ginv + (size_t)pp * tri(UP), i, R);
    const float2* Hp = H + (size_t)pp * S * U;
    const float2* yp = y + (size_t)pp * J * S;
    constexpr int JB = 8;                         // symbols per pass: H_c is read once per JB symbols
    for (int j0 = 0; j0 < J; j0 += JB) {
        float2 b[JB];
#pragma unroll
        for (int k = 0; k < JB; ++k) b[k] = make_float2(0.f, 0.f);
        if (i < U) {
#pragma unroll 4
            for (int s = 0; s < S; ++s) {
                const float2 h = __ldg(Hp + (size_t)s * U + i);
#pragma unroll
                for (int k = 0; k < JB; ++k)
                    if (j0 + k < J) c_fmac(b[k], h, __ldg(yp + (size_t)(j0 + k) * S + s));
            }
        }
#pragma unroll
        for (int k = 0; k < JB; ++k) {
            if (j0 + k >= J) break;
            const float2 v = YREG ? row_apply<UP>(R, sbuf[g], i, b[k]) : b[k];
            if (valid) out[((size_t)p * J + j0 + k) * UP + i] = v;
        }
    }
}

// mode: 0 = Gram + H^H y (CG), 1 = inverse + y^reg (ADMM-UL), 2 = inverse (ADMM-DL, H = H^d),
//       3 = Gram only (ZF-DL, H = H^d)
cudaError_t launch_prelr(const LaunchCtx& L, int UP, int mode, const float2* H, const float2* y, int S, int U, int J,
                         long npairs, float delta, float2* Gout, float2* vout) {
    if (npairs <= 0) return cudaSuccess;
    if (launch_prefold(L, UP, mode, H, y, S, U, J, npairs, delta, Gout, vout)) return cudaGetLastError();
    if (J > 1 && (mode == 0 || mode == 1) &&
        launch_prefold(L, UP, mode == 0 ? 4 : 5, H, y, S, U, J, npairs, delta, Gout, vout)) {
        // N_sym > 1: folded Gram (+ sweep) without the matched filter, then b_j (+ y^reg_j) per symbol
        const int grid = (int)((npairs + 256 / UP - 1) / (256 / UP));
        DBP_DISPATCH_UP(UP,
            if (mode == 1) k_mf_yreg<UPc, true><<<grid, 256, 0, L.stream>>>(H, y, Gout, S, U, J, npairs, vout);
            else k_mf_yreg<UPc, false><<<grid, 256, 0, L.stream>>>(H, y, Gout, S, U, J, npairs, vout));
        L.count(1);
        return cudaGetLastError();
    }
    LrArgs a{H, y, S, U, J, 0, npairs, delta, Gout, vout, L.flag};
    cudaError_t e = cudaSuccess;
    DBP_DISPATCH_UP(UP,
        if (mode == 0) e = (launch_lr_t<UPc, false, 0>(L, a));
        else if (mode == 1) e = (launch_lr_t<UPc, false, 1>(L, a));
        else if (mode == 3) e = (launch_lr_t<UPc, true, 0>(L, a));
        else e = (launch_lr_t<UPc, true, 2>(L, a)));
    return e;
}

}  // namespace dbp
