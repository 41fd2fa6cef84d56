// dbp_kernels.cu -- small kernels of libdbp and their launchers.
//
// Kernel map (SURVEY.md 8(a) rows -> kernels):
//   k_fused    all rows         one launch per solver at world == 1 (dbp_fused.cu)
//   k_prefold  a1-a3 / b1 / c1  per-pair Gram + inverse, UP <= 16 (dbp_prefold.cu)
//   k_prelr    a1-a3 / b1 / c1  the same for UP = 32 or N_sym > 1 (dbp_prelr.cu)
//   k_admm_gj, k_admm_it, k_bf_gj, k_bf_it   iterations (dbp_iter.cu)
//   k_cg_gsum  b1 (sum)         per-GPU Gram sum G_loc = sum_c H_c^H H_c
//                               (Alg. 2 line 9 footnote, P416) + local y^MRC.
//   k_cg_it    b2-b5            replicated CG updates with shuffle allreduce
//                               dot products (P715), split or fused.
//   k_prox_out a7-a8            final prox + hard slicing of the split path.
//   k_slice                     stand-alone slicer (P210).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dbp_device.cuh"
#include "dbp_internal.h"

namespace dbp {

// Final prox + slicing of the split path: s_hat = prox(w^(T)).
template <int UP>
__global__ void k_prox_out(const float2* __restrict__ wbuf, int N, int J, int U, Prox px, Modem md,
                           float2* __restrict__ s_hat, uint8_t* __restrict__ hard) {
    const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long total = (long)N * J * U;
    if (e >= total) return;
    const long nj = e / U;
    const int uu = (int)(e % U);
    float2 s = prox(wbuf[nj * UP + uu], px);
    s_hat[e] = s;
    if (hard) hard[e] = slice_bits(s, md);
}

__global__ void k_slice(const float2* __restrict__ x, long count, Modem md, uint8_t* __restrict__ bits) {
    const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < count) bits[e] = slice_bits(x[e], md);
}

// ============================================================ CG-UL
// k_cg_gsum: G_loc[n] = sum_c Gp[c][n] and wbuf[n][j] = sum_c mf[c][n][j],
// clusters in fixed order c = 0..C_loc-1.
template <int UP>
__global__ void k_cg_gsum(const float2* __restrict__ Gp, const float2* __restrict__ mf, int C_loc, int N,
                          int J, float2* __restrict__ Gloc, float2* __restrict__ wbuf) {
    const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long ng = (long)N * tri(UP);
    const long nm = (long)N * J * UP;
    if (e < ng) {
        float2 acc = make_float2(0.f, 0.f);
        for (int c = 0; c < C_loc; ++c) acc = c_add(acc, Gp[(size_t)c * ng + e]);
        Gloc[e] = acc;
    } else if (e < ng + nm) {
        const long f = e - ng;
        float2 acc = make_float2(0.f, 0.f);
        for (int c = 0; c < C_loc; ++c) acc = c_add(acc, mf[(size_t)c * nm + f]);
        wbuf[f] = acc;
    }
}



// Split CG launch: finish the previous iteration from the allreduced w, then
// form the local w = G_loc p.  Fused (world == 1): all T iterations.
template <int UP, bool FUSED>
__global__ void k_cg_it(CgArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    DBP_POISON_SMEM(smem_raw);
    constexpr int GPB = 256 / UP;                      // (n, j) groups per CTA
    float2* Gs = reinterpret_cast<float2*>(smem_raw);  // [GPB][tri]
    float2* Ps = Gs + (size_t)GPB * tri(UP);           // [GPB][UP]
    const int tid = threadIdx.x;
    const int gi = tid / UP, u = tid % UP;
    const long g = (long)blockIdx.x * GPB + gi;        // (n, j) flat
    const bool valid = g < (long)a.N * a.J;
    const long n = valid ? g / a.J : 0;
    float2* G = Gs + (size_t)gi * tri(UP);
    float2* P = Ps + (size_t)gi * UP;
    for (int e = u; e < tri(UP); e += UP) G[e] = valid ? a.Gloc[n * tri(UP) + e] : make_float2(0.f, 0.f);
    const size_t o = (size_t)g * UP + u;

    float2 x, r, p;
    float rr;
    if (FUSED || a.step == 0) {                          // line 6: r = y^MRC, p = r, x = 0
        r = valid ? a.wbuf[o] : make_float2(0.f, 0.f);
        p = r;
        x = make_float2(0.f, 0.f);
        rr = group_sum<UP>(c_norm2(r));
    } else {
        x = valid ? a.x[o] : make_float2(0.f, 0.f);
        r = valid ? a.r[o] : make_float2(0.f, 0.f);
        p = valid ? a.p[o] : make_float2(0.f, 0.f);
        rr = valid ? a.rr[g] : 0.f;
        float2 w = valid ? a.wbuf[o] : make_float2(0.f, 0.f);
        cg_update<UP>(x, r, p, rr, w, a.rho);
    }
    const int iters = FUSED ? a.T : (a.step < a.T ? 1 : 0);
    for (int it = 0; it < iters; ++it) {
        DBP_SYNCWARP();
        P[u] = p;
        DBP_SYNCWARP();
        float2 w = herm_mv_row<UP>(G, P, u);               // lines 9-11, w = G p
        if (FUSED) cg_update<UP>(x, r, p, rr, w, a.rho);
        else if (valid) a.wbuf[o] = w;
    }
    if (!valid) return;
    if (!FUSED && a.step < a.T) {
        a.x[o] = x; a.r[o] = r; a.p[o] = p;
        if (u == 0) a.rr[g] = rr;
        return;
    }
    if (u < a.U) {
        const size_t oo = (size_t)g * a.U + u;
        a.x_hat[oo] = x;
        if (a.hard) a.hard[oo] = slice_bits(x, a.md);
    }
}

// ============================================================ launchers
static inline int cdiv(long a, long b) { return (int)((a + b - 1) / b); }


cudaError_t launch_prox_out(const LaunchCtx& L, int UP, const float2* wbuf, int N, int J, int U, Prox px,
                            Modem md, float2* s_hat, uint8_t* hard) {
    const long total = (long)N * J * U;
    DBP_DISPATCH_UP(UP, k_prox_out<UPc><<<cdiv(total, 256), 256, 0, L.stream>>>(wbuf, N, J, U, px, md, s_hat, hard));
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_slice(const LaunchCtx& L, const float2* x, long count, Modem md, uint8_t* bits) {
    if (count == 0) return cudaSuccess;
    k_slice<<<cdiv(count, 256), 256, 0, L.stream>>>(x, count, md, bits);
    L.count(1);
    return cudaGetLastError();
}

// --- CG-UL
cudaError_t launch_cg_gsum(const LaunchCtx& L, int UP, const float2* Gp, const float2* mf, int C_loc, int N,
                           int J, float2* Gloc, float2* wbuf) {
    const long total = (long)N * tri(UP) + (long)N * J * UP;
    DBP_DISPATCH_UP(UP, k_cg_gsum<UPc><<<cdiv(total, 256), 256, 0, L.stream>>>(Gp, mf, C_loc, N, J, Gloc, wbuf));
    L.count(1);
    return cudaGetLastError();
}

cudaError_t launch_cg_it(const LaunchCtx& L, int UP, bool fused, CgArgs a) {
    const int gpb = 256 / UP;
    const size_t smem = ((size_t)gpb * tri(UP) + (size_t)gpb * UP) * 8;
    const int grid = cdiv((long)a.N * a.J, gpb);
    DBP_DISPATCH_UP(UP,
        if (fused) {
            auto k = k_cg_it<UPc, true>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k<<<grid, 256, smem, L.stream>>>(a);
        } else {
            auto k = k_cg_it<UPc, false>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k<<<grid, 256, smem, L.stream>>>(a);
        });
    L.count(1);
    return cudaGetLastError();
}

}  // namespace dbp
