// dbp_lanerow.cuh -- "lane = row" building blocks shared by the preprocessing
// (dbp_prelr.cu) and iteration (dbp_iter.cu) kernels: UP lanes of one warp
// hold the UP rows of a pair's U x U operator in registers.
#pragma once

#include "dbp_device.cuh"

namespace dbp {

// Row i of the Hermitian G from its packed lower triangle (global, read-only).
template <int UP>
__device__ __forceinline__ void load_herm_row(const float2* __restrict__ Gp, int i, float2 (&r)[UP]) {
    const int base = (i * (i + 1)) / 2;
#pragma unroll
    for (int j = 0; j < UP; ++j) {
        if (j <= i) r[j] = __ldg(Gp + base + j);
        else { const float2 v = __ldg(Gp + (j * (j + 1)) / 2 + i); r[j] = make_float2(v.x, -v.y); }
    }
}

// Same, from a packed triangle staged in shared memory.
template <int UP>
__device__ __forceinline__ void load_herm_row_s(const float2* Gp, int i, float2 (&r)[UP]) {
    const int base = (i * (i + 1)) / 2;
#pragma unroll
    for (int j = 0; j < UP; ++j) {
        if (j <= i) r[j] = Gp[base + j];
        else { const float2 v = Gp[(j * (j + 1)) / 2 + i]; r[j] = make_float2(v.x, -v.y); }
    }
}

template <int UP>
__device__ __forceinline__ void store_herm_row(float2* __restrict__ Gp, int i, const float2 (&r)[UP]) {
    const int base = (i * (i + 1)) / 2;
#pragma unroll
    for (int j = 0; j < UP; ++j)
        if (j <= i) Gp[base + j] = r[j];
}

// Broadcast-read a UP-vector written by the pair's lanes into registers.
template <int UP>
__device__ __forceinline__ void read_vec(const float2* buf, float2 (&v)[UP]) {
    const float4* p = reinterpret_cast<const float4*>(buf);
#pragma unroll
    for (int k = 0; k < UP / 2; ++k) {
        const float4 q = p[k];
        v[2 * k] = make_float2(q.x, q.y);
        v[2 * k + 1] = make_float2(q.z, q.w);
    }
}

// In-place Gauss-Jordan inverse, lane i holds row i; prow = per-pair UP-line.
template <int UP>
__device__ __forceinline__ bool gj_invert(float2 (&r)[UP], float2* prow, int i) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < UP; ++k) {
        // lane k publishes its row (pivot row)
        if (i == k) {
            float4* p = reinterpret_cast<float4*>(prow);
#pragma unroll
            for (int q = 0; q < UP / 2; ++q) p[q] = make_float4(r[2 * q].x, r[2 * q].y, r[2 * q + 1].x, r[2 * q + 1].y);
        }
        DBP_SYNCWARP();
        float2 pr[UP];
        read_vec<UP>(prow, pr);
        // pivot (real and positive for HPD input), then one divergence-free
        // update for every lane:  r_j <- m r_j - fs pr_j (j != k),  r_k <- -fs,
        // with m = 0, fs = -1/piv on the pivot lane (row k <- row k / piv,
        // (k,k) <- 1/piv) and m = 1, fs = r_k/piv elsewhere (Jordan step).
        const float piv = pr[k].x;
        const bool good = (piv > 0.f) && (piv < INFINITY);
        ok = ok && good;
        const float ip = good ? __frcp_rn(piv) : 0.f;
        const bool me = (i == k);
        const float m = me ? 0.f : 1.f;
        const float2 fs = me ? make_float2(-ip, 0.f) : c_scale(r[k], ip);
#pragma unroll
        for (int j = 0; j < UP; ++j) {
            if (j == k) continue;
            r[j].x = fmaf(-fs.x, pr[j].x, fmaf(fs.y, pr[j].y, m * r[j].x));
            r[j].y = fmaf(-fs.x, pr[j].y, fmaf(-fs.y, pr[j].x, m * r[j].y));
        }
        r[k] = make_float2(-fs.x, -fs.y);
        DBP_SYNCWARP();
    }
    return ok;
}

// y = sum_j R[j] v_j with v published by the pair's lanes in buf (v_i from lane i).
template <int UP>
__device__ __forceinline__ float2 row_apply(const float2 (&R)[UP], float2* buf, int i, float2 vi) {
    buf[i] = vi;
    DBP_SYNCWARP();
    float2 v[UP];
    read_vec<UP>(buf, v);
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < UP; ++j) c_fma(acc, R[j], v[j]);
    DBP_SYNCWARP();
    return acc;
}

// Fixed-order sum over the CTA's clusters for each (subcarrier, user):
// W[nl][c][u] -> out[nl][u] (threads (nl, u) sum c = 0..C-1 in order).
__device__ __forceinline__ float2 cluster_sum(const float2* W, int C, int UP, int nl, int u) {
    float2 acc = make_float2(0.f, 0.f);
    const float2* p = W + (size_t)nl * C * UP + u;
    int c = 0;
    for (; c + 4 <= C; c += 4) {
        const float2 a0 = p[(c + 0) * UP], a1 = p[(c + 1) * UP], a2 = p[(c + 2) * UP], a3 = p[(c + 3) * UP];
        acc = c_add(c_add(c_add(c_add(acc, a0), a1), a2), a3);
    }
    for (; c < C; ++c) acc = c_add(acc, p[c * UP]);
    return acc;
}

}  // namespace dbp
