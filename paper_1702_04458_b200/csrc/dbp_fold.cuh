// dbp_fold.cuh -- the "folded rows" per-pair layout shared by the
// preprocessing kernel k_prefold (dbp_prefold.cu) and the fused
// per-subcarrier solvers (dbp_fused.cu).  See dbp_prefold.cu for the design
// (DESIGN.md section 5.1).
//
// L = UP/4 lanes own one (cluster, subcarrier) pair; lane l holds R = 4 rows
// of the pair's Hermitian U x U matrix, r_m = l, 2L-1-l, 2L+l, 4L-1-l, and
// for row r_m the compile-time columns t < (m+1)L ("slots"; slot (m, t) is
// valid iff t <= r_m, the others are junk and never read).  A warp holds
// PW = 32/L pairs.
#pragma once

#include "dbp_device.cuh"
#include "dbp_lanerow.cuh"

// tuning knobs (build.py -D...): TMA ring depth, UL antenna-loop unroll,
// IEEE vs approximate pivot reciprocal, branch vs select pivot publication
#ifndef DBP_PF_NST
#define DBP_PF_NST 3
#endif
#ifndef DBP_PF_UNROLL
#define DBP_PF_UNROLL 2
#endif
#ifndef DBP_PF_RCPRN
#define DBP_PF_RCPRN 1
#endif

namespace dbp {

constexpr int PF_UNROLL = DBP_PF_UNROLL;

template <int UP>
struct Fold {
    static constexpr int R = 4;
    static constexpr int L = UP / R;                 // lanes per pair: 1, 2, 4
    static constexpr int PW = 32 / L;                // pairs per warp: 32, 16, 8
    static constexpr int SC = 4;                     // antennas per TMA stage
    static constexpr int NST = DBP_PF_NST;           // per-warp ring depth
    static constexpr int NSLOT = 10 * L;             // L * R(R+1)/2
    static constexpr int TRI = UP * (UP + 1) / 2;
    // pitch (float2) of a pair's pivot / vector line in shared memory: = L mod 16, so the
    // 16/L pairs of a 16-lane LDS.64 / STS.64 phase put their L-row blocks (rows mL..mL+L-1)
    // on disjoint banks; even (16-B aligned LDS.128 of c_t pairs) and >= UP + 2
    // (E_k and a dump entry follow the UP column entries)
    static constexpr int PLP = L >= 8 ? UP + 8 : (L >= 4 ? UP + 4 : UP + 2);
    __host__ __device__ static constexpr int off(int m) { return L * m * (m + 1) / 2; }
    __device__ static __forceinline__ int row(int m, int l) { return (m & 1) ? (m + 1) * L - 1 - l : m * L + l; }
};

// One warp's TMA box: UL {UP+2 users (2 out-of-bounds, zero-filled), SC
// antennas, PW pairs} + y {SC, PW}; DL {SC antennas, UP+1 users, PW pairs}.
template <int UP, bool DL, bool MF>
struct FoldStage {
    using F = Fold<UP>;
    static constexpr int HL = DL ? F::SC : UP + 2;              // smem line (float2)
    static constexpr int NL = DL ? UP + 1 : F::SC;              // lines per pair
    static constexpr int HSZ = F::PW * NL * HL;                 // float2
    static constexpr int YSZ = MF ? F::PW * F::SC : 0;
    static constexpr int BYTES = (HSZ + YSZ) * 8;               // complete_tx bytes
    static constexpr int STG = (BYTES + 127) / 128 * 128;       // stage pitch
};

// ---------------------------------------------------------------- Gram
// UL: G_rt += conj(h_sr) h_st (and b_r += conj(h_sr) y_s) over one stage.
// Pair q reads antenna (s + P[q/2]) mod 4 with P = {0, 2, 1, 3}: line (q, s) starts
// at 16-B unit 4(q & 1) + s_q (mod 8), so the 8 pairs' broadcast LDS.128 hit 8
// distinct bank groups, and within each half-warp the 4 pairs' own-row LDS.64
// (2 units per pair) start 2 units apart -- both conflict-free.
template <int UP, bool MF>
__device__ __forceinline__ void fold_gram_ul(f2x (&A)[Fold<UP>::NSLOT], f2x (&E)[4], const float2* stage, int q,
                                             const int (&row)[4]) {
    using F = Fold<UP>;
    using G = FoldStage<UP, false, MF>;
    const float2* hq = stage + q * G::NL * G::HL;
    const float2* yq = stage + G::HSZ + q * F::SC;
#pragma unroll PF_UNROLL
    for (int s = 0; s < F::SC; ++s) {
        const int sr = (s + ((((q >> 1) & 1) << 1) | ((q >> 2) & 1))) & (F::SC - 1);
        const float2* hrow = hq + sr * G::HL;
        float2 o[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) o[m] = hrow[row[m]];
#ifndef DBP_GRAM_TOUTER
#define DBP_GRAM_TOUTER 1
#endif
        if constexpr (DBP_GRAM_TOUTER && UP <= 16) {
            // t-outer: each broadcast pair (h_t, h_t+1) is live only across its slots.  Measured: fused
            // ADMM-UL 99.2 -> 97.4 us; at UP = 32 (k_prefold) the m-outer order is faster (959 vs 1036 us)
#pragma unroll
            for (int t2 = 0; t2 < UP; t2 += 2) {
                const float4 hh = *reinterpret_cast<const float4*>(hrow + t2);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    if (t2 < (m + 1) * F::L) x2_cmac(A[F::off(m) + t2], o[m], hh.x, hh.y);
                    if (t2 + 1 < (m + 1) * F::L) x2_cmac(A[F::off(m) + t2 + 1], o[m], hh.z, hh.w);
                }
            }
        } else {
            float2 h[UP];
            read_vec<UP>(hrow, h);
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int t = 0; t < (m + 1) * F::L; ++t) x2_cmac(A[F::off(m) + t], o[m], h[t].x, h[t].y);
        }
        if (MF) {
            const float2 yv = yq[sr];
#pragma unroll
            for (int m = 0; m < 4; ++m) x2_cmac(E[m], o[m], yv.x, yv.y);
        }
    }
}

// DL: B_rt += H_rs conj(H_ts); pair q reads antenna pair (s/2 + q) mod 2: line
// units 2q + 2t + c_q with c_q alternating between adjacent pairs, so the own-row
// LDS.128 of the two pairs sharing a quarter-warp phase never collide.
template <int UP>
__device__ __forceinline__ void fold_gram_dl(f2x (&A)[Fold<UP>::NSLOT], const float2* stage, int q, const int (&row)[4]) {
    using F = Fold<UP>;
    using G = FoldStage<UP, true, false>;
    const float2* hq = stage + q * G::NL * G::HL;
#pragma unroll 1
    for (int s0 = 0; s0 < F::SC; s0 += 2) {
        const int s = (s0 + 2 * (q & 1)) & (F::SC - 1);
        float4 o[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) o[m] = *reinterpret_cast<const float4*>(hq + row[m] * G::HL + s);
#pragma unroll
        for (int t = 0; t < UP; ++t) {
            const float4 v = *reinterpret_cast<const float4*>(hq + t * G::HL + s);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                if (t < (m + 1) * F::L) {
                    x2_macc(A[F::off(m) + t], make_float2(o[m].x, o[m].y), v.x, v.y);
                    x2_macc(A[F::off(m) + t], make_float2(o[m].z, o[m].w), v.z, v.w);
                }
            }
        }
    }
}

// Real diagonal + delta; dg[m] = diagonal of row r_m.  (Bit-mask predicates:
// a "t == row" compare chain gets folded into a dynamically indexed
// local-memory access by the compiler.)
template <int UP>
__device__ __forceinline__ void fold_diag(f2x (&A)[Fold<UP>::NSLOT], const int (&row)[4], float delta, float (&dg)[4]) {
    using F = Fold<UP>;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        dg[m] = 0.f;
        const unsigned dmask = 1u << row[m];
#pragma unroll
        for (int t = 0; t < (m + 1) * F::L; ++t) {
            const bool d = (dmask >> t) & 1u;
            float2 x = upk2(A[F::off(m) + t]);
            x.x = d ? x.x + delta : x.x;
            x.y = d ? 0.f : x.y;
            dg[m] += d ? x.x : 0.f;
            A[F::off(m) + t] = pk2(x);
        }
    }
}

// Jacobi scaling to unit diagonal: A_rt *= d_r d_t, E_r *= d_r (d = dg^-1/2,
// published to the pair's dline for the column factors).
template <int UP, bool BORDER>
__device__ __forceinline__ void fold_jacobi(f2x (&A)[Fold<UP>::NSLOT], f2x (&E)[4], const float (&dg)[4],
                                            float (&dr)[4], float* dline, const int (&row)[4]) {
    using F = Fold<UP>;
#pragma unroll
    for (int m = 0; m < 4; ++m) dr[m] = dg[m] > 0.f ? rsqrtf(dg[m]) : 1.f;
    DBP_SYNCWARP();
#pragma unroll
    for (int m = 0; m < 4; ++m) dline[row[m]] = dr[m];
    DBP_SYNCWARP();
#pragma unroll
    for (int m = 0; m < 4; ++m) {
#pragma unroll
        for (int t = 0; t < (m + 1) * F::L; ++t) A[F::off(m) + t] = pk2(c_scale(upk2(A[F::off(m) + t]), dr[m] * dline[t]));
        if (BORDER) E[m] = pk2(c_scale(upk2(E[m]), dr[m]));
    }
}

// Hermitian sweep over pivots k = 0..UP-1 (Goodnight form): afterwards the
// valid slots hold -M^{-1} of the (scaled) matrix and, with BORDER, E holds
// M^{-1} E.  pl: the pair's PLP line (pivot column, E_k, dump).  Returns false if
// a pivot was not positive and finite (not HPD).
template <int UP, bool BORDER>
__device__ __forceinline__ bool fold_sweep(f2x (&A)[Fold<UP>::NSLOT], f2x (&E)[4], float2* pl, const int (&row)[4],
                                           int l) {
    using F = Fold<UP>;
    constexpr int L = F::L;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < UP; ++k) {
        const int mk = k / L;
        const int lk = (mk & 1) ? (mk + 1) * L - 1 - k : k - mk * L;   // owner lane of row k
        DBP_SYNCWARP();
        // publish column k of the current matrix: c_j = a_jk (rows >= k from
        // every lane's slot k, rows < k as conj of the owner's row k)
        float2* const dump = pl + UP + 1;
#pragma unroll
        for (int m = 0; m < 4; ++m)
            if (k < (m + 1) * L) *(row[m] >= k ? pl + row[m] : dump) = upk2(A[F::off(m) + k]);
        if (l == lk) {
#pragma unroll
            for (int t = 0; t < k && t < (mk + 1) * L; ++t) pl[t] = c_conj(upk2(A[F::off(mk) + t]));
            if (BORDER) pl[UP] = upk2(E[mk]);
        }
        DBP_SYNCWARP();
        float2 cr[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) cr[m] = pl[row[m]];
        const float2 Ek = BORDER ? pl[UP] : make_float2(0.f, 0.f);
        const float piv = pl[k].x;
        const bool good = (piv > 0.f) && (piv < INFINITY);
        ok = ok && good;
        const float ip = good ? (DBP_PF_RCPRN ? __frcp_rn(piv) : rcp_approx(piv)) : 0.f;
        float2 f[4];
        bool me[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            // pivot row: a_kt / a_kk = a_kt - (1 - 1/a_kk) a_kt (no cancellation: a_kk <= 1)
            me[m] = row[m] == k;
            f[m] = me[m] ? make_float2(1.f - ip, 0.f) : c_scale(cr[m], ip);
            if (BORDER) x2_fms(E[m], f[m], Ek.x, Ek.y);    // E -= f E_k
        }
        // t-outer: each broadcast c_t (two per LDS.128) is live only across its R slots
#pragma unroll
        for (int t2 = 0; t2 < UP; t2 += 2) {
            const float4 cc = *reinterpret_cast<const float4*>(pl + t2);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = t2 + h;
                const float2 ct = h ? make_float2(cc.z, cc.w) : make_float2(cc.x, cc.y);
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    if (t >= (m + 1) * L) continue;
                    f2x& x = A[F::off(m) + t];
                    if (t == k) {
                        x = me[m] ? pk2(-ip, 0.f) : pk2(c_scale(upk2(x), ip));
                    } else {    // x -= f conj(c_t)
                        x2_fmsc(x, f[m], ct.x, ct.y);
                    }
                }
            }
        }
    }
    return ok;
}

// After fold_sweep on the Jacobi-scaled matrix: M^{-1}_rt = -d_r d_t A_rt,
// (M^{-1} b)_r = d_r E_r; `scale` multiplies the inverse (e.g. rho).
template <int UP, bool BORDER>
__device__ __forceinline__ void fold_unscale(f2x (&A)[Fold<UP>::NSLOT], f2x (&E)[4], const float (&dr)[4],
                                             const float* dline, float scale) {
    using F = Fold<UP>;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
#pragma unroll
        for (int t = 0; t < (m + 1) * F::L; ++t)
            A[F::off(m) + t] = pk2(c_scale(upk2(A[F::off(m) + t]), -scale * dr[m] * dline[t]));
        if (BORDER) E[m] = pk2(c_scale(upk2(E[m]), dr[m]));
    }
}

// fold_unscale followed by fold_mv_prep in one pass over the slots: the mat-vec form
// of scale * M^{-1} (junk slots 0, diagonal halved) and (M^{-1} b)_r = d_r E_r.
template <int UP, bool BORDER>
__device__ __forceinline__ void fold_unscale_mv(f2x (&A)[Fold<UP>::NSLOT], f2x (&E)[4], const float (&dr)[4],
                                                const float* dline, float scale, const int (&row)[4]) {
    using F = Fold<UP>;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const unsigned vmask = (2u << row[m]) - 1u, dmask = 1u << row[m];
        const float base = -scale * dr[m];
#pragma unroll
        for (int t = 0; t < (m + 1) * F::L; ++t) {
            const bool v = (vmask >> t) & 1u, d = (dmask >> t) & 1u;
            const float sc = v ? (d ? 0.5f * base : base) * dline[t] : 0.f;
            A[F::off(m) + t] = pk2(c_scale(upk2(A[F::off(m) + t]), sc));
        }
        if (BORDER) E[m] = pk2(c_scale(upk2(E[m]), dr[m]));
    }
}

// Packed lower-triangle store of the valid slots.
template <int UP>
__device__ __forceinline__ void fold_store(float2* G, const f2x (&A)[Fold<UP>::NSLOT], const int (&row)[4]) {
    using F = Fold<UP>;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        float2* Gr = G + (row[m] * (row[m] + 1)) / 2;
#pragma unroll
        for (int t = 0; t < (m + 1) * F::L; ++t)
            if (t <= row[m]) Gr[t] = upk2(A[F::off(m) + t]);
    }
}

// Per-pair stride of the mat-vec partial-sum block: L lanes x (UP + 2) float2.
// Lane stride 9 16-B units (= 1 mod 8), pair stride 36 units (= 4 mod 8 at UP = 16):
// the 8 lanes of each quarter-warp phase of an STS.128 hit 8 distinct bank groups.
template <int UP>
__host__ __device__ constexpr int fold_ybuf_pair() { return (UP / 4) * (UP + 2); }

// Mat-vec form of a Hermitian matrix in folded slots: junk slots zeroed and
// the diagonal halved, so y = M v is  y_r = sum_slots(r) S_rt v_t  +
// sum_lanes sum_slots(t, r) conj(S_tr) v_t  with no validity predicates.
template <int UP>
__device__ __forceinline__ void fold_mv_prep(f2x (&A)[Fold<UP>::NSLOT], const int (&row)[4]) {
    using F = Fold<UP>;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const unsigned vmask = (2u << row[m]) - 1u, dmask = 1u << row[m];
#pragma unroll
        for (int t = 0; t < (m + 1) * F::L; ++t) {
            const bool v = (vmask >> t) & 1u, d = (dmask >> t) & 1u;
            const float sc = v ? (d ? 0.5f : 1.f) : 0.f;
            A[F::off(m) + t] = pk2(c_scale(upk2(A[F::off(m) + t]), sc));
        }
    }
}

// y_{r_m} = (M v)_{r_m} for the pair's 4 rows per lane.  vline: the pair's
// UP-line; ybuf: the pair's L x YLS partial-sum block (fold_ybuf_pair() float2 per
// pair; the padded lane and pair strides put the 32 lanes of a warp on distinct
// 16-B bank groups).  Both in shared memory.
template <int UP>
__device__ __forceinline__ void fold_mv(const f2x (&A)[Fold<UP>::NSLOT], const float2 (&v)[4], float2 (&y)[4],
                                        float2* vline, float2* ybuf, const int (&row)[4], int l) {
    using F = Fold<UP>;
    DBP_SYNCWARP();
#pragma unroll
    for (int m = 0; m < 4; ++m) vline[row[m]] = v[m];
    DBP_SYNCWARP();
    f2x col[UP];
#pragma unroll
    for (int t = 0; t < UP; ++t) col[t] = 0ull;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        f2x acc = 0ull;
#pragma unroll
        for (int t2 = 0; t2 < (m + 1) * F::L; t2 += 2) {
            const float4 vv = *reinterpret_cast<const float4*>(vline + t2);
            const float2 s0 = upk2(A[F::off(m) + t2]);
            x2_mac(acc, s0, vv.x, vv.y);                   // y_r += S_rt v_t
            x2_cmac(col[t2], s0, v[m].x, v[m].y);          // y_t += conj(S_rt) v_r
            if (t2 + 1 < (m + 1) * F::L) {
                const float2 s1 = upk2(A[F::off(m) + t2 + 1]);
                x2_mac(acc, s1, vv.z, vv.w);
                x2_cmac(col[t2 + 1], s1, v[m].x, v[m].y);
            }
        }
        y[m] = upk2(acc);
    }
    constexpr int YLS = UP + 2;                            // lane stride (float2): +16 B per lane
    float4* yb = reinterpret_cast<float4*>(ybuf + l * YLS);
#pragma unroll
    for (int t2 = 0; t2 < UP; t2 += 2) {
        const float2 c0 = upk2(col[t2]), c1 = upk2(col[t2 + 1]);
        yb[t2 / 2] = make_float4(c0.x, c0.y, c1.x, c1.y);
    }
    DBP_SYNCWARP();
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int ll = 0; ll < F::L; ++ll) y[m] = c_add(y[m], ybuf[ll * YLS + row[m]]);
}

}  // namespace dbp
