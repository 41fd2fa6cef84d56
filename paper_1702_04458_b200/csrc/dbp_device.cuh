// dbp_device.cuh -- device building blocks of libdbp (sm_100a).
//
// Complex arithmetic on float2, packed-triangular indexing, the TMA
// (cp.async.bulk / cp.async.bulk.tensor + mbarrier) helpers, the constellation
// slicer / proximal operators and the replicated CG update.
//
// A "pair" is one (cluster c, subcarrier n) of the paper's per-cluster,
// per-subcarrier local problem (P149-155, P706).  Inside a CTA a pair is
// served by a team of TPP consecutive threads of one warp; all teams of a
// warp run the same phase in lock-step, so __syncwarp() orders them.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dbp {

// ---------------------------------------------------------- debug: schedule fuzzing
// compute-sanitizer (racecheck / synccheck) is unavailable on the GPU pool, so a debug build
// (-DDBP_FUZZ=1, scripts/build_variants.py) stands in for it: every warp / CTA barrier is
// preceded and followed by a pseudo-random per-thread __nanosleep (0..511 ns) that reorders
// the threads' arrivals and subsequent shared-memory traffic, and every kernel first fills its
// dynamic shared memory with NaN, so a missing barrier or a read-before-write turns into a
// parity failure of the GPU tests (tests/test_gpu_parity.py run with DBP_LIB=<fuzz build>).
#ifndef DBP_FUZZ
#define DBP_FUZZ 0
#endif
__device__ __forceinline__ void dbp_fuzz_sleep() {
#if DBP_FUZZ
    unsigned x = (unsigned)clock() ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 40503u);
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    __nanosleep(x & 511u);
#endif
}
#define DBP_SYNCWARP() do { ::dbp::dbp_fuzz_sleep(); __syncwarp(); ::dbp::dbp_fuzz_sleep(); } while (0)
#define DBP_SYNCTHREADS() do { ::dbp::dbp_fuzz_sleep(); __syncthreads(); ::dbp::dbp_fuzz_sleep(); } while (0)
#if DBP_FUZZ
#define DBP_POISON_SMEM(base)                                                                   \
    do {                                                                                        \
        unsigned nb_;                                                                           \
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(nb_));                          \
        unsigned* w_ = reinterpret_cast<unsigned*>(base);                                       \
        for (unsigned i_ = threadIdx.x; i_ < nb_ / 4; i_ += blockDim.x) w_[i_] = 0x7fc00001u;   \
        __syncthreads();                                                                        \
    } while (0)
#else
#define DBP_POISON_SMEM(base) do { } while (0)
#endif

// ----------------------------------------------------------------- complex
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 c_scale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 c_conj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 c_mul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// acc += a * b
__device__ __forceinline__ void c_fma(float2& acc, float2 a, float2 b) {
    acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(-a.y, b.y, acc.x);
    acc.y = fmaf(a.x, b.y, acc.y); acc.y = fmaf(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void c_fmac(float2& acc, float2 a, float2 b) {
    acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(a.y, b.y, acc.x);
    acc.y = fmaf(a.x, b.y, acc.y); acc.y = fmaf(-a.y, b.x, acc.y);
}
// acc += a * conj(b)
__device__ __forceinline__ void c_fmacb(float2& acc, float2 a, float2 b) {
    acc.x = fmaf(a.x, b.x, acc.x); acc.x = fmaf(a.y, b.y, acc.x);
    acc.y = fmaf(a.y, b.x, acc.y); acc.y = fmaf(-a.x, b.y, acc.y);
}
__device__ __forceinline__ float c_norm2(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }

// ---- packed f32x2 complex MACs (sm_100 FFMA2: two FP32 FMAs per instruction).
// A complex value is one 64-bit register pair (re, im).  In every helper the
// reused operand `a` / `f` is the FIRST source, so ptxas expresses the sign
// and swap patterns as operand modifiers of that natural pair (.NP negates the
// high half, .LO_HI swaps) and the per-call values become scalar broadcasts
// (.F32): each complex MAC is exactly 2 FFMA2 with no pair construction
// (checked in SASS; the reverse operand order costs a MOV per use).
typedef unsigned long long f2x;
__device__ __forceinline__ f2x pk2(float x, float y) {
    f2x r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ f2x pk2(float2 v) { return pk2(v.x, v.y); }
__device__ __forceinline__ float2 upk2(f2x r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ f2x ffma2(f2x a, f2x b, f2x c) {
    f2x d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// acc += a b          = b.x a + (-b.y) (a.y, -a.x)
__device__ __forceinline__ void x2_mac(f2x& acc, float2 a, float bx, float by) {
    acc = ffma2(pk2(a.x, a.y), pk2(bx, bx), acc);
    acc = ffma2(pk2(a.y, -a.x), pk2(-by, -by), acc);
}
// acc += conj(a) b    = b.x (a.x, -a.y) + b.y (a.y, a.x)
__device__ __forceinline__ void x2_cmac(f2x& acc, float2 a, float bx, float by) {
    acc = ffma2(pk2(a.x, -a.y), pk2(bx, bx), acc);
    acc = ffma2(pk2(a.y, a.x), pk2(by, by), acc);
}
// acc += a conj(b)    = b.x a + b.y (a.y, -a.x)
__device__ __forceinline__ void x2_macc(f2x& acc, float2 a, float bx, float by) {
    acc = ffma2(pk2(a.x, a.y), pk2(bx, bx), acc);
    acc = ffma2(pk2(a.y, -a.x), pk2(by, by), acc);
}
// x -= f conj(c)      = (-c.x) f + (-c.y) (f.y, -f.x)
__device__ __forceinline__ void x2_fmsc(f2x& x, float2 f, float cx, float cy) {
    x = ffma2(pk2(f.x, f.y), pk2(-cx, -cx), x);
    x = ffma2(pk2(f.y, -f.x), pk2(-cy, -cy), x);
}
// x -= f e            = (-e.x) f + e.y (f.y, -f.x)
__device__ __forceinline__ void x2_fms(f2x& x, float2 f, float ex, float ey) {
    x = ffma2(pk2(f.x, f.y), pk2(-ex, -ex), x);
    x = ffma2(pk2(f.y, -f.x), pk2(ey, ey), x);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Packed lower-triangular storage, row-major: (i, j), j <= i.
__host__ __device__ constexpr int tri(int n) { return n * (n + 1) / 2; }
__host__ __device__ __forceinline__ int pidx(int i, int j) { return (i * (i + 1)) / 2 + j; }

// ------------------------------------------------------- TMA bulk copies
// 1-D bulk tensor copy global -> shared, completion tracked by an mbarrier
// (cp.async.bulk ... mbarrier::complete_tx::bytes; SASS UBLKCP).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// 3-D tiled tensor copy (box defined by the CUtensorMap; out-of-bounds elements zero-filled).
__device__ __forceinline__ void tma_load3(void* dst, const void* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load4(void* dst, const void* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
          "r"(smem_u32(bar))
        : "memory");
}
// Cross-GPU consensus words (peer memory over NVLink), NCCL-LL style: a complex value travels
// as two 8-byte words {re, id} {im, id}; 8-byte stores are single-copy atomic, so a reader that
// sees both ids equal to the round id it waits for has that round's value.
__device__ __forceinline__ void st_ll_sys(uint4* p, float2 v, unsigned id) {
    asm volatile("st.relaxed.sys.global.v4.u32 [%0], {%1, %2, %3, %4};"
                 ::"l"(p), "r"(__float_as_uint(v.x)), "r"(id), "r"(__float_as_uint(v.y)), "r"(id) : "memory");
}
// Bounded wait: polls until both ids equal `id`; after DBP_XC_TIMEOUT_NS of %globaltimer (or as
// soon as another thread of this GPU has timed out) it sets bit DBP_FLAG_XC_TIMEOUT of `flag`
// and returns 0 -- a protocol or launch fault on any rank becomes DBP_ERR_CUDA from dbp_sync,
// never a hung GPU.
#ifndef DBP_XC_TIMEOUT_NS
#define DBP_XC_TIMEOUT_NS 4000000000ull
#endif
constexpr int DBP_FLAG_XC_TIMEOUT = 2;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ float2 ld_ll_sys(const uint4* p, unsigned id, int* flag) {
    unsigned a, b, c, d;
    unsigned long long t0 = 0;
    for (unsigned k = 0;; ++k) {
        asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p) : "memory");
        if (b == id && d == id) break;
        if ((k & 255u) == 0u) {
            const unsigned long long now = globaltimer_ns();
            if (k == 0u) t0 = now;
            if (now - t0 > DBP_XC_TIMEOUT_NS || (*(volatile int*)flag & DBP_FLAG_XC_TIMEOUT)) {
                atomicOr(flag, DBP_FLAG_XC_TIMEOUT);
                return make_float2(0.f, 0.f);
            }
        }
    }
    return make_float2(__uint_as_float(a), __uint_as_float(c));
}
// 16-B asynchronous global -> shared copies (LDGSTS), completed by cp_async_wait_all.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Programmatic dependent launch (DBP_OPT_OVERLAP_PREV).  griddep_launch: this CTA lets the next
// kernel on the stream start (it launches once every CTA of this grid has issued it or exited).
// griddep_wait: block until the kernel before this one on the stream has completed and its memory
// is visible -- issued before a solver's first global store, so outputs stay in stream order.
// Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------ constellation
// Gray QAM with Es = 1 (reading 17): per-axis levels
// (2k - (m-1)) / sqrt(norm).  The decision is taken in fp32 with explicit
// round-to-nearest ops (no fma contraction), reading 19:
// k = clamp(ceil((x*scale + m)/2) - 1, 0, m-1), ties toward the negative level.
struct Modem { int m; int bpa; int naxes; float scale; float radius; };

__host__ __device__ inline Modem modem_of(int mod) {
    switch (mod) {
        case 1: return {2, 1, 1, 1.0f, 1.0f};
        case 2: return {2, 1, 2, 1.41421356f, 0.70710678f};
        case 4: return {4, 2, 2, 3.16227766f, 0.94868330f};
        default: return {8, 3, 2, 6.48074070f, 1.08012345f};
    }
}

__device__ __forceinline__ unsigned slice_axis(float x, const Modem& md) {
    float t = __fmul_rn(x, md.scale);
    float u = __fmul_rn(__fadd_rn(t, (float)md.m), 0.5f);
    float k = ceilf(u) - 1.0f;
    if (!(k >= 0.0f)) return 0u;
    if (k > (float)(md.m - 1)) return (unsigned)(md.m - 1);
    return (unsigned)k;
}
__device__ __forceinline__ uint8_t slice_bits(float2 v, const Modem& md) {
    unsigned ki = slice_axis(v.x, md);
    unsigned gi = ki ^ (ki >> 1);
    if (md.naxes == 1) return (uint8_t)gi;
    unsigned kq = slice_axis(v.y, md);
    unsigned gq = kq ^ (kq >> 1);
    return (uint8_t)((gi << md.bpa) | gq);
}

// Proximal step (E2) applied to the consensus sum w (Lemma 1, P325-344):
// MMSE: s = w / (N0/(rho Es) + C)  (Alg. 1 line 13), ZF: w / C,
// BOX: per-axis clamp of w / C to [-r, r], BPSK: real clamp, imag 0.
struct Prox { int reg; float inv_c; float mmse_scale; float r; int bpsk; };
__device__ __forceinline__ float2 prox(float2 w, const Prox& p) {
    if (p.reg == 0) return c_scale(w, p.mmse_scale);
    float2 v = c_scale(w, p.inv_c);
    if (p.reg == 1) return v;
    v.x = fminf(fmaxf(v.x, -p.r), p.r);
    v.y = p.bpsk ? 0.0f : fminf(fmaxf(v.y, -p.r), p.r);
    return v;
}

// --------------------------------------------------- per-pair dense algebra
// Hermitian mat-vec with a packed lower Hermitian matrix G (row r of G v).
template <int UP>
__device__ __forceinline__ float2 herm_mv_row(const float2* G, const float2* v, int r) {
    float2 acc = make_float2(0.f, 0.f);
    for (int j = 0; j <= r; ++j) c_fma(acc, G[pidx(r, j)], v[j]);
    for (int j = r + 1; j < UP; ++j) c_fmac(acc, G[pidx(j, r)], v[j]);
    return acc;
}

// ---------------------------------------------------------------- BF (Alg. 3)
// Line 14 with Lemma 2 (P538, proof P873-890, reading 8):
// z_c = w_c + max{0, 1 - eps/||s - w||} (s - w)/C; eps = 0 is Alg. 3 as
// printed.  Returns the factor multiplying (s - w).
__device__ __forceinline__ float lemma2_scale(float nrm2, float eps, float inv_c) {
    if (!(eps > 0.f)) return inv_c;
    const float nrm = sqrtf(nrm2);
    return nrm > 0.f ? fmaxf(0.f, 1.f - eps / nrm) * inv_c : 0.f;
}

// ---------------------------------------------------------------- CG (Alg. 2)
// sum over the UP-lane group (xor butterfly, the paper's shuffle allreduce P715)
template <int UP>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
    for (int o = UP / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One replicated CG update (Alg. 2 lines 13-18) for lane u given w = sum_c w_c.
template <int UP>
__device__ __forceinline__ void cg_update(float2& x, float2& r, float2& p, float& rr, float2 w, float rho) {
    float2 e = c_add(c_scale(p, rho), w);                                   // line 13
    float phe = group_sum<UP>(fmaf(p.x, e.x, p.y * e.y));                   // Re(p^H e)
    const bool live = rr > 0.f;                                             // reading 4
    float alpha = live ? rr / phe : 0.f;                                    // line 14
    float2 xn = c_add(x, c_scale(p, alpha));                                // line 15
    float2 rn = c_sub(r, c_scale(e, alpha));                                // line 16 (e^(t))
    float rr1 = group_sum<UP>(c_norm2(rn));
    float beta = live ? rr1 / rr : 0.f;                                     // line 17
    if (live) {
        x = xn;
        r = rn;
        p = c_add(rn, c_scale(p, beta));                                    // line 18
        rr = rr1;
    }
}

}  // namespace dbp
