// dbp_internal.h -- launcher interface between the C ABI (dbp_api.cu) and the
// kernels (dbp_kernels.cu).  Not installed; not part of the public ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dbp_device.cuh"

namespace dbp {

#define DBP_DISPATCH_UP(UP_, ...)                                    \
    switch (UP_) {                                                   \
        case 4: { constexpr int UPc = 4; __VA_ARGS__; } break;       \
        case 8: { constexpr int UPc = 8; __VA_ARGS__; } break;       \
        case 16: { constexpr int UPc = 16; __VA_ARGS__; } break;     \
        default: { constexpr int UPc = 32; __VA_ARGS__; } break;     \
    }


struct LaunchCtx {
    cudaStream_t stream;
    int* flag;              // device error flag (Cholesky pivot)
    int64_t* launches;      // host counter
    int pdl = 0;            // launch with programmatic stream serialization (DBP_OPT_OVERLAP_PREV)
    void count(int n) const { if (launches) *launches += n; }
};

enum { PRE_ADMM_ = 0, PRE_BF_ = 1, PRE_CG_ = 2 };

// <<<grid, block, smem, L.stream>>>, with programmatic stream serialization when L.pdl
template <typename K, typename... Args>
static inline bool launch_pdl(K kernel, int grid, int block, size_t smem, const LaunchCtx& L, Args... args) {
    if (!L.pdl) {
        kernel<<<grid, block, smem, L.stream>>>(args...);
        return true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = L.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kernel, args...) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}

struct CgArgs {
    const float2* Gloc;   // [N][tri(UP)]
    float2* wbuf;         // [N][J][UP]
    float2* x;            // [N][J][UP] replicated CG state (split path)
    float2* r;
    float2* p;
    float* rr;            // [N][J]
    float2* x_hat;        // [N][J][U]
    uint8_t* hard;
    int N, J, U, T, step; // step 0: init (r = y^MRC) + matvec; 1..T-1: update + matvec; T: final update
    float rho;
    Modem md;
};



// 3-D TMA tensor map over 8-byte elements (dims innermost first, box may exceed
// the tensor: out-of-bounds elements are zero-filled).  false if unsupported.
bool make_map3(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
               uint32_t b2);
// swz128: CU_TENSOR_MAP_SWIZZLE_128B (16-B chunk c of 128-B row r lands at chunk c ^ (r & 7); the
// shared-memory destination must be 1024-B aligned), box inner extent <= 16 elements.
bool make_map4(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint32_t b0,
               uint32_t b1, uint32_t b2, uint32_t b3, bool swz128 = false);
// Device-side consensus over ranks (NEXT-1, DBP_OPT_DEVICE_CONSENSUS): every rank owns one
// symmetric buffer, mapped into all ranks (CUDA IPC over NVLink):
//   part [2 round parity][8 ranks][cap subcarriers][16 users] uint4 = {re, id, im, id}.
// A round stores the CTA's local partial into every rank's part[par][my_rank][n] with the round
// id in both 8-byte halves (LL protocol), then polls its own part[par][p][n] for every p until
// both ids match and sums in rank order (deterministic, identical on every rank).  Round ids
// grow monotonically across calls (host counter), so nothing is ever reset; parity double
// buffering keeps a fast rank's round r + 2 from overwriting round r before it is read.
struct XArgs {
    uint4* part[8];
    int world, rank, cap, on;
    unsigned base;                       // round id of this call's round t is base + t
};

// single-kernel per-subcarrier solvers (dbp_fused.cu): world == 1, or world > 1 with the
// device-side consensus (xc != nullptr, xc->on)
bool fused_ok(int UP, int C, int N, int J, int S, int U);
bool launch_fused_ul(const LaunchCtx& L, int UP, bool cg, const float2* H, const float2* y, int C, int N, int S, int U,
                     int T, float rho, float gamma, Prox px, Modem md, float2* s_hat, uint8_t* hard,
                     const XArgs* xc = nullptr);
bool launch_fused_central(const LaunchCtx& L, int UP, bool dl, const float2* H, const float2* ys, int C, int N, int S,
                          int U, float reg, Modem md, float2* out, uint8_t* hard);
bool launch_fused_dl(const LaunchCtx& L, int UP, const float2* Hd, const float2* s, int C, int C_glob, int N, int S,
                     int U, int T, float rho, float gamma, float a0, float eps, float2* x, const XArgs* xc = nullptr);
// ADMM-UL with N_sym = 2..7 symbols per subcarrier, gamma == 1, world == 1 (dbp_fusedj.cu)
// (cg: CG-UL with N_sym = 2..7, rho = N0/Es)
bool launch_fused_ulj(const LaunchCtx& L, int UP, bool cg, const float2* H, const float2* y, int C, int N, int S, int U,
                      int J, int T, float rho, Prox px, Modem md, float2* s_hat, uint8_t* hard);
// CG-UL at world 1, N_sym = 1, UP = 16: the cluster-summed Gram on the tensor cores (dbp_cgtc.cu)
bool launch_cg_tc(const LaunchCtx& L, int UP, const float2* H, const float2* y, int C, int N, int S, int U, int J,
                  int T, float rho, Modem md, float2* x_hat, uint8_t* hard);
// G_loc = sum_c H_c^H H_c and y^MRC_loc over the rank's clusters on the tensor cores (dbp_cgg.cu;
// J = 1, UP = 16 / 32, U even, S <= 64): the CG split path's preprocessing
bool launch_cgg_tc(const LaunchCtx& L, int UP, const float2* H, const float2* y, int C, int N, int S, int U,
                   float2* G, float2* mrc);
bool cgg_tc_ok(int UP, int J, int N, int C, int S, int U);
bool cg_tc_ok(int UP, int J, int N, int C, int S);
size_t prelr_smem(int UP, int S, int U, int J, bool ul);
bool launch_prefold(const LaunchCtx& L, int UP, int mode, const float2* H, const float2* y, int S, int U, int J,
                    long npairs, float delta, float2* Gout, float2* vout);
// Lane-row preprocessing: mode 0 = Gram + H^H y (CG), 1 = G^{-1} + y^reg (ADMM-UL), 2 = B^{-1} (ADMM-DL)
cudaError_t launch_prelr(const LaunchCtx& L, int UP, int mode, const float2* H, const float2* y, int S, int U, int J,
                         long npairs, float delta, float2* Gout, float2* vout);
// Gram (+ delta I) per pair -> Gout [pairs][tri(UP)]; matched filter -> mfout [pairs][J][UP] (not for BF)

cudaError_t launch_prox_out(const LaunchCtx& L, int UP, const float2* wbuf, int N, int J, int U, Prox px,
                            Modem md, float2* s_hat, uint8_t* hard);
cudaError_t launch_slice(const LaunchCtx& L, const float2* x, long count, Modem md, uint8_t* bits);

cudaError_t launch_cg_gsum(const LaunchCtx& L, int UP, const float2* Gp, const float2* mf, int C_loc, int N,
                           int J, float2* Gloc, float2* wbuf);
cudaError_t launch_cg_it(const LaunchCtx& L, int UP, bool fused, CgArgs a);

struct UlArgs {
    const float2* G;      // [C_loc][N][tri(UP)]  G = H^H H + rho I (packed lower)
    const float2* mf;     // [C_loc][N][J][UP]    H^H y
    float2* Ginv;         // split: [C_loc][N][tri(UP)] G^{-1} (packed lower)
    float2* yreg;         // split: [C_loc][N][J][UP]
    float2* lam;          // split state
    float2* z;
    float2* wbuf;         // [N][J][UP]
    float2* s_hat;        // [N][J][U]
    uint8_t* hard;
    int* flag;
    int C_loc, N, J, U, T, NT, init;
    int wonly;            // split: gamma == 1 -> carry only w_c = z_c + lambda_c between rounds
    float rho, gamma;
    Prox px;
    Modem md;
};

struct DlArgs {
    const float2* G;      // [C_loc][N][tri(UP)]  B = H H^H + rho^{-1} I (packed lower)
    const float2* Hd;     // [C_loc][N][U][S]
    const float2* s;      // [N][J][U]
    float2* Binv;         // split: [C_loc][N][tri(UP)]
    float2* m;            // split state [C_loc][N][J][UP]
    float2* lam;
    float2* wbuf;         // [N][J][UP]
    float2* x;            // [C_loc][N][J][S]
    int* flag;
    int C_loc, C, N, J, U, S, T, NT, step;
    float rho_inv, gamma, a0, inv_c, eps;
};

size_t iter_smem(int UP, int NT, int C);
bool iter_cfg(int UP, int C_loc, int N, int max_smem, int* NT);
size_t split_smem(int UP, int NT, int CCH, int J);
void split_cfg(int UP, int C_loc, int N, int J, int* NT, int* CCH);
cudaError_t launch_admm_gj(const LaunchCtx& L, int UP, UlArgs a);
cudaError_t launch_admm_it(const LaunchCtx& L, int UP, UlArgs a, int CCH);
cudaError_t launch_bf_gj(const LaunchCtx& L, int UP, DlArgs a);
cudaError_t launch_central_solve(const LaunchCtx& L, int UP, bool dl, const float2* Gloc, const float2* rhs, float delta,
                                 int N, int J, int U, float2* out, uint8_t* hard, Modem md);
cudaError_t launch_zf_out(const LaunchCtx& L, int UP, const float2* Hd, const float2* r, int N, int J, int U, int S,
                          long npairs, float2* x);
cudaError_t launch_bf_it(const LaunchCtx& L, int UP, DlArgs a, int CCH);

// S x S forms of Alg. 1 / Alg. 3 (dbp_ss.cu, NEXT-2): one warp per pair, one launch per round
struct SsArgs {
    const float2* H;      // UL [C_loc][N][S][U]; DL [C_loc][N][U][S]
    const float2* y;      // UL [C_loc][N][J][S]
    const float2* s;      // DL [N][J][U]
    float2* Ainv;         // [C_loc][N][tri(SP)]
    float2* yreg;         // UL [C_loc][N][J][UPW]
    float2* lam;          // [C_loc][N][J][UPW]
    float2* st;           // UL: z; DL: m   [C_loc][N][J][UPW]
    float2* wbuf;         // [N][J][UPW] consensus partial sums (UPW = the API's UP)
    float2* x;            // DL output [C_loc][N][J][S]
    int* flag;
    int C_loc, N, J, S, U, UPW, T, step;   // step: UL 1..T; DL 0 = init, t = 2..T
    float delta, rho, gamma, a0, inv_c, eps;
    Prox px;
};

cudaError_t launch_ss_pre(const LaunchCtx& L, bool dl, SsArgs a);
cudaError_t launch_ss_it(const LaunchCtx& L, bool dl, SsArgs a);

}  // namespace dbp
