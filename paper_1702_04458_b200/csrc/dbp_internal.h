// dbp_internal.h -- launcher interface between the C ABI (dbp_api.cu) and the
// kernels (dbp_kernels.cu).  Not installed; not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dbp_device.cuh"

namespace dbp {

struct LaunchCtx {
    cudaStream_t stream;
    int* flag;              // device error flag (Cholesky pivot)
    int64_t* launches;      // host counter
    void count(int n) const { if (launches) *launches += n; }
};

enum { PRE_ADMM_ = 0, PRE_BF_ = 1, PRE_CG_ = 2 };

struct AdmmArgs {
    const float2* X;      // [C_loc][N][tri(UP)]
    const float2* yreg;   // [C_loc][N][J][UP]
    float2* lam;          // [C_loc][N][J][UP]
    float2* z;            // [C_loc][N][J][UP]
    float2* wbuf;         // [N][J][UP] consensus buffer (allreduced between launches)
    float2* s_hat;        // [N][J][U]
    uint8_t* hard;        // [N][J][U] or null
    int C_loc, N, J, U, T, NT, CCH, init;
    float rho, gamma;
    Prox px;
    Modem md;
};

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

struct BfArgs {
    const float2* Hd;     // [C_loc][N][U][S]
    const float2* s;      // [N][J][U]
    const float2* X;      // [C_loc][N][tri(UP)]
    float2* m;            // [C_loc][N][J][UP]  state (split path)
    float2* lam;          // [C_loc][N][J][UP]
    float2* wbuf;         // [N][J][UP]
    float2* xout;         // [C_loc][N][J][S]
    int C_loc, C, N, J, U, S, T, NT, CCH, step;   // step: 2..T iteration, T+1 = final
    float rho_inv, gamma, a0, inv_c;
};

size_t pre_smem(int UP, int S, int U, int J, int mode);
cudaError_t launch_pre(const LaunchCtx& L, int UP, int mode, const float2* H, const float2* y, int S, int U,
                       int J, long npairs, float delta, float2* Xout, float2* vout);

size_t admm_step_smem(int UP, int NT, int CCH, int J);
size_t admm_fused_smem(int UP, int NT, int C);
cudaError_t launch_admm_step(const LaunchCtx& L, int UP, AdmmArgs a);
cudaError_t launch_admm_fused(const LaunchCtx& L, int UP, AdmmArgs a);
cudaError_t launch_prox_out(const LaunchCtx& L, int UP, const float2* wbuf, int N, int J, int U, Prox px,
                            Modem md, float2* s_hat, uint8_t* hard);
cudaError_t launch_slice(const LaunchCtx& L, const float2* x, long count, Modem md, uint8_t* bits);

cudaError_t launch_cg_gsum(const LaunchCtx& L, int UP, const float2* Gp, const float2* mf, int C_loc, int N,
                           int J, float2* Gloc, float2* wbuf);
cudaError_t launch_cg_it(const LaunchCtx& L, int UP, bool fused, CgArgs a);

size_t bf_step_smem(int UP, int NT, int CCH, int J);
size_t bf_fused_smem(int UP, int NT, int C);
cudaError_t launch_bf_step(const LaunchCtx& L, int UP, BfArgs a);
cudaError_t launch_bf_fused(const LaunchCtx& L, int UP, BfArgs a);

}  // namespace dbp
