// dbp_complexity.cu -- Table I of the paper (P566-595): real-multiplication
// counts per algorithm, mode and metric (host-only, exact integer arithmetic).
//
// The formulas, copied cell by cell from Table I (TM = one cluster's PE,
// AR = all PEs; X = S for the S x S mode, U for the U x U mode):
//   ADMM-DL  TM  pre 2U'X^2 + (10X^3 - X)/3      1st 4SU + 4X^2      next 8SU + 4X^2 + 6U + 1
//            AR  pre C(...)                       1st C(4SU + 4X^2)   next C(8SU + 4X^2 + 2U) + 4U + 1
//            (U' = U for S x S, i.e. 2US^2; U' = S for U x U, i.e. 2SU^2)
//   ADMM-UL  S x S  TM pre 2US^2 + (10S^3 - S)/3 + 4US + 4S^2   1st 2U   next 8SU + 4S^2 + 4U
//                   AR pre C(...)                               1st 2U   next C(8SU + 4S^2 + 2U) + 2U
//            U x U  TM pre 2SU^2 + (10U^3 - U)/3 + 4SU + 4U^2   1st 2U   next 4U^2 + 6U
//                   AR pre C(...)                               1st 2U   next C(4U^2 + 4U) + 2U
//   CG-UL    TM pre 4SU + 2U   1st 8SU + 6U   next 8SU + 12U
//            AR pre 4CSU + 2U  1st C(8SU + 4U) + 2U   next C(8SU + 10U) + 2U
//   ZF-DL    6CSU^2 + (10U^3 - 4U)/3 + 4CSU       (centralized, whole count)
//   MMSE-UL  6CSU^2 + (10U^3 - U)/3 + 4CSU
#include <stdint.h>

#include "dbp.h"

namespace {
int64_t third(int64_t v) { return v / 3; }   // exact: every argument below is a multiple of 3
}

extern "C" dbp_status dbp_complexity(int algo, int mode, int metric, int64_t U, int64_t S, int64_t C, int64_t T,
                                     int64_t out[4]) {
    if (!out || U < 1 || S < 1 || C < 1 || T < 1) return DBP_ERR_INVALID_ARG;
    if (metric != DBP_CPLX_TM && metric != DBP_CPLX_AR) return DBP_ERR_INVALID_ARG;
    const bool ar = metric == DBP_CPLX_AR;
    int64_t pre = 0, first = 0, next = 0;
    switch (algo) {
        case DBP_CPLX_ADMM_DL: {
            if (mode != DBP_CPLX_SxS && mode != DBP_CPLX_UxU) return DBP_ERR_INVALID_ARG;
            const int64_t X = mode == DBP_CPLX_SxS ? S : U;
            const int64_t Y = mode == DBP_CPLX_SxS ? U : S;      // 2 U S^2 (SxS) or 2 S U^2 (UxU)
            const int64_t p = 2 * Y * X * X + third(10 * X * X * X - X);
            pre = ar ? C * p : p;
            first = ar ? C * (4 * S * U + 4 * X * X) : 4 * S * U + 4 * X * X;
            next = ar ? C * (8 * S * U + 4 * X * X + 2 * U) + 4 * U + 1 : 8 * S * U + 4 * X * X + 6 * U + 1;
            break;
        }
        case DBP_CPLX_ADMM_UL: {
            if (mode == DBP_CPLX_SxS) {
                const int64_t p = 2 * U * S * S + third(10 * S * S * S - S) + 4 * U * S + 4 * S * S;
                pre = ar ? C * p : p;
                first = 2 * U;
                next = ar ? C * (8 * S * U + 4 * S * S + 2 * U) + 2 * U : 8 * S * U + 4 * S * S + 4 * U;
            } else if (mode == DBP_CPLX_UxU) {
                const int64_t p = 2 * S * U * U + third(10 * U * U * U - U) + 4 * S * U + 4 * U * U;
                pre = ar ? C * p : p;
                first = 2 * U;
                next = ar ? C * (4 * U * U + 4 * U) + 2 * U : 4 * U * U + 6 * U;
            } else {
                return DBP_ERR_INVALID_ARG;
            }
            break;
        }
        case DBP_CPLX_CG_UL:
            pre = ar ? 4 * C * S * U + 2 * U : 4 * S * U + 2 * U;
            first = ar ? C * (8 * S * U + 4 * U) + 2 * U : 8 * S * U + 6 * U;
            next = ar ? C * (8 * S * U + 10 * U) + 2 * U : 8 * S * U + 12 * U;
            break;
        case DBP_CPLX_ZF_DL:
            out[0] = out[3] = 6 * C * S * U * U + third(10 * U * U * U - 4 * U) + 4 * C * S * U;
            out[1] = out[2] = 0;
            return DBP_OK;
        case DBP_CPLX_MMSE_UL:
            out[0] = out[3] = 6 * C * S * U * U + third(10 * U * U * U - U) + 4 * C * S * U;
            out[1] = out[2] = 0;
            return DBP_OK;
        default:
            return DBP_ERR_INVALID_ARG;
    }
    out[0] = pre;
    out[1] = first;
    out[2] = next;
    out[3] = pre + first + (T - 1) * next;
    return DBP_OK;
}
