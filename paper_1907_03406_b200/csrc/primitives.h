// Per-factor operations and per-primitive entry points (primitives.cpp).
#pragma once
#include "precond.h"

namespace sgf {

// op: 0 solve_forward, 1 solve_transpose, 2 mult_transpose, 3 mult_forward
void factor_apply(Precond* P, int k, int op, double* d_x);
void potrf_batched(Ctx& ctx, int batch, const int* m, const double* const* A, const int* lda, double* const* L,
                   const int* ldl, int* status, int* piv_index, double* piv_value);
// mode: 0 L^-1 B, 1 L^-T B, 2 B L^-T
void trsm_batched(Ctx& ctx, int batch, const int* m, const int* nrhs, const int* mode, const double* const* L,
                  const int* ldl, const double* const* B, const int* ldb, double* const* X, const int* ldx);
void qrcp_batched(Ctx& ctx, int batch, const int* m, const int* c, const double* const* A, const int* lda,
                  double rank_tol, int full_q, double* const* Q, double* const* R, int* const* perm, int* rank,
                  int* steps);
void gemm(Ctx& ctx, int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
          double beta, double* C, int ldc);

}  // namespace sgf
