// Per-factor operations and per-primitive entry points (not the batched hot
// path: inspection, tests, and callers that want one kernel at a time).
//
//   factor_apply   EliminationFactor / CompressionFactor / DenseFactor
//                  solve_forward, solve_transpose, mult_transpose, mult_forward
//                  (reference factorization.py:126-148, 173-183, 199-209), in
//                  place on a device n-vector
//   potrf_batched  cholesky (densela.py:87-116): non-finite / asymmetry checks,
//                  pivot floor 1e-14 * max diag, L with zeros above
//   trsm_batched   tri_solve (densela.py:119-146): L^-1 B, L^-T B, B L^-T
//   qrcp_batched   pivoted_qr (densela.py:149-217): every step up to the
//                  zero-column floor, rank = #{|R_ii| > tol |R_00|}, R, perm,
//                  Q (m x min(m,c), or m x m with full_q)
//   gemm           matmul (densela.py:79-84)
#include <algorithm>
#include <cstring>

#include "primitives.h"

namespace sgf {

namespace {
std::vector<int> to_i32(const std::vector<int64_t>& v) { return std::vector<int>(v.begin(), v.end()); }
}  // namespace

void factor_apply(Precond* P, int k, int op, double* d_x) {
  if (k < 0 || k >= (int)P->factors.size()) fail(SGF_INVALID_ARG, "factor index out of range");
  if (op < 0 || op > 3) fail(SGF_INVALID_ARG, "unknown factor operation");
  cudaStream_t st = P->ctx->stream;
  Factor& f = P->factors[k];
  if (f.type == SGF_FACTOR_ELIMINATION && f.c > 0) materialize_l1_e(P);  // pending level-1 couplings
  Arena scratch(st);
  const int m = f.m, c = f.c;
  const long long ld = f.ld;
  int* d_idx = scratch.upload(to_i32(f.idx));
  int* d_nidx = c ? scratch.upload(to_i32(f.nidx)) : nullptr;
  double* xb = scratch.alloc(std::max(m, 1));
  double* zb = scratch.alloc(std::max(m, 1));
  double* xn = scratch.alloc(std::max(c, 1));
  SGF_CUDA(launch_gather(d_x, d_idx, xb, m, st));
  if (c) SGF_CUDA(launch_gather(d_x, d_nidx, xn, c, st));
  const bool elim = f.type == SGF_FACTOR_ELIMINATION && c > 0;
  if (f.type == SGF_FACTOR_COMPRESSION && (op == 2 || op == 3)) {
    // L Q with Q = I - V T V^T (compact WY of the QR's reflectors)
    const int s = f.steps;
    double* w1 = scratch.alloc(std::max(s, 1));
    double* w2 = scratch.alloc(std::max(s, 1));
    if (op == 3) {  // mult_forward: x_B = L (x_B - V T V^T x_B)
      if (s) {
        SGF_CUDA(launch_dmv(f.V, m, s, m, 0, xb, w1, 1.0, 0.0, st));     // V^T xb  (V column-major m x s)
        SGF_CUDA(launch_dmv(f.Tw, s, s, s, 0, w1, w2, 1.0, 0.0, st));    // T w1
        SGF_CUDA(launch_dmv(f.V, m, m, s, 1, w2, xb, -1.0, 1.0, st));    // xb -= V w2
      }
      SGF_CUDA(launch_dmv(f.L, ld, m, m, 0, xb, zb, 1.0, 0.0, st));
    } else {  // mult_transpose: x_B = (I - V T^T V^T) L^T x_B
      SGF_CUDA(launch_dmv(f.L, ld, m, m, 1, xb, zb, 1.0, 0.0, st));
      if (s) {
        SGF_CUDA(launch_dmv(f.V, m, s, m, 0, zb, w1, 1.0, 0.0, st));
        SGF_CUDA(launch_dmv(f.Tw, s, s, s, 1, w1, w2, 1.0, 0.0, st));   // T^T w1
        SGF_CUDA(launch_dmv(f.V, m, m, s, 1, w2, zb, -1.0, 1.0, st));
      }
    }
    SGF_CUDA(launch_scatter(zb, d_idx, d_x, m, st));
    SGF_CUDA(cudaStreamSynchronize(st));  // scratch is released on return
    return;
  }
  switch (op) {
    case 0:  // solve_forward: z_B = inv x_B; x_N -= E z_B
      SGF_CUDA(launch_dmv(f.inv, ld, m, m, 0, xb, zb, 1.0, 0.0, st));
      SGF_CUDA(launch_scatter(zb, d_idx, d_x, m, st));
      if (elim) {
        SGF_CUDA(launch_dmv(f.E, ld, c, m, 0, zb, xn, -1.0, 1.0, st));
        SGF_CUDA(launch_scatter(xn, d_nidx, d_x, c, st));
      }
      break;
    case 1:  // solve_transpose: x_B = inv^T (x_B - E^T x_N)
      if (elim) SGF_CUDA(launch_dmv(f.E, ld, m, c, 1, xn, xb, -1.0, 1.0, st));
      SGF_CUDA(launch_dmv(f.inv, ld, m, m, 1, xb, zb, 1.0, 0.0, st));
      SGF_CUDA(launch_scatter(zb, d_idx, d_x, m, st));
      break;
    case 2:  // mult_transpose: x_B = L^T x_B + E^T x_N
      SGF_CUDA(launch_dmv(f.L, ld, m, m, 1, xb, zb, 1.0, 0.0, st));
      if (elim) SGF_CUDA(launch_dmv(f.E, ld, m, c, 1, xn, zb, 1.0, 1.0, st));
      SGF_CUDA(launch_scatter(zb, d_idx, d_x, m, st));
      break;
    case 3:  // mult_forward: x_N += E x_B; x_B = L x_B
      if (elim) {
        SGF_CUDA(launch_dmv(f.E, ld, c, m, 0, xb, xn, 1.0, 1.0, st));
        SGF_CUDA(launch_scatter(xn, d_nidx, d_x, c, st));
      }
      SGF_CUDA(launch_dmv(f.L, ld, m, m, 0, xb, zb, 1.0, 0.0, st));
      SGF_CUDA(launch_scatter(zb, d_idx, d_x, m, st));
      break;
  }
  SGF_CUDA(cudaStreamSynchronize(st));  // scratch is released on return
}

void potrf_batched(Ctx& ctx, int batch, const int* m, const double* const* A, const int* lda, double* const* L,
                   const int* ldl, int* status, int* piv_index, double* piv_value) {
  cudaStream_t st = ctx.stream;
  Arena scratch(st);
  std::vector<const double*> ap(A, A + batch);
  std::vector<int> mv(m, m + batch), lv(lda, lda + batch);
  double* d_chk = scratch.alloc(2 * std::max(batch, 1));
  int* d_bad = scratch.alloc_t<int>(std::max(batch, 1));
  SGF_CUDA(launch_dense_check(scratch.upload(ap), scratch.upload(mv), scratch.upload(lv), batch, d_chk, d_bad, st));
  std::vector<CholJob> jobs;
  CopyBatch cin, cout_;
  for (int b = 0; b < batch; ++b) {
    if (m[b] <= 0) continue;
    CholJob j;
    j.m = m[b];
    j.ld = pad_ld(m[b]);
    j.W = scratch.alloc((size_t)j.m * j.ld);
    j.X = scratch.alloc((size_t)j.m * j.ld);
    j.node = b;
    cin.add(A[b], lda[b], 1, j.W, j.ld, 1, j.m, j.m);
    cout_.add(j.W, j.ld, 1, L[b], ldl[b], 1, j.m, j.m);
    jobs.push_back(j);
  }
  cin.launch(scratch, st);
  CholCheck chk;
  chk.arena = &scratch;
  chol_inv_batch(ctx, scratch, jobs, &chk);
  cout_.launch(scratch, st);
  std::vector<double> hchk(2 * std::max(batch, 1));
  std::vector<int> hbad(std::max(batch, 1));
  SGF_CUDA(cudaMemcpyAsync(hchk.data(), d_chk, hchk.size() * 8, cudaMemcpyDeviceToHost, st));
  SGF_CUDA(cudaMemcpyAsync(hbad.data(), d_bad, hbad.size() * 4, cudaMemcpyDeviceToHost, st));
  std::vector<int> js(jobs.size());
  std::vector<double> jp(jobs.size());
  if (!jobs.empty()) {
    SGF_CUDA(cudaMemcpyAsync(js.data(), chk.pend[0].status, js.size() * 4, cudaMemcpyDeviceToHost, st));
    SGF_CUDA(cudaMemcpyAsync(jp.data(), chk.pend[0].piv, jp.size() * 8, cudaMemcpyDeviceToHost, st));
  }
  SGF_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < batch; ++b) {
    status[b] = SGF_OK;
    if (piv_index) piv_index[b] = -1;
    if (piv_value) piv_value[b] = 0.0;
  }
  for (size_t i = 0; i < jobs.size(); ++i) {
    const int b = jobs[i].node;
    if (js[i] != 0) {
      status[b] = SGF_NOT_SPD;
      if (piv_index) piv_index[b] = js[i] - 1;
      if (piv_value) piv_value[b] = jp[i];
    }
  }
  // the input checks come first in the reference (densela.py:43-49, 97-104)
  for (int b = 0; b < batch; ++b) {
    if (hbad[b]) status[b] = SGF_INVALID_ARG;
    else if (hchk[2 * b + 1] > 0.0 && hchk[2 * b] > 1e-12 * hchk[2 * b + 1]) status[b] = SGF_NON_SYMMETRIC;
  }
}

void trsm_batched(Ctx& ctx, int batch, const int* m, const int* nrhs, const int* mode, const double* const* L,
                  const int* ldl, const double* const* B, const int* ldb, double* const* X, const int* ldx) {
  cudaStream_t st = ctx.stream;
  for (int b = 0; b < batch; ++b) {
    if (m[b] <= 0 || nrhs[b] <= 0) continue;
    if (mode[b] == 2) {  // X = B L^-T: rows of B are the vectors (X^T = L^-1 B^T)
      SGF_CUDA(launch_trsv(L[b], ldl[b], m[b], nrhs[b], B[b], ldb[b], 1, X[b], ldx[b], 1, 0, st));
    } else if (mode[b] == 0 || mode[b] == 1) {  // columns of B
      SGF_CUDA(launch_trsv(L[b], ldl[b], m[b], nrhs[b], B[b], 1, ldb[b], X[b], 1, ldx[b], mode[b], st));
    } else {
      fail(SGF_INVALID_ARG, "unknown tri_solve mode");
    }
  }
  SGF_CUDA(cudaStreamSynchronize(st));
}

void qrcp_batched(Ctx& ctx, int batch, const int* m, const int* c, const double* const* A, const int* lda,
                  double rank_tol, int full_q, double* const* Q, double* const* R, int* const* perm, int* rank,
                  int* steps) {
  cudaStream_t st = ctx.stream;
  Arena scratch(st);
  std::vector<QrTask> qt;
  std::vector<int> who;
  std::vector<double*> panel;
  CopyBatch cin;
  int* d_out = scratch.alloc_t<int>(2 * std::max(batch, 1));
  SGF_CUDA(cudaMemsetAsync(d_out, 0, 2 * std::max(batch, 1) * sizeof(int), st));
  int max_m = 1, max_c = 1;
  for (int b = 0; b < batch; ++b) {
    if (m[b] <= 0 || c[b] <= 0) continue;
    const int kmax = std::min(m[b], c[b]);
    double* N = scratch.alloc((size_t)m[b] * c[b]);
    cin.add(A[b], lda[b], 1, N, 1, m[b], m[b], c[b]);  // row-major in, column-major panel
    QrTask t;
    std::memset(&t, 0, sizeof t);
    t.Nm = N;
    t.tau = scratch.alloc(kmax);
    t.nrm2 = scratch.alloc(c[b]);
    t.ref2 = scratch.alloc(c[b]);
    t.perm = perm[b];
    t.m = m[b];
    t.c = c[b];
    t.forced_rank = -1;
    t.full_steps = 1;
    t.tol = rank_tol;
    t.out_rank = d_out + b;
    t.out_steps = d_out + batch + b;
    t.tmp = scratch.alloc((size_t)m[b] * c[b]);
    qt.push_back(t);
    who.push_back(b);
    panel.push_back(N);
    max_m = std::max(max_m, m[b]);
    max_c = std::max(max_c, c[b]);
  }
  cin.launch(scratch, st);
  if (!qt.empty()) SGF_CUDA(launch_qrcp(scratch.upload(qt), (int)qt.size(), max_m, st, max_c));
  std::vector<int> hout(2 * std::max(batch, 1));
  SGF_CUDA(cudaMemcpyAsync(hout.data(), d_out, hout.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
  SGF_CUDA(cudaStreamSynchronize(st));
  CopyBatch cr;
  for (size_t i = 0; i < qt.size(); ++i) {
    const int b = who[i], mb = m[b], cb = c[b], kmax = std::min(mb, cb);
    const int s = hout[batch + b];
    rank[b] = hout[b];
    if (steps) steps[b] = s;
    // R: the upper trapezoid of the first `s` rows (rows past the last step are zero)
    SGF_CUDA(cudaMemsetAsync(R[b], 0, (size_t)kmax * cb * sizeof(double), st));
    for (int r = 0; r < s; ++r) cr.add(panel[i] + (long long)r * mb + r, 1, mb, R[b] + (long long)r * cb + r, cb, 1, 1, cb - r);
    const int qcols = full_q ? mb : kmax;
    double* work = scratch.alloc((size_t)mb * std::max(qcols, 1));
    SGF_CUDA(launch_form_q(panel[i], qt[i].tau, mb, s, qcols, Q[b], work, st));
  }
  cr.launch(scratch, st);
  for (int b = 0; b < batch; ++b)
    if (m[b] <= 0 || c[b] <= 0) {
      rank[b] = 0;
      if (steps) steps[b] = 0;
    }
  SGF_CUDA(cudaStreamSynchronize(st));
}

void gemm(Ctx& ctx, int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
          double beta, double* C, int ldc) {
  cudaStream_t st = ctx.stream;
  Arena scratch(st);
  GemmBatch g;
  if (k > 0) {
    g.add(C, ldc, 1, m, n, alpha, beta, seg(A, lda, 1, B, 1, ldb, k));
    g.launch(scratch, st);
  } else if (beta != 1.0) {
    // C = beta C (no product terms): one zero-length segment
    g.add(C, ldc, 1, m, n, 0.0, beta, seg(A, lda, 1, B, 1, ldb, 0));
    g.launch(scratch, st);
  }
  SGF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace sgf
