// Small dense kernels behind the per-factor methods (factor views'
// solve_forward / solve_transpose / mult_transpose / mult_forward, reference
// factorization.py:126-148, 173-183, 199-209) and the per-primitive C ABI
// (sgf_potrf_batched / sgf_trsm_batched / sgf_qrcp_batched, reference
// densela.py:87-217).  These serve inspection, tests and one-off calls, not
// the level-batched hot path, so they favour simplicity: one warp per output
// row (or one thread per output column for transposed products).
#include <cfloat>
#include <cmath>

#include "common.h"

namespace sgf {

// y = beta*y + alpha * op(M) v, M row-major with leading dimension ld;
// op(M) is rows x inner: M itself (trans = 0) or M^T (trans = 1)
__global__ void __launch_bounds__(256) dmv_kernel(const double* __restrict__ M, long long ld, int rows, int inner,
                                                  int trans, const double* __restrict__ v, double* __restrict__ y,
                                                  double alpha, double beta) {
  if (!trans) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const double* row = M + (long long)warp * ld;
    double s = 0.0;
    for (int j = lane; j < inner; j += 32) s = fma(row[j], v[j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[warp] = (beta == 0.0 ? 0.0 : beta * y[warp]) + alpha * s;
  } else {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double s = 0.0;
    for (int j = 0; j < inner; ++j) s = fma(M[(long long)j * ld + i], v[j], s);
    y[i] = (beta == 0.0 ? 0.0 : beta * y[i]) + alpha * s;
  }
}

cudaError_t launch_dmv(const double* M, long long ld, int rows, int inner, int trans, const double* v, double* y,
                       double alpha, double beta, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  const long long threads = trans ? rows : 32LL * rows;
  count_launch();
  dmv_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(M, ld, rows, inner, trans, v, y, alpha, beta);
  return cudaGetLastError();
}

// Per matrix of a dense batch (row-major, ld): flags[0] |= non-finite entry,
// out[2b] = max |A - A^T|, out[2b+1] = max |A| (densela.py:43-49, 97-104)
__global__ void dense_check_kernel(const double* const* __restrict__ A, const int* __restrict__ m,
                                   const int* __restrict__ ld, double* __restrict__ out, int* __restrict__ bad) {
  const int b = blockIdx.x;
  const double* a = A[b];
  const int n = m[b], l = ld[b];
  double asym = 0.0, scale = 0.0;
  bool nf = false;
  for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    const double x = a[(long long)i * l + j];
    nf |= !isfinite(x);
    scale = fmax(scale, fabs(x));
    asym = fmax(asym, fabs(x - a[(long long)j * l + i]));
  }
  __shared__ double sa[32], ss[32];
  __shared__ int sn;
  if (threadIdx.x == 0) sn = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
    scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  }
  __syncthreads();
  if (nf) atomicOr(&sn, 1);
  if ((threadIdx.x & 31) == 0) {
    sa[threadIdx.x >> 5] = asym;
    ss[threadIdx.x >> 5] = scale;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      sa[0] = fmax(sa[0], sa[w]);
      ss[0] = fmax(ss[0], ss[w]);
    }
    out[2 * b] = sa[0];
    out[2 * b + 1] = ss[0];
    bad[b] = sn;
  }
}

cudaError_t launch_dense_check(const double* const* A, const int* m, const int* ld, int n, double* out, int* bad,
                               cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  dense_check_kernel<<<n, 256, 0, s>>>(A, m, ld, out, bad);
  return cudaGetLastError();
}

// Q = H_0 H_1 ... H_{s-1} applied to the first qcols columns of I_m, one
// thread block per column (reference densela.py:206-210 accumulates the same
// product backward).  V column-major (unit lower trapezoid, m x s), Q
// row-major m x qcols.
__global__ void form_q_kernel(const double* __restrict__ V, const double* __restrict__ tau, int m, int s, int qcols,
                              double* __restrict__ Q, double* __restrict__ work) {
  const int j = blockIdx.x;
  double* q = work + (long long)j * m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) q[i] = (i == j) ? 1.0 : 0.0;
  __shared__ double red[32];
  __syncthreads();
  for (int k = s - 1; k >= 0; --k) {
    const double* w = V + (long long)k * m;
    double d = 0.0;
    for (int i = k + threadIdx.x; i < m; i += blockDim.x) d = fma(i == k ? 1.0 : w[i], q[i], d);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int u = 0; u < (int)(blockDim.x >> 5); ++u) t += red[u];
      red[0] = t;
    }
    __syncthreads();
    const double f = tau[k] * red[0];
    for (int i = k + threadIdx.x; i < m; i += blockDim.x) q[i] -= f * (i == k ? 1.0 : w[i]);
    __syncthreads();
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) Q[(long long)i * qcols + j] = q[i];
}

cudaError_t launch_form_q(const double* V, const double* tau, int m, int s, int qcols, double* Q, double* work,
                          cudaStream_t st) {
  if (qcols <= 0 || m <= 0) return cudaSuccess;
  count_launch();
  form_q_kernel<<<qcols, 256, 0, st>>>(V, tau, m, s, qcols, Q, work);
  return cudaGetLastError();
}


// Triangular solves against a lower-triangular L (row-major, ldl), one block
// per right-hand-side vector, the vector held in shared memory:
//   trans = 0: x = L^{-1} b (forward substitution), 1: x = L^{-T} b (backward).
// Element e of vector v lives at B[v*bvs + e*bes] (X likewise), so the same
// kernel serves L^{-1} B, L^{-T} B (columns of B) and B L^{-T} (rows of B).
// Reference densela.py:119-146 (scipy solve_triangular).
__global__ void trsv_kernel(const double* __restrict__ L, long long ldl, int m, const double* __restrict__ B,
                            long long bvs, long long bes, double* __restrict__ X, long long xvs, long long xes,
                            int trans) {
  extern __shared__ double xs[];
  __shared__ double red[32];
  const int v = blockIdx.x;
  for (int e = threadIdx.x; e < m; e += blockDim.x) xs[e] = B[(long long)v * bvs + (long long)e * bes];
  __syncthreads();
  for (int t = 0; t < m; ++t) {
    const int i = trans ? m - 1 - t : t;
    double d = 0.0;
    if (!trans) {
      for (int j = threadIdx.x; j < i; j += blockDim.x) d = fma(L[(long long)i * ldl + j], xs[j], d);
    } else {
      for (int j = i + 1 + threadIdx.x; j < m; j += blockDim.x) d = fma(L[(long long)j * ldl + i], xs[j], d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
      xs[i] = (xs[i] - s) / L[(long long)i * ldl + i];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m; e += blockDim.x) X[(long long)v * xvs + (long long)e * xes] = xs[e];
}

cudaError_t launch_trsv(const double* L, long long ldl, int m, int nvec, const double* B, long long bvs,
                        long long bes, double* X, long long xvs, long long xes, int trans, cudaStream_t s) {
  if (m <= 0 || nvec <= 0) return cudaSuccess;
  const size_t smem = (size_t)m * sizeof(double);
  static FuncAttrs fa;
  cudaError_t e = ensure_smem(trsv_kernel, smem, fa);
  if (e != cudaSuccess) return e;
  count_launch();
  trsv_kernel<<<nvec, 256, smem, s>>>(L, ldl, m, B, bvs, bes, X, xvs, xes, trans);
  return cudaGetLastError();
}

// ---- sharded factorization / apply / PCG helpers ------------------------------
// flags[b] = 1 when block b (ptrs[b], counts[b] doubles) holds a nonzero
__global__ void nonzero_flags_kernel(const double* const* __restrict__ ptrs, const long long* __restrict__ counts,
                                     int* __restrict__ flags) {
  const int b = blockIdx.x;
  const double* p = ptrs[b];
  int nz = 0;
  for (long long i = threadIdx.x; i < counts[b] && !nz; i += blockDim.x) nz = p[i] != 0.0;
  nz = __syncthreads_or(nz);
  if (threadIdx.x == 0) flags[b] = nz;
}

cudaError_t launch_nonzero_flags(const double* const* ptrs, const long long* counts, int n, int* flags,
                                 cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  nonzero_flags_kernel<<<n, 256, 0, s>>>(ptrs, counts, flags);
  return cudaGetLastError();
}

// dst[b][i] += packed[offs[b] + i]  (one block per destination block)
__global__ void add_packed_kernel(double* const* __restrict__ dst, const long long* __restrict__ counts,
                                  const long long* __restrict__ offs, const double* __restrict__ packed) {
  const int b = blockIdx.x;
  double* d = dst[b];
  const double* s = packed + offs[b];
  for (long long i = threadIdx.x; i < counts[b]; i += blockDim.x) d[i] += s[i];
}

cudaError_t launch_add_packed(double* const* dst, const long long* counts, const long long* offs, int n,
                              const double* packed, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  add_packed_kernel<<<n, 256, 0, s>>>(dst, counts, offs, packed);
  return cudaGetLastError();
}

// out[i] = y[idx[i]] - x[idx[i]]   (changes of the top unknowns)
__global__ void gather_diff_kernel(const double* __restrict__ y, const double* __restrict__ x,
                                   const int* __restrict__ idx, double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const int k = idx[i];
    out[i] = y[k] - x[k];
  }
}
// y[idx[i]] = base[idx[i]] + d[i]  (base may be null: y[idx[i]] = d[i])
__global__ void scatter_base_kernel(double* __restrict__ y, const double* __restrict__ base,
                                    const int* __restrict__ idx, const double* __restrict__ d, long long n) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const int k = idx[i];
    y[k] = (base ? base[k] : 0.0) + d[i];
  }
}
// y[i] = 0 where owned[i] == 0
__global__ void mask_kernel(double* __restrict__ y, const unsigned char* __restrict__ owned, long long n) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    if (!owned[i]) y[i] = 0.0;
}

static unsigned grid_n(long long n) {
  long long g = (n + 255) / 256;
  return (unsigned)(g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g));
}

cudaError_t launch_gather_diff(const double* y, const double* x, const int* idx, double* out, long long n,
                               cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  gather_diff_kernel<<<grid_n(n), 256, 0, s>>>(y, x, idx, out, n);
  return cudaGetLastError();
}
cudaError_t launch_scatter_base(double* y, const double* base, const int* idx, const double* d, long long n,
                                cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  scatter_base_kernel<<<grid_n(n), 256, 0, s>>>(y, base, idx, d, n);
  return cudaGetLastError();
}
cudaError_t launch_mask(double* y, const unsigned char* owned, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  mask_kernel<<<grid_n(n), 256, 0, s>>>(y, owned, n);
  return cudaGetLastError();
}

}  // namespace sgf
