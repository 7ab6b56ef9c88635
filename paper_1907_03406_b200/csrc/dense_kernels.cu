// Small dense kernels: diagonal-tile Cholesky + inverse, tiled block copies
// (merge / gather / densify), CSR -> block scatter, identity blocks,
// triangle zeroing, per-node max diagonal.
#include <cmath>

#include <cstdlib>

#include "common.h"

namespace sgf {

// ---------------------------------------------------------------------------
// Diagonal tile Cholesky (nb <= 64).  Restates the reference pivot rule
// (densela.py:106-110): breakdown when the pivot is <= floor (= 1e-14 x the
// largest diagonal entry of the node's block) or not finite.  The factor
// overwrites the tile; its inverse goes to Dinv (and optionally into the
// diagonal tile of the node's L^{-1}).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) diag_chol_kernel(const DiagTask* __restrict__ tasks,
                                                        int* __restrict__ status,
                                                        double* __restrict__ pivval,
                                                        double* const* __restrict__ xdiag,
                                                        const int* __restrict__ ldx) {
  // left-looking column Cholesky (the reference's order, densela.py:107-114)
  // with the inverse built row by row alongside; a quad of threads per row,
  // two barriers per column
  extern __shared__ double dsm[];
  double(*S)[65] = reinterpret_cast<double(*)[65]>(dsm);
  double(*D)[65] = reinterpret_cast<double(*)[65]>(dsm + 64 * 65);
  double* col = dsm + 2 * 64 * 65;
  const DiagTask T = tasks[blockIdx.x];
  const int nb = T.nb, tid = threadIdx.x;
  const int q = tid >> 2, sub = tid & 3;
  double* W = T.W + (long long)T.k0 * T.ld + T.k0;
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    int r = idx / nb, c = idx % nb;
    S[r][c] = W[(long long)r * T.ld + c];
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const int i = j + q;
    double acc = 0.0;
    if (i < nb)
      for (int k = sub; k < j; k += 4) acc = fma(S[i][k], S[j][k], acc);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (i < nb && sub == 0) col[i] = S[i][j] - acc;
    __syncthreads();
    const double d = col[j];
    if (!(d > *T.floor) || !isfinite(d)) {
      if (tid == 0 && status[T.node] == 0) {
        status[T.node] = T.k0 + j + 1;
        pivval[T.node] = d;
      }
      return;  // uniform: every thread saw the same pivot
    }
    const double djj = sqrt(d);
    if (i < nb && sub == 0) S[i][j] = (i == j) ? djj : col[i] / djj;
    // row j of the inverse: D[j][c] = -(sum_{c<=k<j} L[j][k] D[k][c]) / L[j][j]
    double a2 = 0.0;
    if (q < j)
      for (int k = q + sub; k < j; k += 4) a2 = fma(S[j][k], D[k][q], a2);
    a2 += __shfl_xor_sync(0xffffffffu, a2, 1);
    a2 += __shfl_xor_sync(0xffffffffu, a2, 2);
    if (sub == 0 && q <= j) D[j][q] = (q == j) ? 1.0 / djj : -a2 / djj;
    __syncthreads();
  }
  double* X = xdiag ? xdiag[blockIdx.x] : nullptr;
  const int lx = ldx ? ldx[blockIdx.x] : 0;
  for (int idx = tid; idx < 64 * 64; idx += blockDim.x) {
    const int r = idx >> 6, c = idx & 63;
    const bool in = (r < nb && c < nb && c <= r);
    const double dv = in ? D[r][c] : 0.0;
    T.Dinv[idx] = dv;
    if (r < nb && c < nb) {
      W[(long long)r * T.ld + c] = in ? S[r][c] : 0.0;
      if (X) X[(long long)(T.k0 + r) * lx + T.k0 + c] = dv;
    }
  }
}

// Right-looking variant with the inverse fused into the same sweep: after
// column j of L and row j of L^{-1} are final, one pass updates every later
// row i at every position x <= i -- x > j: the trailing matrix,
// S[i][x] -= L[i][j] L[x][j]; x <= j: the inverse rows, R[i][x] -= L[i][j] D[j][x]
// (R = identity initially, D[j][:] = R[j][:] / L[j][j]).  Two barriers per
// column and no serial dot products: the column latency is a few smem
// round trips instead of a 16-deep dependent FMA chain (the left-looking
// kernel above).  Same breakdown rule and outputs.
__global__ void __launch_bounds__(256) diag_chol_rl_kernel(const DiagTask* __restrict__ tasks,
                                                           int* __restrict__ status, double* __restrict__ pivval,
                                                           double* const* __restrict__ xdiag,
                                                           const int* __restrict__ ldx) {
  extern __shared__ double dsm[];
  double(*S)[65] = reinterpret_cast<double(*)[65]>(dsm);
  double(*D)[65] = reinterpret_cast<double(*)[65]>(dsm + 64 * 65);
  const DiagTask T = tasks[blockIdx.x];
  const int nb = T.nb, tid = threadIdx.x;
  const int x = tid & 63, rg = tid >> 6;
  double* W = T.W + (long long)T.k0 * T.ld + T.k0;
  for (int idx = tid; idx < nb * nb; idx += 256) {
    const int r = idx / nb, c = idx % nb;
    S[r][c] = W[(long long)r * T.ld + c];
    D[r][c] = (r == c) ? 1.0 : 0.0;
  }
  const double floor_ = *T.floor;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double d = S[j][j];
    if (!(d > floor_) || !isfinite(d)) {
      if (tid == 0 && status[T.node] == 0) {
        status[T.node] = T.k0 + j + 1;
        pivval[T.node] = d;
      }
      return;  // uniform: every thread saw the same pivot
    }
    const double djj = sqrt(d);
    // column j of L (rows below j), row j of L^{-1} (columns <= j)
    if (rg == 0) {
      if (x > j && x < nb) S[x][j] = S[x][j] / djj;
    } else if (rg == 1) {
      if (x <= j) D[j][x] = D[j][x] / djj;
    }
    __syncthreads();
    if (rg == 0 && x == 0) S[j][j] = djj;
    const double lxj = (x > j && x < nb) ? S[x][j] : 0.0;
    const double dj = (x <= j) ? D[j][x] : 0.0;
    for (int i = j + 1 + rg; i < nb; i += 4) {
      if (x > i) continue;
      const double lij = S[i][j];
      if (x > j) S[i][x] = fma(-lij, lxj, S[i][x]);
      else D[i][x] = fma(-lij, dj, D[i][x]);
    }
    __syncthreads();
  }
  double* X = xdiag ? xdiag[blockIdx.x] : nullptr;
  const int lx = ldx ? ldx[blockIdx.x] : 0;
  for (int idx = tid; idx < 64 * 64; idx += 256) {
    const int r = idx >> 6, c = idx & 63;
    const bool in = (r < nb && c < nb && c <= r);
    const double dv = in ? D[r][c] : 0.0;
    T.Dinv[idx] = dv;
    if (r < nb && c < nb) {
      W[(long long)r * T.ld + c] = in ? S[r][c] : 0.0;
      if (X) X[(long long)(T.k0 + r) * lx + T.k0 + c] = dv;
    }
  }
}

// Register-resident form of the right-looking sweep above (the default).
// Threads 0-127 hold the factor by columns: column x = t & 63, rows
// [32h, 32h + 32), h = t >> 6.  Threads 128-255 hold the inverse by rows:
// row i = t & 63, columns [32h, 32h + 32).  Step j is one uniform rank-1
// update of both with no per-element branches:
//   S[i][x] -= S[i][j] (S[x][j] / S[j][j])  for x > j   (trailing matrix)
//   D[i][x] -= (S[i][j] / S[j][j]) D[j][x]  for i > j   (inverse rows)
// with S[.][j] and D[j][.] the raw (unscaled) pivot column and row, which the
// owners publish to shared memory at the end of step j - 1 (double-buffered
// by the parity of j: one barrier per column).  Finished columns / rows
// (p <= j) skip the step.  The S update runs over whole columns: rows above
// the pivot only touch the unused upper triangle of the active columns, so
// the published column's rows < j (upper-triangle values) never reach the
// lower triangle or the inverse; the upper triangle of D stays exactly zero
// (D[j][x] = 0 for x > j), so its published rows need no masking either.
// The coefficients need only S[.][j] / S[j][j] (one division per thread and
// column); columns of L and rows of L^{-1} stay raw once final and are
// divided by sqrt(S[j][j]) when written out (no square root on the column
// chain).  Per column a thread issues 16 paired shared loads and 32 FMAs,
// the publishers (the owners of column and row j + 1) 16 paired stores.
// Same breakdown rule and outputs as the kernels above (the rounding
// differs at the last bits).
__global__ void __launch_bounds__(256, 2) diag_chol_reg_kernel(const DiagTask* __restrict__ tasks,
                                                               int* __restrict__ status,
                                                               double* __restrict__ pivval,
                                                               double* const* __restrict__ xdiag,
                                                               const int* __restrict__ ldx) {
  __shared__ __align__(16) double colraw[2][64];  // S[.][j], rows < j zero
  __shared__ __align__(16) double rowraw[2][64];  // D[j][.], columns > j zero
  __shared__ double piv_s[64];                    // raw pivots S[j][j]
  __shared__ double sD[64][65];                   // output staging (coalesced stores)
  const DiagTask T = tasks[blockIdx.x];
  const int nb = T.nb, tid = threadIdx.x;
  const bool isD = tid >= 128;
  const int p = tid & 63, h = (tid >> 6) & 1, base = 32 * h;  // column (S) or row (D) p
  double* W = T.W + (long long)T.k0 * T.ld + T.k0;
  double v[32];
  if (!isD) {
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int i = base + q;
      v[q] = (i < nb && p <= i && p < nb) ? W[(long long)i * T.ld + p] : 0.0;
    }
    if (p == 0) {
#pragma unroll
      for (int q = 0; q < 32; ++q) colraw[0][base + q] = v[q];
    }
  } else {
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = (base + q == p) ? 1.0 : 0.0;
    if (p == 0) {
#pragma unroll
      for (int q = 0; q < 32; ++q) rowraw[0][base + q] = v[q];
    }
  }
  const double floor_ = *T.floor;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const int b = j & 1;
    const double piv = colraw[b][j];
    if (!(piv > floor_) || !isfinite(piv)) {
      if (tid == 0 && status[T.node] == 0) {
        status[T.node] = T.k0 + j + 1;
        pivval[T.node] = piv;
      }
      return;  // uniform: every thread saw the same pivot
    }
    const double2* c2 = reinterpret_cast<const double2*>(colraw[b] + base);
    if (p <= j) {
      // finished column of L / row of L^{-1}: nothing to update
    } else if (!isD) {
      const double f = colraw[b][p] / piv;  // S[x][j] / S[j][j]
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double2 l = c2[q];
        v[2 * q] = fma(-l.x, f, v[2 * q]);
        v[2 * q + 1] = fma(-l.y, f, v[2 * q + 1]);
      }
    } else {
      const double l = colraw[b][p] / piv;
      const double2* r2v = reinterpret_cast<const double2*>(rowraw[b] + base);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double2 dj = r2v[q];
        v[2 * q] = fma(-l, dj.x, v[2 * q]);
        v[2 * q + 1] = fma(-l, dj.y, v[2 * q + 1]);
      }
    }
    if (tid == 0) piv_s[j] = piv;
    // publish column j + 1 of S (rows >= j + 1) and row j + 1 of D (columns <= j + 1)
    const int jn = j + 1;
    if (p == jn) {
      double2* dst = reinterpret_cast<double2*>((isD ? rowraw[b ^ 1] : colraw[b ^ 1]) + base);
#pragma unroll
      for (int q = 0; q < 16; ++q) dst[q] = make_double2(v[2 * q], v[2 * q + 1]);
    }
    __syncthreads();
  }
  // scaled outputs: L[i][x] = raw * rinv_x (i > x), sqrt pivot on the
  // diagonal; L^{-1}[i][x] = raw * rinv_i (x <= i)
  if (!isD) {
    const double dp = p < nb ? sqrt(piv_s[p]) : 1.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int i = base + q;
      if (i < nb && p < nb) W[(long long)i * T.ld + p] = i > p ? v[q] / dp : (i == p ? dp : 0.0);
    }
  } else {
    const double dp = p < nb ? sqrt(piv_s[p]) : 1.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int x = base + q;
      sD[p][x] = (p < nb && x < nb && x <= p) ? v[q] / dp : 0.0;
    }
  }
  __syncthreads();
  double* X = xdiag ? xdiag[blockIdx.x] : nullptr;
  const int lx = ldx ? ldx[blockIdx.x] : 0;
  for (int idx = tid; idx < 64 * 64; idx += 256) {
    const int r = idx >> 6, c = idx & 63;
    const double dv = sD[r][c];
    T.Dinv[idx] = dv;
    if (X && r < nb && c < nb) X[(long long)(T.k0 + r) * lx + T.k0 + c] = dv;
  }
}

cudaError_t launch_diag_chol_ex(const DiagTask* d_tasks, int ntasks, int* d_status, double* d_pivval,
                                double* const* d_xdiag, const int* d_ldx, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  const size_t smem = (2 * 64 * 65 + 64) * sizeof(double);
  static FuncAttrs fa, fa_rl;
  static const int variant = getenv("SGF_DIAG_CHOL") ? atoi(getenv("SGF_DIAG_CHOL")) : 2;
  if (variant == 2) {
    count_launch(); diag_chol_reg_kernel<<<ntasks, 256, 0, s>>>(d_tasks, d_status, d_pivval, d_xdiag, d_ldx);
    return cudaGetLastError();
  }
  if (variant == 1) {
    cudaError_t e = ensure_smem(diag_chol_rl_kernel, smem, fa_rl);
    if (e != cudaSuccess) return e;
    count_launch(); diag_chol_rl_kernel<<<ntasks, 256, smem, s>>>(d_tasks, d_status, d_pivval, d_xdiag, d_ldx);
    return cudaGetLastError();
  }
  cudaError_t e = ensure_smem(diag_chol_kernel, smem, fa);
  if (e != cudaSuccess) return e;
  count_launch(); diag_chol_kernel<<<ntasks, 256, smem, s>>>(d_tasks, d_status, d_pivval, d_xdiag, d_ldx);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Tiled copies: 32x32 tiles through shared memory, so both the read and the
// write are coalesced whatever the two layouts are.  A CTA copies CP_TILES
// consecutive tiles: the task of the first one is found by binary search over
// the per-task tile prefix (a chain of dependent L2 loads -- once per tile it
// bounded the merges at ~3 TB/s), the following ones by walking forward.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int find_task(const long long* prefix, int ntasks, long long tile) {
  int lo = 0, hi = ntasks - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

constexpr int CP_TILES = 8;

__global__ void __launch_bounds__(256) copy_kernel(const CopyTask* __restrict__ tasks,
                                                   const long long* __restrict__ prefix, int ntasks,
                                                   long long ntiles) {
  __shared__ double buf[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (long long t0 = (long long)blockIdx.x * CP_TILES; t0 < ntiles; t0 += (long long)gridDim.x * CP_TILES) {
    const long long t1 = t0 + CP_TILES < ntiles ? t0 + CP_TILES : ntiles;
    int ti = find_task(prefix, ntasks, t0);
    long long start = prefix[ti], next = ti + 1 < ntasks ? prefix[ti + 1] : ntiles;
    for (long long tile = t0; tile < t1; ++tile) {
      while (tile >= next) {  // tasks without tiles have next == start
        ++ti;
        start = next;
        next = ti + 1 < ntasks ? prefix[ti + 1] : ntiles;
      }
      const CopyTask T = tasks[ti];
      const long long local = tile - start;
      const int tcols = (T.cols + 31) / 32;
      const int r0 = (int)(local / tcols) * 32, c0 = (int)(local % tcols) * 32;
      const bool src_rowc = (T.s_cs == 1);  // columns contiguous in the source
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = ty + 8 * u;
        const int r = src_rowc ? q : tx, c = src_rowc ? tx : q;
        const int gr = r0 + r, gc = c0 + c;
        v[u] = (gr < T.rows && gc < T.cols && !(T.lower && gc > gr))
                   ? T.src[(long long)gr * T.s_rs + (long long)gc * T.s_cs] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = ty + 8 * u;
        buf[src_rowc ? q : tx][src_rowc ? tx : q] = v[u];
      }
      __syncthreads();
      const bool dst_rowc = (T.d_cs == 1);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = ty + 8 * u;
        const int r = dst_rowc ? q : tx, c = dst_rowc ? tx : q;
        const int gr = r0 + r, gc = c0 + c;
        if (gr < T.rows && gc < T.cols) T.dst[(long long)gr * T.d_rs + (long long)gc * T.d_cs] = buf[r][c];
      }
      __syncthreads();
    }
  }
}

cudaError_t launch_copy_tiled(const CopyTask* d_tasks, const long long* d_prefix, int ntasks,
                              long long ntiles, cudaStream_t s) {
  if (ntasks <= 0 || ntiles <= 0) return cudaSuccess;
  const long long chunks = (ntiles + CP_TILES - 1) / CP_TILES;
  const long long grid = chunks < (1LL << 30) ? chunks : (1LL << 30);
  count_launch(); copy_kernel<<<(unsigned)grid, 256, 0, s>>>(d_tasks, d_prefix, ntasks, ntiles);
  return cudaGetLastError();
}

// zero the strict upper triangle of square row-major matrices (tiles as copy)
__global__ void __launch_bounds__(256) zero_upper_kernel(const TriTask* __restrict__ tasks,
                                                         const long long* __restrict__ prefix,
                                                         int ntasks, long long ntiles) {
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int ti = find_task(prefix, ntasks, tile);
    const TriTask T = tasks[ti];
    const long long local = tile - prefix[ti];
    const int tc = (T.m + 31) / 32;
    const int r0 = (int)(local / tc) * 32, c0 = (int)(local % tc) * 32;
    if (c0 + 31 <= r0) continue;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int q = ty; q < 32; q += 8) {
      int r = r0 + q, c = c0 + tx;
      if (r < T.m && c < T.m && c > r) T.p[(long long)r * T.ld + c] = 0.0;
    }
  }
}

cudaError_t launch_zero_upper(const void* d_tasks, const long long* d_prefix, int ntasks, long long ntiles,
                              cudaStream_t s) {
  if (ntasks <= 0 || ntiles <= 0) return cudaSuccess;
  long long grid = ntiles < (1LL << 30) ? ntiles : (1LL << 30);
  count_launch(); zero_upper_kernel<<<(unsigned)grid, 256, 0, s>>>((const TriTask*)d_tasks, d_prefix, ntasks, ntiles);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
__global__ void scatter_values_kernel(const double* __restrict__ vals, const long long* __restrict__ dst,
                                      long long nnz, double* __restrict__ base) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    long long d = dst[e];
    if (d >= 0) base[d] = vals[e];
  }
}

cudaError_t launch_scatter_values(const double* vals, const long long* dst, long long nnz, double* base,
                                  cudaStream_t s) {
  if (nnz <= 0) return cudaSuccess;
  long long blocks = (nnz + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  count_launch(); scatter_values_kernel<<<(unsigned)blocks, 256, 0, s>>>(vals, dst, nnz, base);
  return cudaGetLastError();
}

// CSR -> level-1 blocks (blockmatrix.py:97-144): one thread per row; an entry
// (r, col) goes to block (owner[r], owner[col]) when owner[r] <= owner[col]
// (the other orientation is written by its symmetric partner).
__global__ void __launch_bounds__(256) csr_scatter_kernel(const CsrScatter P) {
  for (long long r = blockIdx.x * 256LL + threadIdx.x; r < P.n; r += (long long)gridDim.x * 256) {
    const int ca = P.owner[r];
    const long long lr = P.local[r];
    const int u0 = P.up_ptr[ca], u1 = P.up_ptr[ca + 1];
    const int ra = P.cell_rank ? P.cell_rank[ca] : 0;
    for (long long e = P.indptr[r]; e < P.indptr[r + 1]; ++e) {
      const int col = P.indices[e];
      const int cb = P.owner[col];
      if (P.cell_rank) {  // a block belongs to the rank of its owned cell, shared-shared to rank 0
        const int rb = P.cell_rank[cb];
        const int ob = ra >= 0 ? ra : (rb >= 0 ? rb : 0);
        if (ob != P.my_rank) continue;
      }
      if (cb == ca) {
        P.base[P.diag_off[ca] + lr * P.size[ca] + P.local[col]] = P.values[e];
      } else if (cb > ca) {
        int j = u0;
        while (j < u1 && P.up_cell[j] != cb) ++j;
        if (j < u1) P.base[P.up_off[j] + lr * P.size[cb] + P.local[col]] = P.values[e];
      }
    }
  }
}

// Symmetry of the CSR matrix (blockmatrix.py:105-113): out[0] = max |A - A^T|
// (a missing mirror counts as 0), out[1] = max |A|, both as the bit patterns
// of non-negative doubles (ordered like the values, so atomicMax applies).
// Column indices are sorted per row.
__global__ void __launch_bounds__(256) sym_check_kernel(long long n, const long long* __restrict__ ip,
                                                        const int* __restrict__ ix, const double* __restrict__ v,
                                                        unsigned long long* __restrict__ out) {
  double asym = 0.0, scale = 0.0;
  bool nonfinite = false;
  for (long long r = blockIdx.x * 256LL + threadIdx.x; r < n; r += (long long)gridDim.x * 256) {
    for (long long e = ip[r]; e < ip[r + 1]; ++e) {
      const int c = ix[e];
      const double a = v[e];
      nonfinite |= !isfinite(a);
      scale = fmax(scale, fabs(a));
      long long lo = ip[c], hi = ip[c + 1];
      while (lo < hi) {  // first index with ix >= r
        const long long mid = (lo + hi) >> 1;
        if (ix[mid] < r) lo = mid + 1;
        else hi = mid;
      }
      const double b = (lo < ip[c + 1] && ix[lo] == r) ? v[lo] : 0.0;
      asym = fmax(asym, fabs(a - b));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
    scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, (unsigned long long)__double_as_longlong(asym));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(scale));
  }
  // NaN / Inf anywhere (fmax above skips NaN): out[2] != 0
  if (__any_sync(0xffffffffu, nonfinite) && (threadIdx.x & 31) == 0) atomicMax(out + 2, 1ULL);
}

cudaError_t launch_sym_check(long long n, const long long* ip, const int* ix, const double* v,
                             unsigned long long* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  count_launch(); sym_check_kernel<<<(unsigned)blocks, 256, 0, s>>>(n, ip, ix, v, out);
  return cudaGetLastError();
}

cudaError_t launch_csr_scatter(const void* params, cudaStream_t s) {
  const CsrScatter& P = *(const CsrScatter*)params;
  if (P.n <= 0) return cudaSuccess;
  long long blocks = (P.n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  count_launch(); csr_scatter_kernel<<<(unsigned)blocks, 256, 0, s>>>(P);
  return cudaGetLastError();
}

// r x r identity blocks (compressed node diagonal, factorization.py:345-346)
__global__ void identity_kernel(double* const* __restrict__ ptrs, const int* __restrict__ sizes) {
  double* p = ptrs[blockIdx.x];
  const int r = sizes[blockIdx.x];
  for (long long i = threadIdx.x; i < (long long)r * r; i += blockDim.x) p[i] = (i / r == i % r) ? 1.0 : 0.0;
}

cudaError_t launch_fill_identity(double* const* d_ptrs, const int* d_sizes, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch(); identity_kernel<<<n, 256, 0, s>>>(d_ptrs, d_sizes);
  return cudaGetLastError();
}

// floor[i] = 1e-14 * max(max_j A_i[j,j], 0)   (densela.py:105)
__global__ void max_diag_kernel(const double* const* __restrict__ ptrs, const int* __restrict__ sizes,
                                const int* __restrict__ ld, double* __restrict__ out) {
  __shared__ double red[256];
  const double* p = ptrs[blockIdx.x];
  const int m = sizes[blockIdx.x], l = ld[blockIdx.x];
  double mx = 0.0;
  bool any = false;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double v = p[(long long)i * l + i];
    mx = any ? fmax(mx, v) : v;
    any = true;
  }
  red[threadIdx.x] = any ? mx : -INFINITY;
  __syncthreads();
  for (int s2 = 128; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s2]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = 1e-14 * fmax(red[0], 0.0);
}

cudaError_t launch_max_diag(const double* const* d_ptrs, const int* d_sizes, const int* d_ld, int n,
                            double* d_out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch(); max_diag_kernel<<<n, 256, 0, s>>>(d_ptrs, d_sizes, d_ld, d_out);
  return cudaGetLastError();
}

// Diagnostics (SGF_ZERO_STATS): number of all-zero tr x tk tiles of a strided
// view; one CTA per tile, counters[0] += zero tiles, counters[1] += tiles.
__global__ void zero_tiles_kernel(const double* __restrict__ p, long long rs, long long cs, int rows, int cols,
                                  int tr, int tk, unsigned long long* counters) {
  const int ntc = (cols + tk - 1) / tk;
  const int r0 = (blockIdx.x / ntc) * tr, c0 = (blockIdx.x % ntc) * tk;
  int nz = 0;
  for (int e = threadIdx.x; e < tr * tk; e += blockDim.x) {
    const int r = r0 + e / tk, c = c0 + e % tk;
    if (r < rows && c < cols && p[(long long)r * rs + (long long)c * cs] != 0.0) nz = 1;
  }
  nz = __syncthreads_or(nz);
  if (threadIdx.x == 0) {
    if (!nz) atomicAdd(&counters[0], 1ull);
    atomicAdd(&counters[1], 1ull);
  }
}

cudaError_t launch_zero_tiles(const double* p, long long rs, long long cs, int rows, int cols, int tr, int tk,
                              unsigned long long* counters, cudaStream_t s) {
  const long long nt = (long long)((rows + tr - 1) / tr) * ((cols + tk - 1) / tk);
  if (nt <= 0) return cudaSuccess;
  zero_tiles_kernel<<<(unsigned)nt, 128, 0, s>>>(p, rs, cs, rows, cols, tr, tk, counters);
  return cudaGetLastError();
}

}  // namespace sgf

namespace sgf {
// zero a list of byte ranges (the nonzero-flag and row-mask arrays of a
// batch of operand splits: one launch instead of a memset call per operand,
// ~26k calls = ~19 ms of host time at level 2 of 128^3)
__global__ void __launch_bounds__(256) zero_ranges_kernel(const ZeroRange* __restrict__ r, int n) {
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    uint8_t* p = r[i].p;
    const size_t b = r[i].bytes;
    size_t head = (16 - ((uintptr_t)p & 15)) & 15;
    if (head > b) head = b;
    for (size_t k = threadIdx.x; k < head; k += 256) p[k] = 0;
    const size_t nv = (b - head) / 16;
    uint4* q = reinterpret_cast<uint4*>(p + head);
    for (size_t k = threadIdx.x; k < nv; k += 256) q[k] = make_uint4(0, 0, 0, 0);
    for (size_t k = head + nv * 16 + threadIdx.x; k < b; k += 256) p[k] = 0;
  }
}

cudaError_t launch_zero_ranges(const ZeroRange* d_ranges, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  zero_ranges_kernel<<<(unsigned)std::min(n, 1 << 16), 256, 0, s>>>(d_ranges, n);
  return cudaGetLastError();
}
}  // namespace sgf
