// Level-1 coupling lists (precond.h L1Couplings) built on the device from
// the CSR already resident for the block scatter: count per row, CUB scans,
// fill.  Rows of the interiors eliminated at level 1 come in factor order
// (cell order, then the cell's unknown order = bstart[cell] + local[u]).
#include <cub/cub.cuh>

#include "common.h"

namespace sgf {

namespace {

__global__ void l1_count_kernel(long long n, const long long* __restrict__ ip, const int* __restrict__ ix,
                                const int* __restrict__ owner, const int* __restrict__ local,
                                const char* __restrict__ el, const int* __restrict__ bstart, int* __restrict__ rows,
                                int* __restrict__ bcnt, int* __restrict__ fcnt, int* __restrict__ fflag) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x) {
    const int c = owner[u];
    int k = 0;
    if (el[c]) {
      for (long long e = ip[u]; e < ip[u + 1]; ++e) k += owner[ix[e]] != c;
      const int r = bstart[c] + local[u];
      rows[r] = (int)u;
      bcnt[r] = k;
      fcnt[u] = 0;
      fflag[u] = 0;
    } else {
      for (long long e = ip[u]; e < ip[u + 1]; ++e) k += el[owner[ix[e]]] != 0;
      fcnt[u] = k;
      fflag[u] = k > 0;
    }
  }
}

__global__ void l1_fill_kernel(long long n, const long long* __restrict__ ip, const int* __restrict__ ix,
                               const double* __restrict__ vals, const int* __restrict__ owner,
                               const int* __restrict__ local, const char* __restrict__ el,
                               const int* __restrict__ bstart, const int* __restrict__ brp, int* __restrict__ bci,
                               double* __restrict__ bv, const int* __restrict__ fscan, const int* __restrict__ fidx,
                               int* __restrict__ frid, int* __restrict__ frp, int* __restrict__ fci,
                               double* __restrict__ fv, int nf) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n; u += (long long)gridDim.x * blockDim.x) {
    const int c = owner[u];
    if (el[c]) {
      int k = brp[bstart[c] + local[u]];
      for (long long e = ip[u]; e < ip[u + 1]; ++e)
        if (owner[ix[e]] != c) {
          bci[k] = ix[e];
          bv[k++] = vals[e];
        }
    } else if (fidx[u + 1] > fidx[u]) {
      const int r = fidx[u];
      int k = fscan[u];
      frid[r] = (int)u;
      frp[r] = k;
      for (long long e = ip[u]; e < ip[u + 1]; ++e)
        if (el[owner[ix[e]]]) {
          fci[k] = ix[e];
          fv[k++] = vals[e];
        }
    }
    if (u == 0) frp[nf] = fscan[n];
  }
}

inline unsigned grid_n(long long n) {
  long long b = (n + 255) / 256;
  return (unsigned)(b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b));
}

}  // namespace

cudaError_t l1_couplings_count(long long n, int nb, const long long* ip, const int* ix, const int* owner,
                               const int* local, const char* el, const int* bstart, int* rows, int* bcnt, int* fcnt,
                               int* fflag, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  (void)nb;
  count_launch(); l1_count_kernel<<<grid_n(n), 256, 0, s>>>(n, ip, ix, owner, local, el, bstart, rows, bcnt, fcnt,
                                                             fflag);
  return cudaGetLastError();
}

// exclusive scan of in[0..count) into out[0..count] (out[count] = total)
cudaError_t scan_ints(const int* in, int* out, long long count, void* temp, size_t* temp_bytes, cudaStream_t s) {
  return cub::DeviceScan::ExclusiveSum(temp, *temp_bytes, in, out, (int)(count + 1), s);
}

cudaError_t l1_couplings_fill(long long n, const long long* ip, const int* ix, const double* vals, const int* owner,
                              const int* local, const char* el, const int* bstart, const int* brp, int* bci,
                              double* bv, const int* fscan, const int* fidx, int* frid, int* frp, int* fci,
                              double* fv, int nf, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch(); l1_fill_kernel<<<grid_n(n), 256, 0, s>>>(n, ip, ix, vals, owner, local, el, bstart, brp, bci, bv,
                                                            fscan, fidx, frid, frp, fci, fv, nf);
  return cudaGetLastError();
}

}  // namespace sgf
