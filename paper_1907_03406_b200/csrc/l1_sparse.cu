// Level-1 eliminations with sparse couplings.
//
// At level 1 nothing has been eliminated yet, so the coupling block A_NB of an
// interior B with a neighbour N still holds the original matrix entries: for a
// 5/7-point stencil every row of A_NB has at most one nonzero.  The
// reference's dense products (factorization.py:285-293)
//   E_N   = A_NB L^{-T}                       (c x m per interior)
//   S_ab  = E_a E_b^T = A_aB G A_bB^T,  G = L^{-T} L^{-1} = A_BB^{-1}
// are then gathers: row r of E_N is sum_t a_rt X[:, k_rt] (X = L^{-1}), and a
// Schur entry is sum_{t,u} a_rt a_su G[k_rt, k_su].  G is formed for the
// level-1 apply anyway (precond.h L1Couplings), so the level's two largest
// DMMA GEMMs become two memory-bound kernels.  The flop tally is unchanged
// (it is the reference's analytic count of the dense operations).
//
// l1_rows_kernel: the nonzeros of every coupling row, sorted by column (row
// lists: count, columns, values), from a coalesced pass over the block;
// l1_e_kernel: E rows from the row lists and tiles of L^{-1} in shared memory.
// l1_schur_kernel: one CTA per target block; every entry sums its
// contributors in ascending interior order, then C -= sum (diagonal targets:
// lower triangle only), the accumulation of the target-centric DMMA path.
#include "common.h"

namespace sgf {

namespace {

// Row lists of one coupling block A_NB (rows of N, columns of the interior),
// read in its stored orientation with coalesced loads: stored (N, B) is
// A_NB itself, stored (B, N) its transpose.  Each nonzero lands in its row's
// list through an atomic slot; every list is then sorted by column, so the
// lists (and everything summed from them) do not depend on the slot order.
__global__ void __launch_bounds__(256) l1_rows_kernel(const L1RowTask* __restrict__ tasks, int* __restrict__ rl_n,
                                                      int* __restrict__ rl_k, double* __restrict__ rl_a,
                                                      int* __restrict__ overflow) {
  const L1RowTask T = tasks[blockIdx.x];
  const long long total = (long long)T.srows * T.scols;
  for (long long e = threadIdx.x; e < total; e += 256) {
    const double v = T.p[e];
    if (v == 0.0) continue;
    const int i = (int)(e / T.scols), j = (int)(e % T.scols);
    const int r = T.trans ? j : i, k = T.trans ? i : j;
    const long long row = T.rl0 + r;
    const int slot = atomicAdd(&rl_n[row], 1);
    if (slot < L1_KMAX) {
      rl_k[row * L1_KMAX + slot] = k;
      rl_a[row * L1_KMAX + slot] = v;
    } else {
      atomicExch(overflow, 1);
    }
  }
  __syncthreads();
  const int nr = T.trans ? T.scols : T.srows;
  for (int r = threadIdx.x; r < nr; r += 256) {
    const long long row = T.rl0 + r;
    const int n = min(rl_n[row], L1_KMAX);
    int* k = rl_k + row * L1_KMAX;
    double* a = rl_a + row * L1_KMAX;
    for (int x = 1; x < n; ++x) {  // insertion sort by column
      const int kx = k[x];
      const double ax = a[x];
      int y = x - 1;
      for (; y >= 0 && k[y] > kx; --y) {
        k[y + 1] = k[y];
        a[y + 1] = a[y];
      }
      k[y + 1] = kx;
      a[y + 1] = ax;
    }
  }
}

// E rows of one interior, 16 columns per CTA: E[r, j] = sum_t a_rt X[j, k_rt]
// with X[j0..j0+16) staged in shared memory (odd pitch: the 16 threads of a
// row read one column of the tile without bank conflicts) and the interior's
// row lists copied to shared memory once (coalesced), so the row loop runs
// from shared memory; half-warps write 128-byte row segments of E.
constexpr int L1E_TJ = 16;
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__global__ void __launch_bounds__(256) l1_e_kernel(const L1ETask* __restrict__ tasks, const int* __restrict__ rl_n,
                                                   const int* __restrict__ rl_k, const double* __restrict__ rl_a,
                                                   int max_m) {
  extern __shared__ double xt[];
  const L1ETask T = tasks[blockIdx.x];
  const int j0 = blockIdx.y * L1E_TJ;
  if (j0 >= T.m) return;
  const int nj = min(L1E_TJ, T.m - j0);
  const int kend = min(T.m, j0 + L1E_TJ);  // X[j, k] = 0 for k > j
  const int pitch = T.m | 1;
  double* sa = xt + L1E_TJ * (max_m | 1);
  int* sk = reinterpret_cast<int*>(sa + (long long)T.c * L1_KMAX);
  int* sn = sk + T.c * L1_KMAX;
  // asynchronous copies (cp.async): all of a thread's loads in flight at once
  for (int t = 0; t < nj; ++t)
    for (int k = threadIdx.x; k < kend; k += 256) cp_async8(xt + t * pitch + k, T.X + (long long)(j0 + t) * T.ldx + k);
  for (int i = threadIdx.x; i < T.c * L1_KMAX; i += 256) {
    cp_async8(sa + i, rl_a + T.rl0 * L1_KMAX + i);
    cp_async4(sk + i, rl_k + T.rl0 * L1_KMAX + i);
  }
  for (int i = threadIdx.x; i < T.c; i += 256) cp_async4(sn + i, rl_n + T.rl0 + i);
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int t = threadIdx.x & 15;
  for (int r = threadIdx.x >> 4; r < T.c; r += 16) {
    const int n = min(sn[r], L1_KMAX);
    double s = 0.0;
    for (int u = 0; u < n; ++u) {
      const int k = sk[r * L1_KMAX + u];
      if (k < kend) s = fma(sa[r * L1_KMAX + u], xt[t * pitch + k], s);
    }
    if (t < nj) T.E[(long long)r * T.lde + j0 + t] = s;
  }
}

__device__ __forceinline__ double gsym(const double* G, long long ld, int k, int l) {
  return k >= l ? G[(long long)k * ld + l] : G[(long long)l * ld + k];
}

__global__ void __launch_bounds__(256) l1_schur_kernel(const L1SchurTask* __restrict__ tasks,
                                                       const L1Contrib* __restrict__ contrib,
                                                       const int* __restrict__ rl_n, const int* __restrict__ rl_k,
                                                       const double* __restrict__ rl_a) {
  const L1SchurTask T = tasks[blockIdx.x];
  const int r1 = min(T.rows, T.r0 + 64);
  for (int r = T.r0 + (threadIdx.x >> 6); r < r1; r += 4) {
    const int s_end = T.diag ? r + 1 : T.cols;
    for (int s = threadIdx.x & 63; s < s_end; s += 64) {
      double acc = 0.0;
      for (int c = 0; c < T.nc; ++c) {
        const L1Contrib C = contrib[T.c0 + c];
        const long long ra = C.rl_a + r, sb = C.rl_b + s;
        const int na = rl_n[ra], nb = rl_n[sb];
        double u = 0.0;
        for (int t = 0; t < na; ++t) {
          const int k = rl_k[ra * L1_KMAX + t];
          const double a = rl_a[ra * L1_KMAX + t];
          double v = 0.0;
          for (int w = 0; w < nb; ++w)
            v = fma(rl_a[sb * L1_KMAX + w], gsym(C.G, C.ldg, k, rl_k[sb * L1_KMAX + w]), v);
          u = fma(a, v, u);
        }
        acc += u;
      }
      double* cp = T.C + (long long)r * T.ldc + s;
      *cp -= acc;
    }
  }
}

}  // namespace

cudaError_t launch_l1_rows(const L1RowTask* d_tasks, int ntasks, int* rl_n, int* rl_k, double* rl_a, int* overflow,
                           cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  count_launch();
  l1_rows_kernel<<<ntasks, 256, 0, s>>>(d_tasks, rl_n, rl_k, rl_a, overflow);
  return cudaGetLastError();
}

cudaError_t launch_l1_e(const L1ETask* d_tasks, int ntasks, int max_m, int max_c, const int* rl_n, const int* rl_k,
                        const double* rl_a, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  const size_t smem = (size_t)L1E_TJ * (max_m | 1) * sizeof(double) +
                      (size_t)max_c * (L1_KMAX * (sizeof(double) + sizeof(int)) + sizeof(int));
  if (smem > (size_t)220 << 10) return cudaErrorInvalidValue;  // caller checks l1_e_fits
  static FuncAttrs fa;
  cudaError_t e = ensure_smem(l1_e_kernel, smem, fa);
  if (e != cudaSuccess) return e;
  count_launch();
  l1_e_kernel<<<dim3(ntasks, (max_m + L1E_TJ - 1) / L1E_TJ), 256, smem, s>>>(d_tasks, rl_n, rl_k, rl_a, max_m);
  return cudaGetLastError();
}

cudaError_t launch_l1_schur(const L1SchurTask* d_tasks, int ntasks, const L1Contrib* d_contrib, const int* rl_n,
                            const int* rl_k, const double* rl_a, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  count_launch();
  l1_schur_kernel<<<ntasks, 256, 0, s>>>(d_tasks, d_contrib, rl_n, rl_k, rl_a);
  return cudaGetLastError();
}

}  // namespace sgf
