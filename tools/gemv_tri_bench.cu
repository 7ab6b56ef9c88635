// Triangular GEMV variants (apply sweeps, y = L^{-1} x with L^{-1} lower,
// row-major, ld even): one warp per row (the library kernel) against row
// pairs (i, m-1-i) per warp, whose combined length m+1 keeps every warp
// iteration's loads full.  L2-like batch: 343 matrices of m = 800.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gemv_tri_bench gemv_tri_bench.cu
#include <cstdio>
#include <vector>

struct Task {
  const double* A;
  long long lda;
  const double* x;
  double* y;
  int m;
};

// library form: warp per row, rows r0+warp, +8, ... of a 64-row block
__global__ void __launch_bounds__(256, 8) tri_rows(const Task* __restrict__ tasks, int blocks_per) {
  const Task T = tasks[blockIdx.x / blocks_per];
  const int r0 = (blockIdx.x % blocks_per) * 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = r0 + warp; i < min(T.m, r0 + 64); i += 8) {
    const double2* a = reinterpret_cast<const double2*>(T.A + (long long)i * T.lda);
    const int ke = i + 1, k2 = ke >> 1;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int k = lane;
    for (; k + 96 < k2; k += 128) {
      const double2 a0 = __ldcs(a + k), a1 = __ldcs(a + k + 32), a2 = __ldcs(a + k + 64), a3 = __ldcs(a + k + 96);
      s0 = fma(a0.x, T.x[2 * k], fma(a0.y, T.x[2 * k + 1], s0));
      s1 = fma(a1.x, T.x[2 * k + 64], fma(a1.y, T.x[2 * k + 65], s1));
      s2 = fma(a2.x, T.x[2 * k + 128], fma(a2.y, T.x[2 * k + 129], s2));
      s3 = fma(a3.x, T.x[2 * k + 192], fma(a3.y, T.x[2 * k + 193], s3));
    }
    for (; k < k2; k += 32) {
      const double2 a0 = __ldcs(a + k);
      s0 = fma(a0.x, T.x[2 * k], fma(a0.y, T.x[2 * k + 1], s0));
    }
    if ((ke & 1) && lane == 0) s0 = fma(T.A[(long long)i * T.lda + ke - 1], T.x[ke - 1], s0);
    double s = (s0 + s1) + (s2 + s3);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) T.y[i] = s;
  }
}

// row pairs: warp takes (i, m-1-i); the two rows' 16-byte words are streamed
// as one sequence of length ceil((i+1)/2) + ceil((m-i)/2), 4 loads per lane
__global__ void __launch_bounds__(256, 8) tri_pairs(const Task* __restrict__ tasks, int blocks_per) {
  const Task T = tasks[blockIdx.x / blocks_per];
  const int p0 = (blockIdx.x % blocks_per) * 32;  // 32 pairs per CTA
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npairs = (T.m + 1) / 2;
  for (int p = p0 + warp; p < min(npairs, p0 + 32); p += 8) {
    const int ra = p, rb = T.m - 1 - p;
    const int na = (ra + 2) >> 1;                 // 16-byte words of row a (covers k <= ra, + stored zero)
    const int nb = (rb == ra) ? 0 : (rb + 2) >> 1;
    const double2* a = reinterpret_cast<const double2*>(T.A + (long long)ra * T.lda);
    const double2* b = reinterpret_cast<const double2*>(T.A + (long long)rb * T.lda);
    const int n = na + nb;
    double sa = 0, sb = 0;
    for (int w0 = 0; w0 < n; w0 += 128) {
      double2 v[4];
      int idx[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int w = w0 + lane + 32 * u;
        idx[u] = w;
        v[u] = w < na ? __ldcs(a + w) : (w < n ? __ldcs(b + (w - na)) : make_double2(0.0, 0.0));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int w = idx[u];
        if (w < na) {
          const int k = 2 * w;
          sa = fma(v[u].x, T.x[k], sa);
          if (k + 1 <= ra) sa = fma(v[u].y, T.x[k + 1], sa);
        } else if (w < n) {
          const int k = 2 * (w - na);
          sb = fma(v[u].x, T.x[k], sb);
          if (k + 1 <= rb) sb = fma(v[u].y, T.x[k + 1], sb);
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
      T.y[ra] = sa;
      if (rb != ra) T.y[rb] = sb;
    }
  }
}

int main() {
  for (int m : {800, 512, 2400}) {
    const int nmat = m == 2400 ? 64 : 343, ld = (m + 1) & ~1;
    double *A, *x, *y;
    cudaMalloc(&A, (size_t)nmat * m * ld * 8);
    cudaMalloc(&x, (size_t)nmat * m * 8);
    cudaMalloc(&y, (size_t)nmat * m * 8);
    cudaMemset(A, 0, (size_t)nmat * m * ld * 8);
    cudaMemset(x, 0, (size_t)nmat * m * 8);
    std::vector<Task> h;
    for (int f = 0; f < nmat; ++f) h.push_back(Task{A + (size_t)f * m * ld, ld, x + (size_t)f * m, y + (size_t)f * m, m});
    Task* d;
    cudaMalloc(&d, h.size() * sizeof(Task));
    cudaMemcpy(d, h.data(), h.size() * sizeof(Task), cudaMemcpyHostToDevice);
    const double bytes = 8.0 * nmat * (double)m * (m + 1) / 2;
    const int bpr = (m + 63) / 64, bpp = ((m + 1) / 2 + 31) / 32;
    for (int var = 0; var < 2; ++var) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) {
          if (var == 0) tri_rows<<<nmat * bpr, 256>>>(d, bpr);
          else tri_pairs<<<nmat * bpp, 256>>>(d, bpp);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 10;
      printf("{\"m\":%d,\"nmat\":%d,\"variant\":\"%s\",\"ms\":%.4f,\"gbs\":%.0f,\"err\":\"%s\"}\n", m, nmat,
             var ? "row_pairs" : "row_per_warp", ms, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(A);
    cudaFree(x);
    cudaFree(y);
    cudaFree(d);
  }
  return 0;
}
