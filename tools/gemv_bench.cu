// Standalone harness for the apply GEMV kernels (bandwidth tuning).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1907_03406_b200/csrc \
//        tools/gemv_bench.cu paper_1907_03406_b200/csrc/apply_kernels.cu -o build/gemv_bench
#include <cstdio>
#include <vector>

#include "common.h"

namespace sgf {
unsigned long long g_kernel_launches = 0;
}
using namespace sgf;

int main() {
  // 48 coupling panels of an L3-like elimination: c = 7778 rows, m = 3571 cols
  const int nf = 48, c = 7778, m = 3571;
  for (int ldpad : {0, 1}) {
    const int ld = ldpad ? 3572 : m;
    double *E, *x, *y;
    cudaMalloc(&E, (size_t)nf * c * ld * 8);
    cudaMalloc(&x, (size_t)nf * c * 8);
    cudaMalloc(&y, (size_t)nf * ((c + 255) / 256) * m * 8 + (size_t)nf * c * 8);
    cudaMemset(E, 0, (size_t)nf * c * ld * 8);
    cudaMemset(x, 0, (size_t)nf * c * 8);
    for (int mode : {0, 1}) {
      std::vector<GemvTask> t;
      for (int f = 0; f < nf; ++f) {
        const double* A = E + (size_t)f * c * ld;
        if (mode == 0) {
          for (int r0 = 0; r0 < c; r0 += 64)
            t.push_back(GemvTask{A, ld, x, y + (size_t)f * c, r0, std::min(c, r0 + 64), 0, m, 0});
        } else {
          int nrb = 0;
          for (int r0 = 0; r0 < c; r0 += 256, ++nrb)
            for (int c0 = 0; c0 < m; c0 += 256)
              t.push_back(GemvTask{A, ld, x + (size_t)f * c, y + ((size_t)f * 31 + nrb) * m, r0,
                                   std::min(c, r0 + 256), c0, std::min(m, c0 + 256), 0});
        }
      }
      GemvTask* dt;
      cudaMalloc(&dt, t.size() * sizeof(GemvTask));
      cudaMemcpy(dt, t.data(), t.size() * sizeof(GemvTask), cudaMemcpyHostToDevice);
      launch_gemv(dt, (int)t.size(), mode, 0);
      cudaDeviceSynchronize();
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        launch_gemv(dt, (int)t.size(), mode, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("{\"test\":\"gemv_%s\",\"ld\":%d,\"ms\":%.3f,\"gbs\":%.1f,\"err\":\"%s\"}\n", mode ? "t" : "n", ld, best,
             8.0 * nf * c * m / best / 1e6, cudaGetErrorString(cudaGetLastError()));
      cudaFree(dt);
    }
    cudaFree(E);
    cudaFree(x);
    cudaFree(y);
  }
  return 0;
}
