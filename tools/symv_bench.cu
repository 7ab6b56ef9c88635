// Level-1 symmetric GEMV of apply_inverse (y = G x from the lower triangle):
// register-staged library kernel (SGF_SYMV=0) against the bulk-copy staged
// one (SGF_SYMV=1), bitwise comparison and device time.  cfg4-like batch:
// 3375 matrices of m = 512.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1907_03406_b200/csrc -o symv_bench symv_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1907_03406_b200/csrc/apply_kernels.cu"

namespace sgf {
unsigned long long g_kernel_launches = 0;
}

int main(int argc, char** argv) {
  const int nm = argc > 1 ? atoi(argv[1]) : 3375, m = argc > 2 ? atoi(argv[2]) : 512;
  const long long ld = (m + 1) & ~1;
  const size_t per = (size_t)m * ld;
  double *G, *x, *y0, *y1, *base;
  cudaMalloc(&G, per * nm * 8);
  cudaMalloc(&x, (size_t)m * nm * 8);
  cudaMalloc(&base, (size_t)m * nm * 8);
  cudaMalloc(&y0, (size_t)m * nm * 8);
  cudaMalloc(&y1, (size_t)m * nm * 8);
  {
    std::vector<double> h(per);
    srand(1);
    for (auto& v : h) v = rand() / (double)RAND_MAX - 0.5;
    for (int i = 0; i < nm; ++i) cudaMemcpy(G + per * i, h.data(), per * 8, cudaMemcpyHostToDevice);
    std::vector<double> hx((size_t)m * nm);
    for (auto& v : hx) v = rand() / (double)RAND_MAX - 0.5;
    cudaMemcpy(x, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(base, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice);
  }
  std::vector<sgf::SymvTask> t(nm);
  for (int i = 0; i < nm; ++i) t[i] = sgf::SymvTask{G + per * i, ld, x + (size_t)m * i, base + (size_t)m * i, nullptr, m, -1.0};
  sgf::SymvTask *d0, *d1;
  cudaMalloc(&d0, nm * sizeof(sgf::SymvTask));
  cudaMalloc(&d1, nm * sizeof(sgf::SymvTask));
  for (int i = 0; i < nm; ++i) t[i].y = y0 + (size_t)m * i;
  cudaMemcpy(d0, t.data(), nm * sizeof(t[0]), cudaMemcpyHostToDevice);
  for (int i = 0; i < nm; ++i) t[i].y = y1 + (size_t)m * i;
  cudaMemcpy(d1, t.data(), nm * sizeof(t[0]), cudaMemcpyHostToDevice);
  const double bytes = 8.0 * nm * ((double)m * (m + 1) / 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int v = 0; v < 2; ++v) {
    setenv("SGF_SYMV", v ? "1" : "0", 1);
    // the variant is latched per process in launch_symv: call the templates directly
    auto run = [&]() {
      if (v == 0) return sgf::symv_q<8>(d0, nm, 0);
      return sgf::symv_bulk_q<8, 2>(d1, nm, 0);
    };
    for (int w = 0; w < 3; ++w) run();
    cudaDeviceSynchronize();
    const int reps = 20;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) run();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"variant\": \"%s\", \"nm\": %d, \"m\": %d, \"us\": %.1f, \"GBs\": %.0f, \"err\": \"%s\"}\n",
           v ? "bulk" : "regs", nm, m, 1e3 * ms / reps, bytes / (1e6 * ms / reps), cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<double> h0((size_t)m * nm), h1((size_t)m * nm);
  cudaMemcpy(h0.data(), y0, h0.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(h1.data(), y1, h1.size() * 8, cudaMemcpyDeviceToHost);
  printf("{\"bitwise_equal\": %s}\n", memcmp(h0.data(), h1.data(), h0.size() * 8) == 0 ? "true" : "false");
  return 0;
}
