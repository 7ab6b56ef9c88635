// Unit test of OzBatch (ozaki.cu via libsgf.so): split + batched emulated
// FP64 products against a CPU reference, with partial tiles, transposed
// operands, several segments per block, lower-only and triangular-B tiles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_1907_03406_b200/csrc -I include \
//        -o tools/oz_batch_test tools/oz_batch_test.cu -L paper_1907_03406_b200 -lsgf -Xlinker -rpath=$PWD/paper_1907_03406_b200
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "runtime.h"

using namespace sgf;

// present only in the OZ_PROFILE build of libsgf.so
extern "C" int sgf_oz_prof_read(unsigned long long* out, int reset) __attribute__((weak));

static std::mt19937_64 rng(7);

static std::vector<double> rnd(size_t n, double spread) {
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  std::vector<double> v(n);
  for (auto& x : v) x = d(rng) * std::pow(10.0, spread * d(rng));
  return v;
}

int main() {
  cudaStream_t st;
  cudaStreamCreate(&st);
  Arena mem(st);
  int fails = 0;
  struct Case {
    int M, N, K;
    bool transA, lower, tri, two;
  };
  const Case cases[] = {{128, 64, 64, false, false, false, false},  {200, 150, 300, false, false, false, true},
                        {257, 257, 190, true, true, false, true},    {96, 130, 130, false, false, true, false},
                        {512, 384, 1000, true, false, false, true}, {300, 300, 129, false, true, true, false}};
  for (const Case& c : cases) {
    const int M = c.M, N = c.N, K = c.K;
    auto A1 = rnd((size_t)M * K, 2.0), B1 = rnd((size_t)N * K, 2.0), A2 = rnd((size_t)M * K, 2.0),
         B2 = rnd((size_t)N * K, 2.0), C0 = rnd((size_t)M * N, 1.0);
    if (c.tri)  // B lower triangular (N x K with N == K)
      for (int j = 0; j < N; ++j)
        for (int k = j + 1; k < K; ++k) B1[(size_t)j * K + k] = B2[(size_t)j * K + k] = 0.0;
    // device copies; A stored transposed (K x M, column access) when transA
    auto up = [&](const std::vector<double>& h) {
      double* d = mem.alloc(h.size());
      cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      return d;
    };
    std::vector<double> A1s = A1, A2s = A2;
    if (c.transA)
      for (int i = 0; i < M; ++i)
        for (int k = 0; k < K; ++k) {
          A1s[(size_t)k * M + i] = A1[(size_t)i * K + k];
          A2s[(size_t)k * M + i] = A2[(size_t)i * K + k];
        }
    double *dA1 = up(A1s), *dA2 = up(A2s), *dB1 = up(B1), *dB2 = up(B2), *dC = up(C0);
    OzBatch oz;
    const long long ars = c.transA ? 1 : K, acs = c.transA ? M : 1;
    OzOperand a1 = oz.split(mem, dA1, ars, acs, M, K), b1 = oz.split(mem, dB1, K, 1, N, K);
    OzOperand a2 = oz.split(mem, dA2, ars, acs, M, K), b2 = oz.split(mem, dB2, K, 1, N, K);
    oz.launch_splits(mem, st);
    std::vector<std::pair<std::pair<OzOperand, OzOperand>, double>> terms = {{{a1, b1}, -1.0}};
    if (c.two) terms.push_back({{a2, b2}, 0.5});
    oz.add(dC, N, 1, M, N, 1.0, terms, c.lower, c.tri);
    oz.launch(mem, st);
    std::vector<double> C(C0.size());
    cudaStreamSynchronize(st);
    cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
    double worst = 0.0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        if (c.lower && (j / 128) * 128 >= (i / 128) * 128 + 128) continue;  // tiles above the diagonal are skipped
        long double s = C0[(size_t)i * N + j], sa = std::fabs(C0[(size_t)i * N + j]);
        double ma = 0, mb = 0;  // the scheme's error scale: K * max|A_i| * max|B_j| * 2^-56
        for (int k = 0; k < K; ++k) {
          ma = std::fmax(ma, std::fabs(A1[(size_t)i * K + k]));
          mb = std::fmax(mb, std::fabs(B1[(size_t)j * K + k]));
        }
        for (int k = 0; k < K; ++k) {
          const long double p1 = (long double)A1[(size_t)i * K + k] * B1[(size_t)j * K + k];
          s -= p1;
          sa += fabsl(p1);
          if (c.two) {
            const long double p2 = 0.5L * A2[(size_t)i * K + k] * B2[(size_t)j * K + k];
            s += p2;
            sa += fabsl(p2);
          }
        }
        // bound of the scheme: truncated slices and dropped diagonals contribute at most
        // ~50 K 2^-56 max|A_i| max|B_j|; FP64 accumulation a few ulps of sum |a||b|
        worst = std::fmax(worst, (double)(fabsl(s - C[(size_t)i * N + j]) / (64.0 * K * ma * mb * 0x1p-56 + 4e-16 * sa)));
      }
    const bool ok = worst <= 1.0;
    fails += !ok;
    printf("{\"M\":%d,\"N\":%d,\"K\":%d,\"transA\":%d,\"lower\":%d,\"tri\":%d,\"two\":%d,\"max_err\":%.3e,\"ok\":%d}\n",
           M, N, K, c.transA, c.lower, c.tri, c.two, worst, ok);
  }
  // timing: a Schur-like batch (two products per tile, K = 1664)
  {
    const int M = 4096, N = 4096, K = 1664;
    auto A1 = rnd((size_t)M * K, 1.0), B1 = rnd((size_t)N * K, 1.0);
    double* dA = mem.alloc(A1.size());
    double* dB = mem.alloc(B1.size());
    double* dC = mem.alloc((size_t)M * N);
    cudaMemcpy(dA, A1.data(), A1.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B1.data(), B1.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0, (size_t)M * N * 8);
    OzBatch oz;
    OzOperand a = oz.split(mem, dA, K, 1, M, K), b = oz.split(mem, dB, K, 1, N, K);
    oz.launch_splits(mem, st);
    for (int rep = 0; rep < 2; ++rep) {
      oz.add(dC, N, 1, M, N, 1.0, {{{a, b}, -1.0}, {{a, b}, 1.0}}, false, false);
      const double useful = oz.useful;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      oz.launch(mem, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (sgf_oz_prof_read) {
        unsigned long long c[8];
        sgf_oz_prof_read(c, 1);
        printf("{\"cycles\": {\"mma_wait_operands\": %llu, \"mma_wait_epilogue\": %llu, \"mma_issue\": %llu, "
               "\"epilogue_drain_thread0\": %llu, \"epilogue_wait_thread0\": %llu}}\n", c[0], c[1], c[2], c[3], c[4]);
      }
      printf("{\"timing\":\"2 products per 128x128 tile\",\"M\":%d,\"N\":%d,\"K\":%d,\"ms\":%.3f,\"fp64_tflops\":%.1f,"
             "\"int8_tops\":%.0f}\n", M, N, K, ms, useful / (ms * 1e-3) / 1e12, 36 * useful / (ms * 1e-3) / 1e12);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("cuda: %s, failures: %d\n", cudaGetErrorString(e), fails);
  return fails || e != cudaSuccess;
}
