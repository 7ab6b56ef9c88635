// Unit test of OzBatch (ozaki.cu via libsgf.so): split + batched emulated
// FP64 products against a long-double reference, with partial tiles,
// transposed operands, several segments per block, lower-only and
// triangular-B tiles, and graded operands:
//   grade 0  entries 10^U[-2,2]
//   grade 1  rows scaled by 10^U[-8,8] (each row of A and of B)
//   grade 2  columns k of A and of B both scaled by 10^v_k, v ~ U[-8,8]
//            (entries within a row span 10^+-8, large terms aligned in k)
//   grade 3  columns of A scaled by 10^v_k, of B by 10^-v_k (within-row
//            span 10^+-8, maxima misaligned: the adversarial case of any
//            row-scaled Ozaki scheme)
// Gates: every case within the scheme's bound 4 K 2^-62 max|A_i| max|B_j|
// (+ FP64 accumulation); grades 0-2 also within the componentwise FP64 bound
// gamma_K sum_k |a_ik||b_jk| (gamma_K = K u / (1 - K u), u = 2^-53); grade 3
// reports its ratio to that bound (it exceeds it: the row maxima the digits
// are cut against are far above the aligned products).
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

// apply the grading of a case to an R x K row-major operand (sign: +1 for A, -1 for B)
static void grade_op(std::vector<double>& X, int R, int K, int grade, const std::vector<double>& colv, int side) {
  std::uniform_real_distribution<double> u(-8.0, 8.0);
  if (grade == 1)
    for (int i = 0; i < R; ++i) {
      const double f = std::pow(10.0, u(rng));
      for (int k = 0; k < K; ++k) X[(size_t)i * K + k] *= f;
    }
  if (grade == 2 || grade == 3)
    for (int i = 0; i < R; ++i)
      for (int k = 0; k < K; ++k) X[(size_t)i * K + k] *= std::pow(10.0, (grade == 3 && side < 0 ? -1 : 1) * colv[k]);
}

int main() {
  cudaStream_t st;
  cudaStreamCreate(&st);
  Arena mem(st);
  int fails = 0;
  struct Case {
    int M, N, K;
    bool transA, lower, tri, two;
    int grade;
  };
  const Case cases[] = {{128, 64, 64, false, false, false, false, 0},  {200, 150, 300, false, false, false, true, 0},
                        {257, 257, 190, true, true, false, true, 0},    {96, 130, 130, false, false, true, false, 0},
                        {512, 384, 1000, true, false, false, true, 0}, {300, 300, 129, false, true, true, false, 0},
                        {256, 256, 1024, false, false, false, false, 1}, {256, 200, 2048, true, false, false, true, 1},
                        {256, 256, 1024, false, false, false, false, 2}, {300, 256, 3000, true, false, false, false, 2},
                        {256, 256, 1024, false, false, false, false, 3}};
  for (const Case& c : cases) {
    const int M = c.M, N = c.N, K = c.K;
    const double spread = c.grade ? 0.3 : 2.0;
    auto A1 = rnd((size_t)M * K, spread), B1 = rnd((size_t)N * K, spread), A2 = rnd((size_t)M * K, spread),
         B2 = rnd((size_t)N * K, spread), C0 = rnd((size_t)M * N, 1.0);
    if (c.grade) {
      std::uniform_real_distribution<double> u(-8.0, 8.0);
      std::vector<double> colv(K);
      for (auto& v : colv) v = u(rng);
      grade_op(A1, M, K, c.grade, colv, +1);
      grade_op(A2, M, K, c.grade, colv, +1);
      grade_op(B1, N, K, c.grade, colv, -1);
      grade_op(B2, N, K, c.grade, colv, -1);
      for (auto& x : C0) x = 0.0;  // C holds the product alone (its scale varies per row)
    }
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
    double worst = 0.0, worst_fp64 = 0.0;
    const double uu = 0x1p-53, gamma = K * uu / (1.0 - K * uu);
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        if (c.lower && (j / 128) * 128 >= (i / 128) * 128 + 128) continue;  // tiles above the diagonal are skipped
        long double s = C0[(size_t)i * N + j], sa = std::fabs(C0[(size_t)i * N + j]);
        double ma = 0, mb = 0, ma2 = 0, mb2 = 0;  // the scheme's error scale: K max|A_i| max|B_j| 2^-62
        for (int k = 0; k < K; ++k) {
          ma = std::fmax(ma, std::fabs(A1[(size_t)i * K + k]));
          mb = std::fmax(mb, std::fabs(B1[(size_t)j * K + k]));
          if (c.two) {
            ma2 = std::fmax(ma2, std::fabs(A2[(size_t)i * K + k]));
            mb2 = std::fmax(mb2, std::fabs(B2[(size_t)j * K + k]));
          }
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
        // bound of the scheme: truncated digits (2^-62 of each row maximum) and the
        // dropped pairs contribute at most ~4 K 2^-62 max|A_i| max|B_j|; the FP64
        // epilogue a few ulps of sum |a||b|
        const double err = (double)fabsl(s - C[(size_t)i * N + j]);
        worst = std::fmax(worst, err / (4.0 * K * (ma * mb + 0.5 * ma2 * mb2) * 0x1p-62 + 4e-16 * (double)sa));
        worst_fp64 = std::fmax(worst_fp64, err / (gamma * (double)sa + 1e-300));
      }
    const bool ok = worst <= 1.0 && (c.grade == 3 || worst_fp64 <= 1.0);
    fails += !ok;
    printf("{\"M\":%d,\"N\":%d,\"K\":%d,\"transA\":%d,\"lower\":%d,\"tri\":%d,\"two\":%d,\"grade\":%d,"
           "\"err_over_scheme_bound\":%.3e,\"err_over_fp64_gamma_K_bound\":%.3e,\"ok\":%d}\n",
           M, N, K, c.transA, c.lower, c.tri, c.two, c.grade, worst, worst_fp64, ok);
  }
  // timing: Schur-like batches (two products per tile at K = 1664; four at
  // K = 640, where the epilogue weighs as it does under the block-sparse K lists)
  for (int tcase = 0; tcase < 2; ++tcase) {
    const int M = 4096, N = 4096, K = tcase == 0 ? 1664 : 640, nprod = tcase == 0 ? 2 : 4;
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
      std::vector<std::pair<std::pair<OzOperand, OzOperand>, double>> terms;
      for (int q = 0; q < nprod; ++q) terms.push_back({{a, b}, q % 2 ? 1.0 : -1.0});
      oz.add(dC, N, 1, M, N, 1.0, terms, false, false);
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
      printf("{\"timing\":\"%d products per 128x128 tile\",\"M\":%d,\"N\":%d,\"K\":%d,\"ms\":%.3f,\"fp64_tflops\":%.1f,"
             "\"int8_tops\":%.0f}\n", nprod, M, N, K, ms, useful / (ms * 1e-3) / 1e12, 36 * useful / (ms * 1e-3) / 1e12);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("cuda: %s, failures: %d\n", cudaGetErrorString(e), fails);
  return fails || e != cudaSuccess;
}
