// Standalone harness for the batched DMMA GEMM (kernel tuning).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1907_03406_b200/csrc \
//        tools/gemm_bench.cu paper_1907_03406_b200/csrc/gemm_dmma.cu -o build/gemm_bench
// Prints TFLOP/s of: one large NT GEMM (Schur-like, beta=1), a batch of
// m=512 problems (L1-like), and the DMMA issue rate vs warps per SM.
#include <cstdio>
#include <vector>

#include "common.h"

namespace sgf {
unsigned long long g_kernel_launches = 0;
}
using namespace sgf;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dmma_rate(double* out, int iters) {
  double c[CH][2];
  double a = threadIdx.x * 1e-3, b = 1.0000001;
  for (int i = 0; i < CH; i++) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; it++)
#pragma unroll
    for (int i = 0; i < CH; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double r = 0;
  for (int i = 0; i < CH; i++) r += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

static float time_gemm(std::vector<GemmTask>& tasks, std::vector<GemmSeg>& segs, int big, int reps) {
  // one product per task, one tile record per task (tile coordinates from
  // the task's origin, in units of the launch's tile shape)
  const int bm = big == 1 ? 128 : 64, bn = big == 1 ? 128 : (big == 2 ? 16 : 64);
  std::vector<GemmTile> tiles(tasks.size());
  for (size_t i = 0; i < tasks.size(); ++i) {
    tiles[i] = GemmTile{(uint32_t)i, (uint16_t)(tasks[i].m0 / bm), (uint16_t)(tasks[i].n0 / bn)};
    tasks[i].m0 = tasks[i].n0 = 0;
  }
  GemmTask* dt; GemmSeg* ds; GemmTile* dtl;
  cudaMalloc(&dt, tasks.size() * sizeof(GemmTask));
  cudaMalloc(&dtl, tiles.size() * sizeof(GemmTile));
  cudaMalloc(&ds, segs.size() * sizeof(GemmSeg));
  cudaMemcpy(dt, tasks.data(), tasks.size() * sizeof(GemmTask), cudaMemcpyHostToDevice);
  cudaMemcpy(dtl, tiles.data(), tiles.size() * sizeof(GemmTile), cudaMemcpyHostToDevice);
  cudaMemcpy(ds, segs.data(), segs.size() * sizeof(GemmSeg), cudaMemcpyHostToDevice);
  launch_gemm(dt, dtl, (int)tasks.size(), ds, big, 0);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(a);
    launch_gemm(dt, dtl, (int)tasks.size(), ds, big, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  cudaFree(dt); cudaFree(ds); cudaFree(dtl);
  return best;
}

static void tiles(std::vector<GemmTask>& v, double* C, long long ldc, int M, int N, int seg0, int nseg, int bm,
                  double alpha, double beta) {
  for (int m0 = 0; m0 < M; m0 += bm)
    for (int n0 = 0; n0 < N; n0 += bm) {
      GemmTask t; t.C = C; t.c_rs = ldc; t.c_cs = 1; t.M = M; t.N = N; t.m0 = m0; t.n0 = n0;
      t.seg0 = seg0; t.nseg = nseg; t.alpha = alpha; t.beta = beta; v.push_back(t);
    }
}

int main(int argc, char** argv) {
  const bool only64 = argc > 1;
  double* out; CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {1, 2, 4, 8, 16}) {
    if (only64) break;
    int iters = 4000;
    dmma_rate<8><<<148, 32 * warps>>>(out, 10);
    cudaEventRecord(e0);
    dmma_rate<8><<<148, 32 * warps>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"test\":\"dmma_rate\",\"warps_per_sm\":%d,\"tflops\":%.2f}\n", warps,
           2.0 * 256 * 8 * iters * 148.0 * warps / ms / 1e9);
  }
  // large NT GEMM: C(MxN) += A(MxK) B(NxK)^T, all k-contiguous
  const int M = 7680, N = 7680, K = 3584;
  double *A, *B, *C;
  CK(cudaMalloc(&A, (size_t)M * K * 8)); CK(cudaMalloc(&B, (size_t)N * K * 8)); CK(cudaMalloc(&C, (size_t)M * N * 8));
  cudaMemset(A, 0, (size_t)M * K * 8); cudaMemset(B, 0, (size_t)N * K * 8); cudaMemset(C, 0, (size_t)M * N * 8);
  for (int big : {1, 0}) {
    if (only64 && big) continue;
    std::vector<GemmTask> t; std::vector<GemmSeg> s;
    GemmSeg g; g.A = A; g.B = B; g.a_rs = K; g.a_ks = 1; g.b_rs = K; g.b_ks = 1; g.K = K; g.flags = 0;
    s.push_back(g);
    tiles(t, C, N, M, N, 0, 1, big ? 128 : 64, -1.0, 1.0);
    float ms = time_gemm(t, s, big, only64 ? 0 : 3);
    if (only64) return 0;
    printf("{\"test\":\"nt_large\",\"tile\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", big ? 128 : 64, ms,
           2.0 * M * N * K / ms / 1e9);
  }
  // transposed-B layout (B(j,k) j-contiguous), e.g. TRTRI / compression
  for (int big : {1, 0}) {
    std::vector<GemmTask> t; std::vector<GemmSeg> s;
    GemmSeg g; g.A = A; g.B = B; g.a_rs = K; g.a_ks = 1; g.b_rs = 1; g.b_ks = N; g.K = K; g.flags = 0;
    s.push_back(g);
    tiles(t, C, N, M, N, 0, 1, big ? 128 : 64, 1.0, 0.0);
    float ms = time_gemm(t, s, big, 3);
    printf("{\"test\":\"nn_large\",\"tile\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", big ? 128 : 64, ms,
           2.0 * M * N * K / ms / 1e9);
  }
  // batch of 512-wide panels (L1-like: c=384 rows, m=512)
  {
    const int nb = 400, c = 384, m = 512;
    double *E, *X, *O;
    CK(cudaMalloc(&E, (size_t)nb * c * m * 8)); CK(cudaMalloc(&X, (size_t)nb * m * m * 8));
    CK(cudaMalloc(&O, (size_t)nb * c * m * 8));
    cudaMemset(E, 0, (size_t)nb * c * m * 8); cudaMemset(X, 0, (size_t)nb * m * m * 8);
    for (int big : {1, 0}) {
      std::vector<GemmTask> t; std::vector<GemmSeg> s;
      for (int i = 0; i < nb; i++) {
        GemmSeg g; g.A = E + (size_t)i * c * m; g.B = X + (size_t)i * m * m; g.a_rs = m; g.a_ks = 1;
        g.b_rs = m; g.b_ks = 1; g.K = m; g.flags = 0;
        s.push_back(g);
        tiles(t, O + (size_t)i * c * m, m, c, m, i, 1, big ? 128 : 64, 1.0, 0.0);
      }
      float ms = time_gemm(t, s, big, 3);
      printf("{\"test\":\"batch512\",\"tile\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", big ? 128 : 64, ms,
             2.0 * nb * c * m * m / ms / 1e9);
    }
  }
  return 0;
}
