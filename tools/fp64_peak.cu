// FP64 peak microbenchmark for B200 (sm_100a): DFMA (CUDA cores) and DMMA
// (mma.sync f64 -> SASS DMMA.8x8x4) issue throughput. Used to fix the FP64
// roofline denominator, which MEASURED_PEAKS.json does not carry.
#include <cstdio>
#include <cuda_runtime.h>

#define CHK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_loop(double* out, int iters, double s) {
  double a[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) a[i] = fma(a[i], s, 1e-9);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int CH>
__global__ void dmma_loop(double* out, int iters, double s) {
  double c[CH][2];
  double a = threadIdx.x * 1e-3, b = s;
#pragma unroll
  for (int i = 0; i < CH; i++) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) r += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CHK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CHK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out;
  CHK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int tpb : {256, 512, 1024}) {
    int blocks = nsm * (2048 / tpb);
    dfma_loop<8><<<blocks, tpb>>>(out, 100, 1.0000001);
    CHK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; r++) {
      cudaEventRecord(e0);
      dfma_loop<8><<<blocks, tpb>>>(out, iters, 1.0000001);
      cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("{\"kind\":\"dfma\",\"tpb\":%d,\"tflops\":%.2f}\n", tpb, flops / best / 1e9);
  }
  for (int tpb : {128, 256, 512}) {
    int blocks = nsm * 4;
    dmma_loop<8><<<blocks, tpb>>>(out, 100, 1.0000001);
    CHK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; r++) {
      cudaEventRecord(e0);
      dmma_loop<8><<<blocks, tpb>>>(out, iters, 1.0000001);
      cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 256 * 8 * iters * (double)blocks * (tpb / 32);
    printf("{\"kind\":\"dmma\",\"tpb\":%d,\"tflops\":%.2f}\n", tpb, flops / best / 1e9);
  }
  printf("{\"sm\":%d,\"clock_khz\":%d}\n", nsm, clk);
  return 0;
}
