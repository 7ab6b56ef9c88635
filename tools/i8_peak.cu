// Issue-rate peak of tcgen05.mma kind::i8 (M=128, K=32) on this B200: one
// CTA per SM, one thread issuing back-to-back MMAs on smem operands into TMEM
// (operand contents irrelevant), for N = 64 / 128 / 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_peak i8_peak.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46);
}

template <int N>
__global__ void __launch_bounds__(128, 1) peak_kernel(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = smem_desc(smem_u32(smem)), db = smem_desc(smem_u32(smem + 16384));
    for (int i = 0; i < iters; ++i)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(i));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&done)));
  }
  asm volatile(
      "{\n\t.reg .pred p;\n\tW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&done)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(N < 32 ? 32 : N));
  if (threadIdx.x == 0 && iters < 0) *sink = 1;
}

template <int N>
static void run(int sms) {
  const int iters = 20000;
  const size_t smem = 48 * 1024;
  cudaFuncSetAttribute(peak_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int* sink;
  cudaMalloc(&sink, 4);
  peak_kernel<N><<<sms, 128, smem>>>(100, sink);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  peak_kernel<N><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = 2.0 * 128 * N * 32 * (double)iters * sms;
  printf("{\"test\":\"tcgen05_i8_issue\",\"M\":128,\"N\":%d,\"K\":32,\"ctas\":%d,\"ms\":%.3f,\"tops\":%.1f,\"err\":\"%s\"}\n", N,
         sms, ms, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64>(sms);
  run<128>(sms);
  run<256>(sms);
  return 0;
}
