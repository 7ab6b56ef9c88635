// Experiment: INT8 GEMM on the 5th-generation tensor cores (tcgen05.mma
// kind::i8, int32 accumulators in TMEM), the building block for FP64 GEMM
// emulation (Ozaki scheme).  C[M x N] (int32) = A[M x K] . B[N x K]^T, both
// operands int8 and pre-tiled on the host into the UMMA canonical K-major,
// no-swizzle layout (8-row x 16-byte core matrices), so one bulk copy
// (cp.async.bulk, mbarrier complete_tx) moves a whole stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8gemm_test i8gemm_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int BM = 128, BN = 128, KT = 64;  // tile rows, tile cols, K bytes per stage
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * KT, B_BYTES = BN * KT;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// K-major, no swizzle: LBO = distance between the two 16-byte K chunks of a
// row (one K=32 MMA step), SBO = distance between 8-row core-matrix groups
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  return d;                // base offset 0, layout SWIZZLE_NONE (0)
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}

__global__ void __launch_bounds__(128, 1)
    i8gemm_kernel(const int8_t* __restrict__ At, const int8_t* __restrict__ Bt, int32_t* __restrict__ C, int M, int N,
                  int K) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tm = blockIdx.y, tn = blockIdx.x;
  const int nk = K / KT;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {  // producer
    const int8_t* a = At + (size_t)tm * nk * A_BYTES;
    const int8_t* b = Bt + (size_t)tn * nk * B_BYTES;
    for (int k = 0; k < nk; ++k) {
      const int s = k % STAGES;
      if (k >= STAGES) mbar_wait(&empty[s], ((k / STAGES) - 1) & 1);
      mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
      bulk_g2s(sA + s * A_BYTES, a + (size_t)k * A_BYTES, A_BYTES, &full[s]);
      bulk_g2s(sB + s * B_BYTES, b + (size_t)k * B_BYTES, B_BYTES, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    // kind::i8: D s32 (bits 4-5 = 2), A/B signed (bits 7-9, 10-12 = 1), K-major,
    // N >> 3 at bit 17, M >> 4 at bit 24
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    for (int k = 0; k < nk; ++k) {
      const int s = k % STAGES;
      mbar_wait(&full[s], (k / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
      for (int kk = 0; kk < KT / 32; ++kk) {
        // tile layout: byte(r, kc) = kc * (R*16) + (r/8)*128 + (r%8)*16
        const uint64_t da = smem_desc(a0 + 2 * kk * (BM * 16), BM * 16, 128);
        const uint64_t db = smem_desc(b0 + 2 * kk * (BN * 16), BN * 16, 128);
        mma_i8(tmem, da, db, idesc, (k | kk) ? 1u : 0u);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(&done);
  }
  // epilogue: all 4 warps, warp w owns TMEM lanes 32w..32w+31 (= rows)
  mbar_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = tm * BM + warp * 32 + lane;
#pragma unroll
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (row < M)
      for (int j = 0; j < 16; ++j) C[(size_t)row * N + tn * BN + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
}

// host: pre-tile a row-major R x K int8 matrix (R multiple of the tile rows)
static void tile_kmajor(const std::vector<int8_t>& X, int R, int K, int TR, std::vector<int8_t>& out) {
  const int nk = K / KT;
  out.assign((size_t)R * K, 0);
  for (int tr = 0; tr < R / TR; ++tr)
    for (int k = 0; k < nk; ++k) {
      int8_t* t = out.data() + ((size_t)tr * nk + k) * TR * KT;
      for (int r = 0; r < TR; ++r)
        for (int kb = 0; kb < KT; ++kb) {
          const int kc = kb / 16, w = kb % 16;
          t[kc * (TR * 16) + (r / 8) * 128 + (r % 8) * 16 + w] = X[(size_t)(tr * TR + r) * K + k * KT + kb];
        }
    }
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 256, N = argc > 2 ? atoi(argv[2]) : 256, K = argc > 3 ? atoi(argv[3]) : 256;
  const bool check = M * (long long)N * K <= (1LL << 33);
  std::mt19937 rng(1);
  std::uniform_int_distribution<int> d(-127, 127);
  std::vector<int8_t> A((size_t)M * K), B((size_t)N * K), At, Bt;
  for (auto& v : A) v = (int8_t)d(rng);
  for (auto& v : B) v = (int8_t)d(rng);
  tile_kmajor(A, M, K, BM, At);
  tile_kmajor(B, N, K, BN, Bt);
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, At.size()));
  CK(cudaMalloc(&dB, Bt.size()));
  CK(cudaMalloc(&dC, (size_t)M * N * 4));
  CK(cudaMemcpy(dA, At.data(), At.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bt.data(), Bt.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0, (size_t)M * N * 4));
  const size_t smem = (size_t)STAGES * (A_BYTES + B_BYTES);
  CK(cudaFuncSetAttribute(i8gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(N / BN, M / BM);
  i8gemm_kernel<<<grid, 128, smem>>>(dA, dB, dC, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  long long bad = 0;
  if (check) {
    std::vector<int32_t> C((size_t)M * N);
    CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        long long s = 0;
        for (int k = 0; k < K; ++k) s += (int)A[(size_t)i * K + k] * (int)B[(size_t)j * K + k];
        if (s != C[(size_t)i * N + j]) {
          if (bad < 5) printf("mismatch (%d,%d): %lld vs %d\n", i, j, s, C[(size_t)i * N + j]);
          ++bad;
        }
      }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) i8gemm_kernel<<<grid, 128, smem>>>(dA, dB, dC, M, N, K);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("{\"M\":%d,\"N\":%d,\"K\":%d,\"checked\":%d,\"mismatches\":%lld,\"ms\":%.4f,\"tops\":%.1f}\n", M, N, K,
         (int)check, bad, ms, 2.0 * M * N * K / (ms * 1e-3) / 1e12);
  return bad ? 1 : 0;
}
