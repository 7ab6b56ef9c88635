// Experiment: FP64 GEMM emulated on the INT8 tensor cores (Ozaki scheme I).
// C = A . B^T with A (M x K), B (N x K) in FP64.  Every row of A and of B is
// scaled by a power of two (|x| < 1) and cut into S = 8 signed 7-bit slices,
// x = 2^e sum_t d_t 2^-7t (truncation, exact in FP64).  The products of slice
// pairs (t, u) with t + u <= S + 1 are accumulated exactly in int32 TMEM, one
// accumulator per diagonal d = t + u (8 x 64 columns = all 512 TMEM columns),
// and the epilogue sums 2^-7d S_d in FP64 and applies the row/column scales.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ozaki_test ozaki_test.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
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

constexpr int S = 8;                        // slices per operand
constexpr int BM = 128, BN = 64, KT = 64;   // tile rows / cols, K bytes per stage
constexpr int STAGES = 2;
constexpr int A_TILE = BM * KT, B_TILE = BN * KT;      // one slice tile
constexpr int A_STAGE = S * A_TILE, B_STAGE = S * B_TILE;

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
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
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

// At: [tm][k][t] slice tiles of A (A_TILE bytes each), Bt: [tn][k][u] of B;
// ea, eb: row exponents; C row-major M x N
__global__ void __launch_bounds__(128, 1)
    ozaki_kernel(const int8_t* __restrict__ At, const int8_t* __restrict__ Bt, const int* __restrict__ ea,
                 const int* __restrict__ eb, double* __restrict__ C, int M, int N, int K) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
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
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {  // producer: one bulk copy per operand per stage
    const int8_t* a = At + (size_t)tm * nk * A_STAGE;
    const int8_t* b = Bt + (size_t)tn * nk * B_STAGE;
    for (int k = 0; k < nk; ++k) {
      const int s = k % STAGES;
      if (k >= STAGES) mbar_wait(&empty[s], ((k / STAGES) - 1) & 1);
      mbar_expect_tx(&full[s], A_STAGE + B_STAGE);
      bulk_g2s(sA + s * A_STAGE, a + (size_t)k * A_STAGE, A_STAGE, &full[s]);
      bulk_g2s(sB + s * B_STAGE, b + (size_t)k * B_STAGE, B_STAGE, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    for (int k = 0; k < nk; ++k) {
      const int s = k % STAGES;
      mbar_wait(&full[s], (k / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = smem_u32(sA + s * A_STAGE), b0 = smem_u32(sB + s * B_STAGE);
#pragma unroll
      for (int t = 0; t < S; ++t)
#pragma unroll
        for (int u = 0; u < S - t; ++u) {  // t + u <= S - 1  (slices 1-based: t+u <= S+1)
          const uint32_t acc_col = (uint32_t)(t + u) * BN;
#pragma unroll
          for (int kk = 0; kk < KT / 32; ++kk) {
            const uint64_t da = smem_desc(a0 + t * A_TILE + 2 * kk * (BM * 16), BM * 16, 128);
            const uint64_t db = smem_desc(b0 + u * B_TILE + 2 * kk * (BN * 16), BN * 16, 128);
            // the first product into each diagonal overwrites it
            const bool first = (k == 0) && (kk == 0) && (t == 0 || u == S - 1 - t ? false : false);
            (void)first;
            const uint32_t accum = (k > 0 || kk > 0 || t > 0) ? 1u : (u == 0 ? 0u : 0u);
            // diagonal dd = t+u is first written by the pair (t = 0, u = dd) at k = kk = 0
            const uint32_t acc_flag = (k > 0 || kk > 0 || t > 0) ? 1u : 0u;
            (void)accum;
            mma_i8(tmem + acc_col, da, db, idesc, acc_flag);
          }
        }
      mma_commit(&empty[s]);
    }
    mma_commit(&done);
  }
  mbar_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = tm * BM + warp * 32 + lane;
  const double rs = ldexp(1.0, ea[row]);
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll
    for (int dd = S - 1; dd >= 0; --dd) {  // smallest terms first
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + dd * BN + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      const double sc = ldexp(1.0, -7 * (dd + 2));
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = fma((double)(int32_t)v[j], sc, acc[j]);
    }
    for (int j = 0; j < 16; ++j) {
      const int col = tn * BN + c0 + j;
      C[(size_t)row * N + col] = acc[j] * rs * ldexp(1.0, eb[col]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// host: exponent + slices of a row-major R x K FP64 matrix, tiled [rt][k][t]
static void split_tile(const std::vector<double>& X, int R, int K, int TR, std::vector<int8_t>& out,
                       std::vector<int>& e) {
  const int nk = K / KT;
  out.assign((size_t)S * R * K, 0);
  e.assign(R, 0);
  std::vector<int8_t> sl((size_t)S * K);
  for (int r = 0; r < R; ++r) {
    double mx = 0.0;
    for (int k = 0; k < K; ++k) mx = std::fmax(mx, std::fabs(X[(size_t)r * K + k]));
    int ex = 0;
    if (mx > 0) std::frexp(mx, &ex);  // mx = f 2^ex, f in [0.5, 1): |x| 2^-ex < 1
    e[r] = ex;
    for (int k = 0; k < K; ++k) {
      double v = std::ldexp(X[(size_t)r * K + k], -ex);
      for (int t = 0; t < S; ++t) {
        v *= 128.0;
        const double d = std::trunc(v);
        sl[(size_t)t * K + k] = (int8_t)d;
        v -= d;
      }
    }
    const int rt = r / TR, rr = r % TR;
    for (int k = 0; k < K; ++k)
      for (int t = 0; t < S; ++t) {
        const int kt = k / KT, kb = k % KT, kc = kb / 16, w = kb % 16;
        const size_t tile = (((size_t)rt * nk + kt) * S + t) * (size_t)TR * KT;
        out[tile + kc * (TR * 16) + (rr / 8) * 128 + (rr % 8) * 16 + w] = sl[(size_t)t * K + k];
      }
  }
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 256, N = argc > 2 ? atoi(argv[2]) : 128, K = argc > 3 ? atoi(argv[3]) : 256;
  const bool check = (long long)M * N * K <= (1LL << 32);
  std::mt19937_64 rng(3);
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  std::vector<double> A((size_t)M * K), B((size_t)N * K);
  // rows with a spread of magnitudes (as in Schur complements)
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < K; ++k) A[(size_t)i * K + k] = d(rng) * std::pow(10.0, 3.0 * d(rng));
  for (int j = 0; j < N; ++j)
    for (int k = 0; k < K; ++k) B[(size_t)j * K + k] = d(rng) * std::pow(10.0, 3.0 * d(rng));
  std::vector<int8_t> At, Bt;
  std::vector<int> ea, eb;
  split_tile(A, M, K, BM, At, ea);
  split_tile(B, N, K, BN, Bt, eb);
  int8_t *dA, *dB;
  int *dea, *deb;
  double* dC;
  CK(cudaMalloc(&dA, At.size()));
  CK(cudaMalloc(&dB, Bt.size()));
  CK(cudaMalloc(&dea, M * 4));
  CK(cudaMalloc(&deb, N * 4));
  CK(cudaMalloc(&dC, (size_t)M * N * 8));
  CK(cudaMemcpy(dA, At.data(), At.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bt.data(), Bt.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dea, ea.data(), M * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(deb, eb.data(), N * 4, cudaMemcpyHostToDevice));
  const size_t smem = (size_t)STAGES * (A_STAGE + B_STAGE);
  CK(cudaFuncSetAttribute(ozaki_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(N / BN, M / BM);
  ozaki_kernel<<<grid, 128, smem>>>(dA, dB, dea, deb, dC, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  double maxrel = 0.0, maxrel_dgemm = 0.0;
  if (check) {
    std::vector<double> C((size_t)M * N);
    CK(cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        long double s = 0, sa = 0;
        double sd = 0;
        for (int k = 0; k < K; ++k) {
          const long double p = (long double)A[(size_t)i * K + k] * B[(size_t)j * K + k];
          s += p;
          sa += fabsl(p);
          sd = std::fma(A[(size_t)i * K + k], B[(size_t)j * K + k], sd);
        }
        // error relative to sum |a||b| (the scale of a dot product's rounding)
        maxrel = std::fmax(maxrel, (double)(fabsl(s - C[(size_t)i * N + j]) / sa));
        maxrel_dgemm = std::fmax(maxrel_dgemm, (double)(fabsl(s - sd) / sa));
      }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 5;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) ozaki_kernel<<<grid, 128, smem>>>(dA, dB, dea, deb, dC, M, N, K);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const int pairs = S * (S + 1) / 2;
  printf("{\"M\":%d,\"N\":%d,\"K\":%d,\"checked\":%d,\"max_err_vs_sumabs\":%.3e,\"fp64_fma_err\":%.3e,"
         "\"ms\":%.4f,\"fp64_equiv_tflops\":%.1f,\"int8_tops\":%.1f}\n",
         M, N, K, (int)check, maxrel, maxrel_dgemm, ms, 2.0 * M * N * K / (ms * 1e-3) / 1e12,
         2.0 * pairs * M * N * K / (ms * 1e-3) / 1e12);
  return 0;
}
