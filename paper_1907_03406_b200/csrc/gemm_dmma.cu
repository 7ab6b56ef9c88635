// Batched FP64 GEMM on the B200 FP64 tensor path (mma.sync m8n8k4 f64 ->
// SASS DMMA.8x8x4; tcgen05 has no f64 kind on sm_100a).
//
// One CTA computes one output tile of one task.  A task accumulates over a
// list of K-segments, each with its own operand pointers and (row, k)
// strides, so the same kernel serves
//   * the blocked Cholesky / triangular-inverse panel updates,
//   * the coupling solve E = A_NB L^{-T} (as A_NB * (L^{-1})^T, triangular K range),
//   * the target-centric Schur update  A_NiNj -= sum_x E_x[Ni] E_x[Nj]^T
//     (reference factorization.py:288-293, contributors accumulated in
//     ascending interior order inside one tile: no atomics, deterministic),
//   * the compression GEMMs (M_BN Phi_N, L^{-1} X, Q1^T L^{-1} M_BN, WY updates).
// Operands are streamed global -> shared with cp.async (LDGSTS) through a
// 3-stage pipeline; each operand tile is stored [row][k] or [k][row]
// depending on which global stride is unit, with padding chosen so the
// DMMA fragment reads are bank-conflict free in both layouts.
#include "common.h"

namespace sgf {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN>
__device__ __forceinline__ void seg_krange(const GemmSeg& S, int m0, int n0, int& kb, int& ke) {
  kb = 0;
  ke = S.K;
  if (S.flags & SEG_KLIM_M) ke = min(ke, m0 + BM);
  if (S.flags & SEG_KLIM_N) ke = min(ke, n0 + BN);
  if (S.flags & SEG_KSTART_M) kb = max(kb, m0);
  if (S.flags & SEG_KSTART_N) kb = max(kb, n0);
  kb = (kb / 16) * 16;
}

template <int BM, int BN, int WM, int WN, int NT, int STAGES>
__global__ void __launch_bounds__(NT) gemm_f64_kernel(const GemmTask* __restrict__ tasks,
                                                      const GemmSeg* __restrict__ segs) {
  constexpr int BK = 16;
  constexpr int SK = BK + 4;   // [row][k] stride (== 4 mod 16: conflict free)
  constexpr int SMA = BM + 4;  // [k][row] strides
  constexpr int SMB = BN + 4;
  constexpr int A_EL = (BM * SK > BK * SMA) ? BM * SK : BK * SMA;
  constexpr int B_EL = (BN * SK > BK * SMB) ? BN * SK : BK * SMB;
  constexpr int WARPS_N = BN / WN;
  constexpr int FM = WM / 8, FN = WN / 8;

  extern __shared__ double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * A_EL;
  __shared__ int s_kc[STAGES][2];

  const GemmTask T = tasks[blockIdx.x];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;

  // count k-tiles over all segments
  int njobs = 0;
  for (int s = 0; s < T.nseg; ++s) {
    int kb, ke;
    seg_krange<BM, BN>(segs[T.seg0 + s], T.m0, T.n0, kb, ke);
    if (ke > kb) njobs += (ke - kb + BK - 1) / BK;
  }

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // loader iterator
  int l_seg = 0, l_k = 0, l_kb = 0, l_ke = 0;
  auto l_setup = [&](int s) {
    while (s < T.nseg) {
      seg_krange<BM, BN>(segs[T.seg0 + s], T.m0, T.n0, l_kb, l_ke);
      if (l_ke > l_kb) break;
      ++s;
    }
    l_seg = s;
    l_k = l_kb;
  };
  l_setup(0);

  auto load_stage = [&](int st) {
    const GemmSeg S = segs[T.seg0 + l_seg];
    const int k0 = l_k, ke = l_ke;
    const bool akc = (S.a_ks == 1);
    const bool bkc = (S.b_ks == 1);
    double* dA = sA + st * A_EL;
    double* dB = sB + st * B_EL;
#pragma unroll 4
    for (int idx = tid; idx < BM * BK; idx += NT) {
      int r, k;
      if (akc) { r = idx / BK; k = idx % BK; } else { r = idx % BM; k = idx / BM; }
      const int gi = T.m0 + r, gk = k0 + k;
      const bool v = (gi < T.M) && (gk < ke);
      const double* src = v ? S.A + (long long)gi * S.a_rs + (long long)gk * S.a_ks : S.A;
      cp_async8(dA + (akc ? r * SK + k : k * SMA + r), src, v);
    }
#pragma unroll 4
    for (int idx = tid; idx < BN * BK; idx += NT) {
      int r, k;
      if (bkc) { r = idx / BK; k = idx % BK; } else { r = idx % BN; k = idx / BN; }
      const int gj = T.n0 + r, gk = k0 + k;
      const bool v = (gj < T.N) && (gk < ke);
      const double* src = v ? S.B + (long long)gj * S.b_rs + (long long)gk * S.b_ks : S.B;
      cp_async8(dB + (bkc ? r * SK + k : k * SMB + r), src, v);
    }
    if (tid == 0) { s_kc[st][0] = akc; s_kc[st][1] = bkc; }
    l_k += BK;
    if (l_k >= l_ke) l_setup(l_seg + 1);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < njobs) load_stage(s);
    cp_commit();
  }

  for (int j = 0; j < njobs; ++j) {
    if (j + STAGES - 1 < njobs) load_stage((j + STAGES - 1) % STAGES);
    cp_commit();
    cp_wait<STAGES - 1>();
    __syncthreads();
    const int st = j % STAGES;
    const double* cA = sA + st * A_EL;
    const double* cB = sB + st * B_EL;
    const bool akc = s_kc[st][0], bkc = s_kc[st][1];
    const int a_r = akc ? SK : 1, a_k = akc ? 1 : SMA;
    const int b_r = bkc ? SK : 1, b_k = bkc ? 1 : SMB;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[FM], bf[FN];
      const int k = kk * 4 + t;
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = cA[(wm * WM + i * 8 + g) * a_r + k * a_k];
#pragma unroll
      for (int i = 0; i < FN; ++i) bf[i] = cB[(wn * WN + i * 8 + g) * b_r + k * b_k];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int jn = 0; jn < FN; ++jn) dmma884(acc[i][jn][0], acc[i][jn][1], af[i], bf[jn]);
    }
    __syncthreads();
  }
  cp_wait<0>();

  // epilogue: C = beta*C + alpha*acc
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int gi = T.m0 + wm * WM + i * 8 + g;
    if (gi >= T.M) continue;
#pragma unroll
    for (int jn = 0; jn < FN; ++jn) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gj = T.n0 + wn * WN + jn * 8 + 2 * t + e;
        if (gj >= T.N) continue;
        double* c = T.C + (long long)gi * T.c_rs + (long long)gj * T.c_cs;
        const double a = acc[i][jn][e];
        *c = (T.beta == 0.0) ? T.alpha * a : fma(T.alpha, a, T.beta * (*c));
      }
    }
  }
}

template <int BM, int BN, int WM, int WN, int NT, int STAGES>
static cudaError_t launch_cfg(const GemmTask* d_tasks, int ntasks, const GemmSeg* d_segs, cudaStream_t s) {
  constexpr int BK = 16;
  constexpr int A_EL = (BM * (BK + 4) > BK * (BM + 4)) ? BM * (BK + 4) : BK * (BM + 4);
  constexpr int B_EL = (BN * (BK + 4) > BK * (BN + 4)) ? BN * (BK + 4) : BK * (BN + 4);
  const size_t smem = (size_t)STAGES * (A_EL + B_EL) * sizeof(double);
  auto kern = gemm_f64_kernel<BM, BN, WM, WN, NT, STAGES>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // gridDim.x is limited to 2^31-1; tasks are launched in chunks of 1<<30
  for (int off = 0; off < ntasks; off += (1 << 30)) {
    int cnt = ntasks - off < (1 << 30) ? ntasks - off : (1 << 30);
    count_launch(); kern<<<cnt, NT, smem, s>>>(d_tasks + off, d_segs);
  }
  return cudaGetLastError();
}

cudaError_t launch_gemm(const GemmTask* d_tasks, int ntasks, const GemmSeg* d_segs, int big_tiles,
                        cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  if (big_tiles) return launch_cfg<128, 128, 64, 32, 256, 3>(d_tasks, ntasks, d_segs, s);
  return launch_cfg<64, 64, 32, 32, 128, 3>(d_tasks, ntasks, d_segs, s);
}

}  // namespace sgf
