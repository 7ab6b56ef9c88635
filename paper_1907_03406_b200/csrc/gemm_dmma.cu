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
// multi-stage pipeline.  Each operand tile is stored [row][k] or [k][row]
// depending on which global stride is unit (padding 4 doubles keeps the DMMA
// fragment reads bank-conflict free in both layouts).  Per segment every
// thread precomputes its load pointers, so a stage issues one 64-bit add and
// one LDGSTS per element.
#include <cstdlib>

#include "common.h"

namespace sgf {

__device__ __forceinline__ void cp_async8(unsigned saddr, const void* gmem, bool valid) {
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

constexpr int GEMM_KLIST = 512;  // listed K steps (K <= 8192 at BK 16)

template <int BM, int BN, int BK>
__device__ __forceinline__ void seg_krange(const GemmSeg& S, int m0, int n0, int& kb, int& ke) {
  kb = 0;
  ke = S.K;
  if (S.flags & SEG_KLIM_M) ke = min(ke, m0 + BM);
  if (S.flags & SEG_KLIM_N) ke = min(ke, n0 + BN);
  if (S.flags & SEG_KSTART_M) kb = max(kb, m0);
  if (S.flags & SEG_KSTART_N) kb = max(kb, n0);
  kb = (kb / BK) * BK;
}

// Per-thread load plan for one operand of one segment.  The shared tile is
// always [row][k] (stride BK+4 == 4 mod 16 doubles: conflict-free DMMA
// fragment reads); k-contiguous operands are read along k, row-contiguous
// (transposed) operands along rows.
template <int BR, int BK, int NT>
struct LoadPlan {
  static constexpr int E = BR * BK / NT;  // elements per thread per stage
  static constexpr int SK = BK + 4;
  const double* base;
  long long estep;   // global offset between consecutive elements of this thread
  long long kscale;  // global stride of k
  int kfix;          // k of this thread's elements (k-contiguous) or of element 0
  unsigned rowmask;  // bit e: row in range
  int soff;          // smem offset of element 0
  bool kc;

  __device__ __forceinline__ void setup(const double* P, long long rs, long long ks, int row0, int rows) {
    const int tid = threadIdx.x;
    kc = (ks == 1) || (rs != 1);
    kscale = ks;
    rowmask = 0;
    if (kc) {
      constexpr int RSTEP = NT / BK;
      const int r0 = tid / BK;
      kfix = tid % BK;
      base = P + (long long)(row0 + r0) * rs + (long long)kfix * ks;
      estep = (long long)RSTEP * rs;
      soff = r0 * SK + kfix;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (row0 + r0 + e * RSTEP < rows) rowmask |= 1u << e;
    } else {
      constexpr int KSTEP = NT / BR;
      const int r0 = tid % BR;
      kfix = tid / BR;
      base = P + (long long)(row0 + r0) * rs + (long long)kfix * ks;
      estep = (long long)KSTEP * ks;
      soff = r0 * SK + kfix;
      if (row0 + r0 < rows) rowmask = (E >= 32) ? 0xffffffffu : ((1u << (E & 31)) - 1);
    }
  }

  __device__ __forceinline__ void issue(unsigned sbase, int k0, int ke) const {
    const double* p = base + (long long)k0 * kscale;
    const unsigned s = sbase + 8u * (unsigned)soff;
    if (kc) {
      constexpr int RSTEP = NT / BK;
      const bool kin = (k0 + kfix < ke);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const bool v = kin && ((rowmask >> e) & 1u);
        cp_async8(s + 8u * (e * RSTEP * SK), p, v);  // src-size 0: nothing is read
        p += estep;
      }
    } else {
      constexpr int KSTEP = NT / BR;
      const bool rin = rowmask != 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const bool v = rin && (k0 + kfix + e * KSTEP < ke);
        cp_async8(s + 8u * (e * KSTEP), p, v);
        p += estep;
      }
    }
  }
};

template <int BM, int BN, int WM, int WN, int NT, int STAGES, int BK>
__global__ void __launch_bounds__(NT) gemm_f64_kernel(const GemmTask* __restrict__ descs,
                                                      const GemmTile* __restrict__ tiles,
                                                      const GemmSeg* __restrict__ segs) {
  using LA = LoadPlan<BM, BK, NT>;
  using LB = LoadPlan<BN, BK, NT>;
  constexpr int A_EL = BM * LA::SK;
  constexpr int B_EL = BN * LB::SK;
  constexpr int WARPS_N = BN / WN;
  constexpr int FM = WM / 8, FN = WN / 8;

  extern __shared__ double smem[];
  const unsigned sA0 = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned sB0 = sA0 + STAGES * A_EL * 8;

  const GemmTile tr = tiles[blockIdx.x];
  GemmTask Tt = descs[tr.desc];
  Tt.m0 = (int)tr.mt * BM;
  Tt.n0 = (int)tr.nt * BN;
  const GemmTask& T = Tt;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, t = lane & 3;

  // single-segment tasks whose A carries tile flags: the K steps over a
  // nonzero A tile, listed once in shared memory (all-zero tiles skipped)
  __shared__ short klist[GEMM_KLIST];
  __shared__ int klist_n;
  bool use_list = false;
  if (T.nseg == 1 && segs[T.seg0].a_nz) {
    const GemmSeg S0 = segs[T.seg0];
    int kb, ke;
    seg_krange<BM, BN, BK>(S0, T.m0, T.n0, kb, ke);
    const int nsteps = ke > kb ? (ke - kb + BK - 1) / BK : 0;
    use_list = nsteps <= GEMM_KLIST && BM % 64 == 0;
    if (use_list && warp == 0) {
      int cnt = 0;
      for (int j0 = 0; j0 < nsteps; j0 += 32) {
        const int j = j0 + lane;
        bool f = false;
        if (j < nsteps) {
          const int k = kb + j * BK, kend = min(ke, k + BK);
          for (int rt = T.m0 / 64; rt < (T.m0 + BM) / 64; ++rt)
            for (int c = k / 16; c * 16 < kend; ++c) f |= S0.a_nz[(size_t)rt * S0.a_nzk + c] != 0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (f) klist[cnt + __popc(m & ((1u << lane) - 1u))] = (short)(kb + j * BK);
        cnt += __popc(m);
      }
      if (lane == 0) klist_n = cnt;
    }
    __syncthreads();
  }
  int njobs = 0;
  if (use_list) {
    njobs = klist_n;
  } else {
    for (int s = 0; s < T.nseg; ++s) {
      int kb, ke;
      seg_krange<BM, BN, BK>(segs[T.seg0 + s], T.m0, T.n0, kb, ke);
      if (ke > kb) njobs += (ke - kb + BK - 1) / BK;
    }
  }

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // loader state
  LA la;
  LB lb;
  int l_seg = -1, l_k = 0, l_ke = 0;
  auto next_seg = [&](int s) {
    int kb = 0, ke = 0;
    while (s < T.nseg) {
      seg_krange<BM, BN, BK>(segs[T.seg0 + s], T.m0, T.n0, kb, ke);
      if (ke > kb) break;
      ++s;
    }
    l_seg = s;
    if (s < T.nseg) {
      const GemmSeg S = segs[T.seg0 + s];
      la.setup(S.A, S.a_rs, S.a_ks, T.m0, T.M);
      lb.setup(S.B, S.b_rs, S.b_ks, T.n0, T.N);
      l_k = kb;
      l_ke = ke;
    }
  };
  next_seg(0);
  int l_j = 0;  // next job (listed K step) to load
  auto load_stage = [&](int st) {
    if (use_list) {
      const int k = klist[l_j++];
      la.issue(sA0 + st * A_EL * 8, k, l_ke);
      lb.issue(sB0 + st * B_EL * 8, k, l_ke);
      return;
    }
    la.issue(sA0 + st * A_EL * 8, l_k, l_ke);
    lb.issue(sB0 + st * B_EL * 8, l_k, l_ke);
    l_k += BK;
    if (l_k >= l_ke) next_seg(l_seg + 1);
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
    const double* cA = smem + st * A_EL;
    const double* cB = smem + STAGES * A_EL + st * B_EL;
    const double* pa = cA + (wm * WM + g) * LA::SK + t;
    const double* pb = cB + (wn * WN + g) * LB::SK + t;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = pa[i * 8 * LA::SK + kk * 4];
#pragma unroll
      for (int i = 0; i < FN; ++i) bf[i] = pb[i * 8 * LB::SK + kk * 4];
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

// nonzero flags of 64 x 16 tiles, one warp per tile (32 elements per lane,
// coalesced along the view's contiguous dimension)
__global__ void __launch_bounds__(256) nz_flags64_kernel(const NzFlagJob* __restrict__ jobs,
                                                         const long long* __restrict__ tile_prefix, int njobs) {
  const long long gt = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gt >= tile_prefix[njobs]) return;
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tile_prefix[mid] <= gt) lo = mid;
    else hi = mid - 1;
  }
  const NzFlagJob J = jobs[lo];
  const int nkc = (J.cols + 15) / 16;
  const long long t = gt - tile_prefix[lo];
  const int r0 = (int)(t / nkc) * 64, c0 = (int)(t % nkc) * 16;
  const bool rowc = J.cs == 1;
  bool nz = false;
#pragma unroll 8
  for (int i = 0; i < 32; ++i) {
    const int e = lane + 32 * i;
    const int r = r0 + (rowc ? e / 16 : e % 64), c = c0 + (rowc ? e % 16 : e / 64);
    if (r < J.rows && c < J.cols) nz |= J.p[(long long)r * J.rs + (long long)c * J.cs] != 0.0;
  }
  nz = __any_sync(0xffffffffu, nz);
  if (lane == 0) J.out[t] = nz ? 1 : 0;
}

cudaError_t launch_nz_flags64(const NzFlagJob* d_jobs, const long long* d_tile_prefix, int njobs, long long ntiles,
                              cudaStream_t s) {
  if (njobs <= 0 || ntiles <= 0) return cudaSuccess;
  count_launch();
  nz_flags64_kernel<<<(unsigned)((ntiles * 32 + 255) / 256), 256, 0, s>>>(d_jobs, d_tile_prefix, njobs);
  return cudaGetLastError();
}

template <int BM, int BN, int WM, int WN, int NT, int STAGES, int BK>
static cudaError_t launch_cfg(const GemmTask* d_descs, const GemmTile* d_tiles, int ntasks, const GemmSeg* d_segs,
                              cudaStream_t s) {
  constexpr int A_EL = BM * (BK + 4);
  constexpr int B_EL = BN * (BK + 4);
  const size_t smem = (size_t)STAGES * (A_EL + B_EL) * sizeof(double);
  auto kern = gemm_f64_kernel<BM, BN, WM, WN, NT, STAGES, BK>;
  static FuncAttrs fa;
  cudaError_t e = ensure_smem(kern, smem, fa);
  if (e != cudaSuccess) return e;
  // gridDim.x is limited to 2^31-1; tasks are launched in chunks of 1<<30
  for (int off = 0; off < ntasks; off += (1 << 30)) {
    int cnt = ntasks - off < (1 << 30) ? ntasks - off : (1 << 30);
    count_launch(); kern<<<cnt, NT, smem, s>>>(d_descs, d_tiles + off, d_segs);
  }
  return cudaGetLastError();
}

cudaError_t launch_gemm(const GemmTask* d_descs, const GemmTile* d_tiles, int ntasks, const GemmSeg* d_segs,
                        int big_tiles, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  static int variant = getenv("SGF_GEMM_VARIANT") ? atoi(getenv("SGF_GEMM_VARIANT")) : 0;
  if (big_tiles == 1) return launch_cfg<128, 128, 64, 32, 256, 3, 32>(d_descs, d_tiles, ntasks, d_segs, s);
  // narrow products (N <= 16: the compression's basis columns, pi = 4): a
  // 64 x 16 tile (4 warps of 16 x 16) instead of 64 x 64, 4x less wasted
  // DMMA work and B traffic per useful column
  if (big_tiles == 2) return launch_cfg<64, 16, 16, 16, 128, 2, 16>(d_descs, d_tiles, ntasks, d_segs, s);
  switch (variant) {
    case 1: return launch_cfg<64, 64, 32, 32, 128, 4, 16>(d_descs, d_tiles, ntasks, d_segs, s);
    case 2: return launch_cfg<64, 64, 32, 32, 128, 3, 16>(d_descs, d_tiles, ntasks, d_segs, s);
    case 3: return launch_cfg<64, 64, 32, 32, 128, 2, 32>(d_descs, d_tiles, ntasks, d_segs, s);
    case 4: return launch_cfg<64, 64, 32, 64, 64, 3, 32>(d_descs, d_tiles, ntasks, d_segs, s);
    case 5: return launch_cfg<64, 64, 64, 32, 64, 3, 32>(d_descs, d_tiles, ntasks, d_segs, s);
    case 6: return launch_cfg<64, 64, 32, 32, 128, 2, 16>(d_descs, d_tiles, ntasks, d_segs, s);
    case 8: return launch_cfg<64, 64, 32, 32, 128, 4, 8>(d_descs, d_tiles, ntasks, d_segs, s);
    case 9: return launch_cfg<64, 64, 32, 32, 128, 3, 32>(d_descs, d_tiles, ntasks, d_segs, s);
    // default: 64x64 tile, 4 warps of 32x32, BK=16, 2 stages (41 KB smem -> 4 CTAs
    // = 16 warps per SM): 33.9 TFLOP/s = 91% of the measured DMMA peak on a
    // 7680^2 x 3584 NT problem (tools/gemm_bench.cu)
    default: return launch_cfg<64, 64, 32, 32, 128, 2, 16>(d_descs, d_tiles, ntasks, d_segs, s);
  }
}

}  // namespace sgf
