// FP64 GEMM emulated on the INT8 tensor cores (Ozaki scheme I) for the large
// Schur and coupling products of the factorization.
//
// tcgen05 has no f64 kind; DMMA (mma.sync f64) tops out at ~37 TFLOP/s.  The
// 5th-generation tensor cores run kind::i8 at ~4.5 POPS with exact int32
// accumulation in TMEM, so an FP64 product can be assembled from int8 ones:
// every row of an operand is scaled by a power of two (|x| < 1), truncated to
// a 62-bit fixed-point integer F = trunc(|x| 2^62) (sign applied) and written
// as S = 8 balanced base-256 digits d_t in [-128, 127] (two's-complement
// bytes with carries: exact), x = 2^e sum_t d_t 2^-(8t+6), so
//   (A B^T)_ij = 2^(ea_i + eb_j) sum_{t,u} 2^-(8(t+u)+12) (A_t B_u^T)_ij .
// Pairs with t + u <= S - 1 are kept (36 of 64; the dropped ones weigh
// <= 2^-62 of the row maxima, like the truncation); pairs of one diagonal
// d = t + u accumulate exactly in one int32 TMEM accumulator (<= 8 pairs x
// K x 2^14 < 2^31 for K <= 16384).  The MMA shape is M=128, N=128
// (tools/i8_peak.cu: N=64 issues at only 61% of the 4.5 POPS reached from
// N=128 on), so the 8 diagonals x 128 columns do not fit the 512 TMEM columns
// at once: a product runs in two passes over K, diagonals d = 0..3 (slices
// 0..3 only) then d = 4..7, each pass draining its 4 accumulators into the
// FP64 output.  The epilogue sums 2^-(8d+12) S_d in FP64.  Error <= ~2 K
// 2^-62 max|A_i| max|B_j| (tools/oz_batch_test.cu, graded rows included).
// (A first version used 7-bit sign-magnitude slices, 56 bits: on BASELINE
// cfg5 its level-3 Schur updates moved apply_inverse by 5.6e-10 against the
// reference, over the 1e-10 gate; the balanced 8-bit digits cost nothing.)
//
// Operand layout (written by oz_split_kernel): for an R-row operand padded to
// Rp rows (multiple of 128) and Kp columns (multiple of 32),
//   byte(r, k, t) = ((k/32 * S + t) * Rp/8 + r/8) * 256 + ((k%32)/16) * 128 + (r%8) * 16 + k%16
// i.e. the UMMA canonical K-major no-swizzle layout with LBO = 128 bytes (the
// two K chunks of one K=32 MMA) and SBO = 256 bytes (8-row groups); the 128
// rows of a tile of one (k-tile, slice) are one contiguous 4 KB range, moved
// by one bulk copy.
#include <cmath>
#include <cstdlib>

#include "common.h"
#include "ptx_util.cuh"

namespace sgf {

namespace {

constexpr int OZ_S = 8;
constexpr int OZ_BM = 128, OZ_BN = 128, OZ_KT = 32;
constexpr int OZ_STAGES = 3;
constexpr int OZ_A_TILE = OZ_BM * OZ_KT, OZ_B_TILE = OZ_BN * OZ_KT;
constexpr int OZ_A_STAGE = OZ_S * OZ_A_TILE, OZ_B_STAGE = OZ_S * OZ_B_TILE;
constexpr int OZ_H = OZ_S / 2;  // diagonals (and, in pass 0, slices) per pass
constexpr int OZ_EPI_WARPS = 8;  // epilogue: warp w drains TMEM lane quadrant w % 4, column half w / 4
constexpr int OZ_PROD_WARP = OZ_EPI_WARPS, OZ_MMA_WARP = OZ_EPI_WARPS + 1;
constexpr int OZ_THREADS = 32 * (OZ_EPI_WARPS + 2);
constexpr int OZ_EC = 16;  // epilogue chunk: columns per TMEM load / staging pass

#ifdef OZ_PROFILE
// cycles: [0] MMA waiting for operands, [1] MMA waiting for the epilogue,
// [2] MMA issuing, [3] epilogue draining, [4] epilogue waiting for the MMA
__device__ unsigned long long oz_prof[8];
#define OZ_T0() const long long _t0 = clock64()
#define OZ_ACC(i) atomicAdd(&oz_prof[i], (unsigned long long)(clock64() - _t0))
#else
#define OZ_T0()
#define OZ_ACC(i)
#endif

using namespace ptx;
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  // K-major, no swizzle: LBO 128 B between the two K chunks of one MMA step,
  // SBO 256 B between 8-row core-matrix groups, version 1 (Blackwell)
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
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

// The S balanced base-256 digits of x 2^-ex (|x| 2^-ex < 1), most
// significant first: F = trunc(|x| 2^(62-ex)) with x's sign (oz_fixed), then
// d = F mod 256 in [-128, 127], F = (F - d) / 256, least significant first
// (oz_pack4).  oz_fixed: the 62-bit fixed-point integer of x 2^-ex.
__device__ __forceinline__ long long oz_fixed(double x, int ex) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int bexp = (int)((bits >> 52) & 0x7FF);
  unsigned long long F = 0;
  if (bexp != 0) {  // zero (and subnormals, far below any row maximum) give 0
    const unsigned long long mant = (bits & 0xFFFFFFFFFFFFFull) | (1ull << 52);
    const int sh = bexp - 1075 + 62 - ex;  // F = |x| 2^(62-ex) < 2^62 (sh <= 9)
    F = sh >= 0 ? (sh < 10 ? mant << sh : 0) : (sh > -53 ? mant >> (-sh) : 0);
  }
  return ((long long)bits < 0) ? -(long long)F : (long long)F;
}

// Slice words of 4 consecutive elements: out[t] holds the (int8) digit t of
// elements 0..3 in its bytes 0..3.  The balanced base-256 digits of v are the
// bytes of u = v + 0x80..80 minus 128 (adding 128 to every digit leaves them
// in [0, 255], so no carries), i.e. as int8 bytes: byte_j(u) ^ 0x80, digit
// t (most significant first) = byte 7 - t.  Four byte permutes per slice
// word instead of eight dependent extract/subtract/shift steps per element
// (d = (int8)(v & 0xFF), v = (v - d) >> 8, least significant digit first).
__device__ __forceinline__ void oz_pack4(const double (&x)[4], int ex, uint32_t (&out)[OZ_S]) {
  constexpr unsigned long long B = 0x8080808080808080ull;
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const unsigned long long u = ((unsigned long long)oz_fixed(x[e], ex) + B) ^ B;
    lo[e] = (uint32_t)u;
    hi[e] = (uint32_t)(u >> 32);
  }
#pragma unroll
  for (int t = 0; t < OZ_S; ++t) {
    const int j = 3 - (t & 3);  // byte within the word: t = 0..3 from hi, 4..7 from lo
    const uint32_t* W = t < 4 ? hi : lo;
    const uint32_t a01 = __byte_perm(W[0], W[1], (uint32_t)(j | ((j + 4) << 4)));
    const uint32_t a23 = __byte_perm(W[2], W[3], (uint32_t)(j | ((j + 4) << 4)));
    out[t] = __byte_perm(a01, a23, 0x5410);
  }
}

// One warp per group of 8 operand rows: lane l works on row (l & 7) and on
// the 16-element K chunks c = (l >> 3) + 4 i, so for every slice the warp
// stores two contiguous 256-byte runs (the core matrices of two K tiles).
// Pass 1: row maxima (-> power-of-two exponents); pass 2: slices.
__global__ void __launch_bounds__(256) oz_split_kernel(const OzSplitJob* __restrict__ jobs,
                                                       const long long* __restrict__ group_prefix, int njobs) {
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= group_prefix[njobs]) return;
  int lo = 0, hi = njobs - 1;  // job containing row group gw
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (group_prefix[mid] <= gw) lo = mid;
    else hi = mid - 1;
  }
  const OzSplitJob J = jobs[lo];
  const int r = (int)(gw - group_prefix[lo]) * 8 + (lane & 7);
  const int c0 = lane >> 3;
  const bool live = r < J.R;
  const double* row = J.x + (long long)r * J.rs;
  double mx = 0.0;
  int kf = J.K;  // first nonzero column of the row seen by this lane
  if (live)
    for (int k0 = c0 * 16; k0 < J.K; k0 += 64)
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (k0 + q < J.K) {
          const double x = row[(long long)(k0 + q) * J.cs];
          mx = fmax(mx, fabs(x));
          if (x != 0.0) kf = min(kf, k0 + q);
        }
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  kf = min(kf, __shfl_xor_sync(0xffffffffu, kf, 8));
  kf = min(kf, __shfl_xor_sync(0xffffffffu, kf, 16));
  int ex = 0;
  if (mx > 0.0) frexp(mx, &ex);  // |x| 2^-ex < 1
  if (lane < 8) J.exps[r] = live ? ex : 0;
  if (lane < 8 && live && J.kfirst) J.kfirst[r] = kf;
  const size_t blk = (size_t)J.Rp * OZ_KT;  // bytes of one (k-tile, slice) block
  for (int k0 = c0 * 16; k0 < J.Kp; k0 += 64) {
    unsigned w[OZ_S][4];
    bool nzv = false;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      double x4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = k0 + 4 * p + e;
        x4[e] = (live && k < J.K) ? row[(long long)k * J.cs] : 0.0;
        nzv |= x4[e] != 0.0;
      }
      uint32_t o[OZ_S];
      oz_pack4(x4, ex, o);
#pragma unroll
      for (int t = 0; t < OZ_S; ++t) w[t][p] = o[t];
    }
    const int kt = k0 / OZ_KT, kc = (k0 % OZ_KT) / 16;
    const size_t off = (size_t)(r >> 3) * 256 + (size_t)kc * 128 + (size_t)(r & 7) * 16;
    unsigned any = 0u;
#pragma unroll
    for (int t = 0; t < OZ_S; ++t) {
      uint4 v4 = make_uint4(w[t][0], w[t][1], w[t][2], w[t][3]);
      any |= v4.x | v4.y | v4.z | v4.w;
      *reinterpret_cast<uint4*>(J.out + ((size_t)kt * OZ_S + t) * blk + off) = v4;
    }
    if (J.nz && any) J.nz[(size_t)(r >> 7) * (J.Kp / OZ_KT) + kt] = 1;  // benign race: every writer stores 1
    if (J.rmask && nzv) atomicOr(&J.rmask[(size_t)r * J.mwords + (kt >> 5)], 1u << (kt & 31));
  }
}

// Same split for row-contiguous operands (cs == 1), one CTA per 8-row group
// with coalesced reads: warp w streams row w (lane = column), once for the
// row maxima and once into a shared 8 x 512 tile from which the slices are
// cut in the store-friendly lane mapping of oz_split_kernel.  (The warp-per-
// group form reads 16-element runs per lane and fetched ~2x the operand bytes
// from HBM.)  Identical output.
constexpr int OZS_TK = 512, OZS_PITCH = OZS_TK + 4;
constexpr int OZS_MW = 16;  // row-mask words (K <= 16384)
__global__ void __launch_bounds__(256) oz_split_cta_kernel(const OzSplitJob* __restrict__ jobs,
                                                           const long long* __restrict__ group_prefix, int njobs) {
  __shared__ double tile[8 * OZS_PITCH];
  __shared__ int sex[8];
  const long long gw = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int lo = 0, hi = njobs - 1;  // job containing row group gw
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (group_prefix[mid] <= gw) lo = mid;
    else hi = mid - 1;
  }
  const OzSplitJob J = jobs[lo];
  const int g0 = (int)(gw - group_prefix[lo]) * 8;
  // trans: the 8 rows of a group are contiguous for every k (rs == 1): thread
  // t reads row t & 7 at k = t >> 3 (+32 i), 64-byte runs per k
  const bool trans = J.cs != 1;
  if (!trans) {  // pass 1: row maxima (and first nonzero), warp w = row g0 + w
    const int r = g0 + warp;
    double mx = 0.0;
    int kf = J.K;
    if (r < J.R) {
      const double* row = J.x + (long long)r * J.rs;
      for (int k = lane; k < J.K; k += 32) {
        const double x = __ldg(row + k);
        mx = fmax(mx, fabs(x));
        if (x != 0.0) kf = min(kf, k);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      kf = min(kf, __shfl_xor_sync(0xffffffffu, kf, o));
    }
    if (lane == 0) {
      int e = 0;
      if (mx > 0.0) frexp(mx, &e);  // |x| 2^-ex < 1
      sex[warp] = e;
      if (r < J.R) J.exps[r] = e;
      if (r < J.R && J.kfirst) J.kfirst[r] = kf;
    }
  } else {
    const int r = g0 + (threadIdx.x & 7);
    double mx = 0.0;
    int kf = J.K;
    if (r < J.R)
      for (int k = threadIdx.x >> 3; k < J.K; k += 32) {
        const double x = __ldg(J.x + r + (long long)k * J.cs);
        mx = fmax(mx, fabs(x));
        if (x != 0.0) kf = min(kf, k);
      }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    kf = min(kf, __shfl_xor_sync(0xffffffffu, kf, 8));
    kf = min(kf, __shfl_xor_sync(0xffffffffu, kf, 16));
    __shared__ double wm[8][8];
    __shared__ int wk[8][8];
    if (lane < 8) {
      wm[warp][lane] = mx;
      wk[warp][lane] = kf;
    }
    __syncthreads();
    if (threadIdx.x < 8) {
      double m = 0.0;
      int kmin = J.K;
      for (int w = 0; w < 8; ++w) {
        m = fmax(m, wm[w][threadIdx.x]);
        kmin = min(kmin, wk[w][threadIdx.x]);
      }
      int e = 0;
      if (m > 0.0) frexp(m, &e);
      sex[threadIdx.x] = e;
      if (g0 + (int)threadIdx.x < J.R) {
        J.exps[g0 + threadIdx.x] = e;
        if (J.kfirst) J.kfirst[g0 + threadIdx.x] = kmin;
      }
    }
  }
  __shared__ uint32_t smask[8][OZS_MW];  // per row: bit kt = 32-column tile kt holds a nonzero value
  if (J.rmask)
    for (int i = threadIdx.x; i < 8 * OZS_MW; i += 256) smask[i / OZS_MW][i % OZS_MW] = 0u;
  __syncthreads();
  const int rl = lane & 7, r = g0 + rl;
  const int ex = sex[rl];
  const size_t blk = (size_t)J.Rp * OZ_KT;  // bytes of one (k-tile, slice) block
  for (int kb = 0; kb < J.Kp; kb += OZS_TK) {
    if (!trans) {  // stage rows g0..g0+7, columns [kb, kb + 512)
      const int rr = g0 + warp;
      const double* row = J.x + (long long)rr * J.rs;
#pragma unroll 4
      for (int i = lane; i < OZS_TK; i += 32) {
        const int k = kb + i;
        tile[warp * OZS_PITCH + i] = (rr < J.R && k < J.K) ? __ldg(row + k) : 0.0;
      }
    } else {
      const int rr = g0 + (threadIdx.x & 7);
#pragma unroll 4
      for (int i = threadIdx.x >> 3; i < OZS_TK; i += 32) {
        const int k = kb + i;
        tile[(threadIdx.x & 7) * OZS_PITCH + i] = (rr < J.R && k < J.K) ? __ldg(J.x + rr + (long long)k * J.cs) : 0.0;
      }
    }
    __syncthreads();
    const int ci = warp * 4 + (lane >> 3);  // 16-element chunk of the tile
    const int k0 = kb + ci * 16;
    if (k0 < J.Kp) {
      unsigned w[OZ_S][4];
      bool nzv = false;  // a nonzero value (not digit) in this 16-column chunk of the row
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        double x4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          x4[e] = tile[rl * OZS_PITCH + ci * 16 + 4 * p + e];
          nzv |= x4[e] != 0.0;
        }
        uint32_t o[OZ_S];
        oz_pack4(x4, ex, o);
#pragma unroll
        for (int t = 0; t < OZ_S; ++t) w[t][p] = o[t];
      }
      const int kt = k0 / OZ_KT, kc = (k0 % OZ_KT) / 16;
      if (J.rmask && nzv) atomicOr(&smask[rl][kt >> 5], 1u << (kt & 31));
      const size_t off = (size_t)(r >> 3) * 256 + (size_t)kc * 128 + (size_t)(r & 7) * 16;
      unsigned any = 0u;
#pragma unroll
      for (int t = 0; t < OZ_S; ++t) {
        uint4 v4 = make_uint4(w[t][0], w[t][1], w[t][2], w[t][3]);
        any |= v4.x | v4.y | v4.z | v4.w;
        *reinterpret_cast<uint4*>(J.out + ((size_t)kt * OZ_S + t) * blk + off) = v4;
      }
      if (J.nz && any) J.nz[(size_t)(r >> 7) * (J.Kp / OZ_KT) + kt] = 1;  // benign race: every writer stores 1
    }
    __syncthreads();
  }
  if (J.rmask)
    for (int i = threadIdx.x; i < 8 * J.mwords; i += 256) {
      const int rr = g0 + i / J.mwords, wi = i % J.mwords;
      if (rr < J.R) J.rmask[(size_t)rr * J.mwords + wi] = smask[i / J.mwords][wi];
    }
}

// Split of row-contiguous operands with rows of at most OZR_KMAX columns
// (the couplings E and A_NB, L^{-1}, A21 ...), one CTA per R rows: the rows
// are fetched once (by the bulk copy engine when 16-byte aligned) into shared memory
// (pass 1 then reads them there for the row maxima; the CTA kernel above
// streams every row twice from HBM, the second time after it was evicted
// from L2), then cut into slices.  A CTA writes its R rows' 16-byte pieces
// of every 8-row core matrix (the other rows of the group are other CTAs).
// R = 2 for long rows (up to 3 CTAs per SM overlap staging and cutting),
// 4 or 8 for short ones (per-CTA overheads).
// Identical output to the kernels above.
constexpr int OZR_KMAX = 6912;
template <int OZR_ROWS>
__global__ void __launch_bounds__(256) oz_split_rows_kernel(const OzSplitJob* __restrict__ jobs,
                                                            const long long* __restrict__ group_prefix, int njobs) {
  extern __shared__ __align__(16) double srow[];  // [OZR_ROWS][pitch]
  __shared__ __align__(8) uint64_t bar;
  __shared__ double smx[8];
  __shared__ int skf[8], sex[OZR_ROWS];
  __shared__ uint32_t smask[OZR_ROWS][OZS_MW];
  const long long gw = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int lo = 0, hi = njobs - 1;  // job containing row group gw
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (group_prefix[mid] <= gw) lo = mid;
    else hi = mid - 1;
  }
  const OzSplitJob J = jobs[lo];
  const int g0 = (int)(gw - group_prefix[lo]) * OZR_ROWS;
  const int pitch = J.Kp + 2;  // doubles; 16-byte multiple, staggers the rows' banks
  const int nlive = max(0, min(OZR_ROWS, J.R - g0));
  // 16-byte aligned rows: the bulk copy engine (an odd last column is loaded
  // directly); otherwise every thread loads (coalesced along the row)
  const bool aligned = J.rs % 2 == 0 && ((uintptr_t)J.x & 15) == 0;
  const int kb2 = aligned ? J.K & ~1 : 0;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::mbar_init_fence();
    ptx::mbar_expect_tx(&bar, (uint32_t)nlive * kb2 * 8u);
    for (int i = 0; i < nlive; ++i)
      if (kb2) ptx::bulk_g2s(srow + i * pitch, J.x + (long long)(g0 + i) * J.rs, (uint32_t)kb2 * 8u, &bar);
  }
  for (int i = threadIdx.x; i < OZR_ROWS * OZS_MW; i += 256) smask[i / OZS_MW][i % OZS_MW] = 0u;
  // zero padding (columns K .. Kp) and dead rows; the odd last column
  // (per row over the columns the bulk copy does not write: a flat loop over
  // every staged element with a division each was a third of the kernel's stalls)
  for (int rr = 0; rr < OZR_ROWS; ++rr) {
    const bool live = rr < nlive;
    for (int k = (live ? kb2 : 0) + threadIdx.x; k < pitch; k += 256)
      srow[rr * pitch + k] = (live && k < J.K) ? J.x[(long long)(g0 + rr) * J.rs + k] : 0.0;
  }
  __syncthreads();
  ptx::mbar_wait(&bar, 0);
  {  // pass 1: row maxima and first nonzero, warps (row w % R, part w / R of 8 / R)
    constexpr int NP = 8 / OZR_ROWS;
    const int rr = warp % OZR_ROWS, h = warp / OZR_ROWS;
    const int part = (J.Kp / NP + 15) & ~15;
    const int k0 = min(J.Kp, h * part), k1 = h == NP - 1 ? J.Kp : min(J.Kp, (h + 1) * part);
    const double* row = srow + rr * pitch;
    double mx = 0.0;
    int kf = J.K;
    for (int k = k0 + lane; k < k1; k += 32) {
      const double x = row[k];
      mx = fmax(mx, fabs(x));
      if (x != 0.0) kf = min(kf, k);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      kf = min(kf, __shfl_xor_sync(0xffffffffu, kf, o));
    }
    if (lane == 0) {
      smx[warp] = mx;
      skf[warp] = kf;
    }
  }
  __syncthreads();
  if (threadIdx.x < OZR_ROWS) {
    const int t = threadIdx.x;
    double m = 0.0;
    int kf = J.K;
    for (int p = t; p < 8; p += OZR_ROWS) {
      m = fmax(m, smx[p]);
      kf = min(kf, skf[p]);
    }
    int e = 0;
    if (m > 0.0) frexp(m, &e);  // |x| 2^-ex < 1
    sex[t] = e;
    if (t < nlive) {
      J.exps[g0 + t] = e;
      if (J.kfirst) J.kfirst[g0 + t] = kf;
    }
  }
  if (g0 + OZR_ROWS > J.R && threadIdx.x >= OZR_ROWS && threadIdx.x < 2 * OZR_ROWS) {
    const int t = threadIdx.x - OZR_ROWS;  // padded rows of the operand: exponent 0
    if (g0 + t >= J.R && g0 + t < J.Rp) J.exps[g0 + t] = 0;
  }
  __syncthreads();
  // pass 2: items (row, 16-column chunk), 8 slices of 16 bytes each
  const size_t blk = (size_t)J.Rp * OZ_KT;  // bytes of one (k-tile, slice) block
  const int nch = J.Kp / 16;
  for (int item = threadIdx.x; item < OZR_ROWS * nch; item += 256) {
    const int rr = item % OZR_ROWS, ch = item / OZR_ROWS;
    const int r = g0 + rr, k0 = ch * 16;
    const int ex = sex[rr];
    const double2* src = reinterpret_cast<const double2*>(srow + rr * pitch + k0);
    unsigned w[OZ_S][4];
    bool nzv = false;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const double2 v0 = src[2 * p], v1 = src[2 * p + 1];
      const double x4[4] = {v0.x, v0.y, v1.x, v1.y};
      nzv |= (x4[0] != 0.0) | (x4[1] != 0.0) | (x4[2] != 0.0) | (x4[3] != 0.0);
      uint32_t o[OZ_S];
      oz_pack4(x4, ex, o);
#pragma unroll
      for (int t = 0; t < OZ_S; ++t) w[t][p] = o[t];
    }
    const int kt = k0 / OZ_KT, kc = (k0 % OZ_KT) / 16;
    const size_t off = (size_t)(r >> 3) * 256 + (size_t)kc * 128 + (size_t)(r & 7) * 16;
    unsigned any = 0u;
#pragma unroll
    for (int t = 0; t < OZ_S; ++t) {
      uint4 v4 = make_uint4(w[t][0], w[t][1], w[t][2], w[t][3]);
      any |= v4.x | v4.y | v4.z | v4.w;
      *reinterpret_cast<uint4*>(J.out + ((size_t)kt * OZ_S + t) * blk + off) = v4;
    }
    if (J.nz && any) J.nz[(size_t)(r >> 7) * (J.Kp / OZ_KT) + kt] = 1;  // benign race: every writer stores 1
    if (J.rmask && nzv) atomicOr(&smask[rr][kt >> 5], 1u << (kt & 31));
  }
  if (J.rmask) {
    __syncthreads();
    for (int i = threadIdx.x; i < nlive * J.mwords; i += 256) {
      const int rr = i / J.mwords, wi = i % J.mwords;
      J.rmask[(size_t)(g0 + rr) * J.mwords + wi] = smask[rr][wi];
    }
  }
}

// K tiles of one segment: for the first two segments of a tile whose
// operands carry nonzero flags, the list of the K tiles where both the A
// tile and the B tile hold a nonzero (an absent flag array counts as all
// nonzero; built once per CTA in shared memory; every other K tile is a
// product with an all-zero operand tile, an exact zero, and is skipped),
// otherwise the range [kstart, nk) (flags of later segments, or of
// products with more than 256 K tiles, are not used).  The producer and MMA
// loops stay simple counted loops either way (a data-dependent skip inside
// the MMA issue loop cost 7-9% on dense products).
constexpr int OZ_KLIST = 256, OZ_KLSEG = 2;
struct OzKRange {
  const uint8_t* list;  // nullptr: dense range
  int kstart, count;
  __device__ __forceinline__ int k(int idx) const { return list ? (int)list[idx] : kstart + idx; }
};

__global__ void __launch_bounds__(OZ_THREADS, 1)
    oz_gemm_kernel(const OzTask* __restrict__ tasks, const OzSeg* __restrict__ segs) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + OZ_STAGES * OZ_A_STAGE;
  __shared__ __align__(8) uint64_t full[OZ_STAGES], empty[OZ_STAGES], tmem_full, tmem_empty;
  __shared__ uint32_t tmem_base;
  __shared__ uint8_t klist[OZ_KLSEG][OZ_KLIST];
  __shared__ int kcount[OZ_KLSEG];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const OzTask T = tasks[blockIdx.x];
  if (warp < OZ_KLSEG && warp < T.nseg) {  // K-tile lists of segments 0 and 1 (warp w: segment w)
    const OzSeg G = segs[T.seg0 + warp];
    const int nk = min(G.nk, T.klim);
    if ((G.a_nz || G.b_nz) && nk <= OZ_KLIST) {
      const uint8_t* fa = G.a_nz ? G.a_nz + (size_t)(T.m0 / OZ_BM) * G.nk : nullptr;
      const uint8_t* fb = G.b_nz ? G.b_nz + (size_t)(T.n0 / OZ_BN) * G.nk : nullptr;
      int cnt = 0;
      for (int k0 = T.kstart; k0 < nk; k0 += 32) {
        const int k = k0 + lane;
        const bool f = k < nk && (!fa || fa[k] != 0) && (!fb || fb[k] != 0);
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (f) klist[warp][cnt + __popc(m & ((1u << lane) - 1u))] = (uint8_t)k;
        cnt += __popc(m);
      }
      if (lane == 0) kcount[warp] = cnt;
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tmem_full, 1);
    mbar_init(&tmem_empty, 32 * OZ_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == OZ_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  auto krange = [&](int si, const OzSeg& G) {
    OzKRange r;
    const int nk = min(G.nk, T.klim);
    r.kstart = T.kstart;
    r.list = nullptr;
    r.count = max(0, nk - T.kstart);
    if ((G.a_nz || G.b_nz) && si < OZ_KLSEG && nk <= OZ_KLIST) {
      r.list = klist[si];
      r.count = kcount[si];
    }
    return r;
  };

  if (warp == OZ_PROD_WARP) {
    if (lane == 0) {  // producer: stages of all segments in order
      int it = 0;
      for (int si = 0; si < T.nseg; ++si) {
        const OzSeg G = segs[T.seg0 + si];
        const OzKRange kr = krange(si, G);
        const int8_t* a = G.a + (size_t)T.m0 * OZ_KT;
        const int8_t* b = G.b + (size_t)T.n0 * OZ_KT;
        const size_t ablk = (size_t)G.a_rp * OZ_KT, bblk = (size_t)G.b_rp * OZ_KT;
        for (int pass = 0; pass < 2; ++pass) {
          const int ns = pass == 0 ? OZ_H : OZ_S;  // slices used by the pass
          for (int idx = 0; idx < kr.count; ++idx) {
            const int k = kr.k(idx);
            const int s = it % OZ_STAGES;
            ++it;
            if (it > OZ_STAGES) mbar_wait(&empty[s], (((it - 1) / OZ_STAGES) - 1) & 1);
            mbar_expect_tx(&full[s], (uint32_t)ns * (OZ_A_TILE + OZ_B_TILE));
            for (int t = 0; t < ns; ++t) {
              bulk_g2s(sA + s * OZ_A_STAGE + t * OZ_A_TILE, a + ((size_t)k * OZ_S + t) * ablk, OZ_A_TILE, &full[s]);
              bulk_g2s(sB + s * OZ_B_STAGE + t * OZ_B_TILE, b + ((size_t)k * OZ_S + t) * bblk, OZ_B_TILE, &full[s]);
            }
          }
        }
      }
    }
  } else if (warp == OZ_MMA_WARP) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc =
          (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_BN >> 3) << 17) | ((uint32_t)(OZ_BM >> 4) << 24);
      int it = 0, drains = 0;
      for (int si = 0; si < T.nseg; ++si) {
        const OzSeg G = segs[T.seg0 + si];
        const OzKRange kr = krange(si, G);
        for (int pass = 0; pass < 2; ++pass, ++drains) {
          if (drains > 0) {
            OZ_T0();
            mbar_wait(&tmem_empty, (drains - 1) & 1);  // epilogue drained the accumulators
            OZ_ACC(1);
          }
          asm volatile("tcgen05.fence::after_thread_sync;");
          bool k0 = true;  // first K tile of the pass: the accumulators start from it
          for (int idx = 0; idx < kr.count; ++idx) {
            const int s = it % OZ_STAGES;
            const int ph = (it / OZ_STAGES) & 1;
            ++it;
            {
              OZ_T0();
              mbar_wait(&full[s], ph);
              OZ_ACC(0);
            }
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t a0 = smem_u32(sA + s * OZ_A_STAGE), b0 = smem_u32(sB + s * OZ_B_STAGE);
            OZ_T0();
            if (pass == 0) {
              // diagonals 0..3 (slice pairs t + u <= 3); (0, d) writes diagonal d first
#pragma unroll
              for (int t = 0; t < OZ_H; ++t)
#pragma unroll
                for (int u = 0; u < OZ_H - t; ++u)
                  mma_i8(tmem + (uint32_t)(t + u) * OZ_BN, smem_desc(a0 + t * OZ_A_TILE),
                         smem_desc(b0 + u * OZ_B_TILE), idesc, (!k0 || t > 0) ? 1u : 0u);
            } else {
              // diagonals 4..7; (t, 7 - t... ) ordering: for t ascending the first
              // pair of diagonal d is (max(0, d-7), ...) -> track the first write
#pragma unroll
              for (int t = 0; t < OZ_S; ++t)
#pragma unroll
                for (int u = 0; u < OZ_S - t; ++u) {
                  const int d = t + u;
                  if (d < OZ_H) continue;
                  const bool first = k0 && (t == (d > OZ_S - 1 ? d - (OZ_S - 1) : 0));
                  mma_i8(tmem + (uint32_t)(d - OZ_H) * OZ_BN, smem_desc(a0 + t * OZ_A_TILE),
                         smem_desc(b0 + u * OZ_B_TILE), idesc, first ? 0u : 1u);
                }
            }
            mma_commit(&empty[s]);
            OZ_ACC(2);
            k0 = false;
          }
          mma_commit(&tmem_full);
        }
      }
    }
  } else {
    // epilogue, warps 0-7: thread = tile row (TMEM lane) of quadrant warp % 4,
    // columns [64 (warp / 4), +64) in chunks of 16.  Two warps per SM
    // sub-partition keep the TMEM-load -> convert -> C read-modify-write
    // chains of one overlapping the other's (one warp per quadrant over all
    // 128 columns ran them back to back: the drain took as long as the MMAs)
    const int quad = warp & 3, half = warp >> 2;
    const int lr = quad * 32 + lane;
    const int row = T.m0 + lr;
    // staging tile of this warp: 32 rows x 16 columns, column index XOR-swizzled
    // by the row (conflict-free row writes and column reads of 8-byte words),
    // so the C read-modify-write runs with the lanes on 16 consecutive
    // columns of 2 rows (coalesced) instead of one row per thread
    double* stg = reinterpret_cast<double*>(smem + OZ_STAGES * (OZ_A_STAGE + OZ_B_STAGE)) + warp * 32 * OZ_EC;
    int drains = 0;
    for (int si = 0; si < T.nseg; ++si) {
      const OzSeg G = segs[T.seg0 + si];
      const bool live = row < T.M;
      const double rs = live ? ldexp(G.alpha, G.ea[row]) : 0.0;
      // no K tile at all (every A tile zero): the accumulators were never written
      const bool empty_seg = krange(si, G).count == 0;
      for (int pass = 0; pass < 2; ++pass, ++drains) {
        {
          OZ_T0();
          mbar_wait(&tmem_full, drains & 1);
          if (threadIdx.x == 0) OZ_ACC(4);
        }
        asm volatile("tcgen05.fence::after_thread_sync;");
        OZ_T0();
        const bool first = (si == 0 && pass == 0);
#pragma unroll 1
        for (int c0 = half * (OZ_BN / 2); c0 < (half + 1) * (OZ_BN / 2); c0 += OZ_EC) {
          // the four diagonals' 16 columns in flight together, one wait
          uint32_t v[OZ_H][OZ_EC];
#pragma unroll
          for (int dd = 0; dd < OZ_H; ++dd)
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(v[dd][0]), "=r"(v[dd][1]), "=r"(v[dd][2]), "=r"(v[dd][3]), "=r"(v[dd][4]), "=r"(v[dd][5]),
                  "=r"(v[dd][6]), "=r"(v[dd][7]), "=r"(v[dd][8]), "=r"(v[dd][9]), "=r"(v[dd][10]), "=r"(v[dd][11]),
                  "=r"(v[dd][12]), "=r"(v[dd][13]), "=r"(v[dd][14]), "=r"(v[dd][15])
                : "r"(tmem + ((uint32_t)(quad * 32) << 16) + dd * OZ_BN + c0));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          double acc[OZ_EC];
#pragma unroll
          for (int j = 0; j < OZ_EC; ++j) acc[j] = 0.0;
#pragma unroll
          for (int dd = OZ_H - 1; dd >= 0; --dd) {  // smallest terms first
            const double sc = ldexp(1.0, -(8 * (dd + pass * OZ_H) + 12));
#pragma unroll
            for (int j = 0; j < OZ_EC; ++j) acc[j] = fma((double)(int32_t)v[dd][j], sc, acc[j]);
          }
#pragma unroll
          for (int j = 0; j < OZ_EC; ++j) stg[lane * OZ_EC + (j ^ (lane & 15))] = acc[j] * rs;
          __syncwarp();
          const int cl = lane & 15, rh = lane >> 4;  // column within the chunk, row parity
          const int col = T.n0 + c0 + cl;
          const bool cok = col < T.N && !empty_seg;
          const double cs = cok ? ldexp(1.0, G.eb[col]) : 0.0;
          // all loads of the 16 row pairs first (independent), then the stores
          const int nrow = min(32, T.M - (T.m0 + quad * 32));
          double* cbase = T.C + (long long)(T.m0 + quad * 32 + rh) * T.c_rs + (long long)col * T.c_cs;
          const bool need_c = !(first && T.beta == 0.0);
          double cv[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            cv[i] = (need_c && 2 * i + rh < nrow && col < T.N) ? __ldcg(cbase + (long long)(2 * i) * T.c_rs) : 0.0;
          const double bscale = first ? T.beta : 1.0;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int r = 2 * i + rh;
            if (r < nrow && col < T.N)
              cbase[(long long)(2 * i) * T.c_rs] = fma(bscale, cv[i], stg[r * OZ_EC + (cl ^ (r & 15))] * cs);
          }
          __syncwarp();
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(&tmem_empty);
        if (threadIdx.x == 0) OZ_ACC(3);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == OZ_MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace

#ifdef OZ_PROFILE
extern "C" int sgf_oz_prof_read(unsigned long long* out, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, oz_prof, sizeof(oz_prof));
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(oz_prof, z, sizeof(z));
  }
  return e == cudaSuccess ? 0 : 1;
}
#endif

// d_group_prefix: per job the first global 8-row group (njobs + 1 entries)
int oz_split_rows_per_cta(int max_kp) { return max_kp <= 1024 ? 8 : (max_kp <= 2048 ? 4 : 2); }
template <int R>
static cudaError_t split_rows_launch(const OzSplitJob* d_jobs, const long long* d_prefix, int njobs, long long ngroups,
                                     int max_kp, cudaStream_t s) {
  const size_t smem = (size_t)R * (max_kp + 2) * sizeof(double);
  static FuncAttrs fa;
  cudaError_t e = ensure_smem(oz_split_rows_kernel<R>, smem, fa);
  if (e != cudaSuccess) return e;
  oz_split_rows_kernel<R><<<(unsigned)ngroups, 256, smem, s>>>(d_jobs, d_prefix, njobs);
  return cudaGetLastError();
}
cudaError_t launch_oz_split_rows(const OzSplitJob* d_jobs, const long long* d_group_prefix, int njobs,
                                 long long total_groups, int max_kp, cudaStream_t s) {
  if (njobs <= 0 || total_groups <= 0) return cudaSuccess;
  count_launch();
  switch (oz_split_rows_per_cta(max_kp)) {
    case 8: return split_rows_launch<8>(d_jobs, d_group_prefix, njobs, total_groups, max_kp, s);
    case 4: return split_rows_launch<4>(d_jobs, d_group_prefix, njobs, total_groups, max_kp, s);
    default: return split_rows_launch<2>(d_jobs, d_group_prefix, njobs, total_groups, max_kp, s);
  }
}
bool oz_split_rows_ok(const OzSplitJob& j) { return j.cs == 1 && j.Kp <= OZR_KMAX && j.R > 0; }

cudaError_t launch_oz_split(const OzSplitJob* d_jobs, const long long* d_group_prefix, int njobs,
                            long long total_groups, cudaStream_t s, bool all_rowc) {
  if (njobs <= 0 || total_groups <= 0) return cudaSuccess;
  count_launch();
  static const int cta = getenv("SGF_OZ_SPLIT_WARP") ? 0 : 1;
  if (cta && all_rowc && total_groups < (1LL << 31)) {
    oz_split_cta_kernel<<<(unsigned)total_groups, 256, 0, s>>>(d_jobs, d_group_prefix, njobs);
    return cudaGetLastError();
  }
  const long long threads = total_groups * 32;
  oz_split_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(d_jobs, d_group_prefix, njobs);
  return cudaGetLastError();
}

cudaError_t launch_oz_gemm(const OzTask* d_tasks, int ntasks, const OzSeg* d_segs, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  const size_t smem = (size_t)OZ_STAGES * (OZ_A_STAGE + OZ_B_STAGE) + OZ_EPI_WARPS * 32 * OZ_EC * sizeof(double);
  static FuncAttrs fa;
  cudaError_t e = ensure_smem(oz_gemm_kernel, smem, fa);
  if (e != cudaSuccess) return e;
  count_launch();
  oz_gemm_kernel<<<ntasks, OZ_THREADS, smem, s>>>(d_tasks, d_segs);
  return cudaGetLastError();
}

}  // namespace sgf
