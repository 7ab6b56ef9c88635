// Preconditioner application and PCG vector kernels (HBM-bound paths).
//
// apply_inverse (reference factorization.py:255-262) runs, per factor group
// (level, eliminations | compressions | final dense), batched GEMVs over the
// stored factor matrices: row-major reads for y = A x, column-coalesced reads
// with per-row-block partials for y = A^T x.  Every reduction has a fixed
// order (partials are summed in row-block order, scatter-adds into shared
// separator unknowns in ascending factor order), so results are bitwise
// reproducible run to run.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.h"
#include "ptx_util.cuh"

namespace sgf {

// ---------------------------------------------------------------------------
// y = A x for a row block (mode N).  One warp per row, lanes stride columns.
// ---------------------------------------------------------------------------
// Matrices have an even leading dimension and 16-byte aligned bases
// (pad_ld), so rows are streamed with 128-bit loads: 4 x 16 B in flight per
// lane, evict-first (each entry is read once per sweep); x stays cached.
// (256, 8): at most 32 registers so 8 CTAs = 64 warps fit per SM (the
// register limit capped residency at 4 CTAs and left HBM latency exposed).
// LPR lanes per row (8/16/32): short rows (small nodes, triangles) share a
// warp so each lane still has 4 loads in flight and the reduction is shorter.
// Triangular matrix in row pairs (task.tri == 2, rows of pair p: p and
// c1-1-p, pairs [r0, r1)): the two rows hold c1+1 entries together, so each
// warp iteration streams 4 full 16-byte loads per lane (row-per-warp leaves
// the tail of every short row latency-bound; tools/gemv_tri_bench.cu:
// +20-28% on 512..2400-row triangles).
__device__ __forceinline__ void gemv_tri_pairs(const GemvTask& T) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = T.c1;
  for (int p = T.r0 + warp; p < T.r1; p += 8) {
    const int ra = p, rb = m - 1 - p;
    const int na = (ra + 2) >> 1;  // 16-byte words covering k <= ra (A[ra][ra+1] is a stored zero)
    const int nb = (rb == ra) ? 0 : (rb + 2) >> 1;
    const double2* a = reinterpret_cast<const double2*>(T.A + (long long)ra * T.lda);
    const double2* b = reinterpret_cast<const double2*>(T.A + (long long)rb * T.lda);
    const int n = na + nb;
    const double* x = T.x;
    double sa = 0.0, sb = 0.0;
    for (int w0 = 0; w0 < n; w0 += 128) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int w = w0 + lane + 32 * u;
        v[u] = w < na ? __ldcs(a + w) : (w < n ? __ldcs(b + (w - na)) : make_double2(0.0, 0.0));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int w = w0 + lane + 32 * u;
        if (w < na) {
          const int k = 2 * w;
          sa = fma(v[u].x, x[k], sa);
          if (k + 1 <= ra) sa = fma(v[u].y, x[k + 1], sa);
        } else if (w < n) {
          const int k = 2 * (w - na);
          sb = fma(v[u].x, x[k], sb);
          if (k + 1 <= rb) sb = fma(v[u].y, x[k + 1], sb);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
      T.y[ra] = sa;
      if (rb != ra) T.y[rb] = sb;
    }
  }
}

// SPARSE: the rows' leading zeros / all-zero 256-column chunks (task.kfirst,
// task.rmask) are skipped; its own instantiation keeps the dense kernel at
// 32 registers.
template <int LPR, bool SPARSE = false>
__global__ void __launch_bounds__(256, SPARSE ? 6 : 8) gemv_n_kernel(const GemvTask* __restrict__ tasks) {
  constexpr int RPW = 32 / LPR;  // rows per warp pass
  const GemvTask T = tasks[blockIdx.x];
  if (LPR == 32 && T.tri == 2) {
    gemv_tri_pairs(T);
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane % LPR, grp = lane / LPR;
  for (int i0 = T.r0 + warp * RPW; i0 < T.r1; i0 += 8 * RPW) {  // warp-uniform
    const int i = i0 + grp;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (i < T.r1) {
      const double* arow = T.A + (long long)i * T.lda;
      const double2* a = reinterpret_cast<const double2*>(arow);
      const int ke = T.tri ? min(T.c1, i + 1) : T.c1;  // c0 == 0 for every task
      const int k2 = ke >> 1;
      const double* x = T.x;
      // leading zeros of the row (couplings E): start at the first nonzero
      // 16-byte word (the interior zero runs are left to the bulk kernel of
      // the long rows: per-iteration skips cost more than they save here)
      int k = (SPARSE && T.kfirst ? min(T.kfirst[i], ke) >> 1 : 0) + sub;
      for (; k + 3 * LPR < k2; k += 4 * LPR) {
        const double2 a0 = __ldcs(a + k), a1 = __ldcs(a + k + LPR), a2 = __ldcs(a + k + 2 * LPR),
                      a3 = __ldcs(a + k + 3 * LPR);
        s0 = fma(a0.x, x[2 * k], fma(a0.y, x[2 * k + 1], s0));
        s1 = fma(a1.x, x[2 * (k + LPR)], fma(a1.y, x[2 * (k + LPR) + 1], s1));
        s2 = fma(a2.x, x[2 * (k + 2 * LPR)], fma(a2.y, x[2 * (k + 2 * LPR) + 1], s2));
        s3 = fma(a3.x, x[2 * (k + 3 * LPR)], fma(a3.y, x[2 * (k + 3 * LPR) + 1], s3));
      }
      if (k < k2) {  // tail: up to 4 predicated loads issued together
        const double2 z = make_double2(0.0, 0.0);
        const double2 a0 = __ldcs(a + k);
        const double2 a1 = k + LPR < k2 ? __ldcs(a + k + LPR) : z;
        const double2 a2 = k + 2 * LPR < k2 ? __ldcs(a + k + 2 * LPR) : z;
        const double2 a3 = k + 3 * LPR < k2 ? __ldcs(a + k + 3 * LPR) : z;
        s0 = fma(a0.x, x[2 * k], fma(a0.y, x[2 * k + 1], s0));
        if (k + LPR < k2) s1 = fma(a1.x, x[2 * (k + LPR)], fma(a1.y, x[2 * (k + LPR) + 1], s1));
        if (k + 2 * LPR < k2) s2 = fma(a2.x, x[2 * (k + 2 * LPR)], fma(a2.y, x[2 * (k + 2 * LPR) + 1], s2));
        if (k + 3 * LPR < k2) s3 = fma(a3.x, x[2 * (k + 3 * LPR)], fma(a3.y, x[2 * (k + 3 * LPR) + 1], s3));
      }
      if ((ke & 1) && sub == 0) s0 = fma(arow[ke - 1], x[ke - 1], s0);
    }
    double s = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (i < T.r1 && sub == 0) T.y[i] = s;
  }
}

constexpr int GT_MAXROWS = 256;  // rows of a transposed task with leading-zero rows (apply.cpp GT_ROWS)

// ---------------------------------------------------------------------------
// part[k] = sum_{i in [r0,r1)} A[i,k] x[i] (mode T): each thread owns two
// adjacent columns (one 16-byte load per row), 512 columns per CTA.
// ---------------------------------------------------------------------------
// Block-sparse rows (couplings E): with task.rmask, row i's all-zero
// 32-column tiles (16 per CTA: c0 is a multiple of 512) are staged in
// shared memory as a 16-bit mask per row; with only task.kfirst, row i
// holds zeros left of kfirst[i].  A thread loads a row's entries only where
// its column pair can be nonzero; columns that are zero in every row of the
// task get an exact zero partial without reading A.  Same sums as the dense
// form: the skipped entries are exact zeros.
__global__ void __launch_bounds__(256, 5) gemv_t_lead_kernel(const GemvTask* __restrict__ tasks) {
  const GemvTask T = tasks[blockIdx.x];
  __shared__ int skf[GT_MAXROWS];  // per row: first nonzero column, or (rmask) the CTA's 16 tile bits
  __shared__ int cany;             // OR of the tile bits / min of the first nonzero columns
  const bool tiles = T.rmask != nullptr;
  const int k = T.c0 + 2 * threadIdx.x;  // c0 is even
  const int nr = T.r1 - T.r0;
  const int tb = T.c0 >> 5;              // first 32-column tile of the CTA (a multiple of 16)
  if (threadIdx.x == 0) cany = tiles ? 0 : T.c1;
  __syncthreads();
  int acc = tiles ? 0 : T.c1;
  for (int i = threadIdx.x; i < nr; i += blockDim.x) {
    int v;
    if (tiles) {
      v = (int)((T.rmask[(size_t)(T.r0 + i) * T.mwords + (tb >> 5)] >> (tb & 31)) & 0xFFFFu);
      acc |= v;
    } else {
      v = T.kfirst[T.r0 + i];
      acc = min(acc, v);
    }
    skf[i] = v;
  }
  if (tiles) {
    if (acc) atomicOr(&cany, acc);
  } else if (acc < T.c1) {
    atomicMin(&cany, acc);
  }
  __syncthreads();
  if (k >= T.c1) return;
  const int bit = 1 << (threadIdx.x >> 4);  // this thread's tile among the CTA's 16
  if (tiles ? !(cany & bit) : k + 1 < cany) {
    T.y[k] = 0.0;
    if (k + 1 < T.c1) T.y[k + 1] = 0.0;
    return;
  }
  const long long ld = T.lda;
  const double2* a = reinterpret_cast<const double2*>(T.A + k + (long long)T.r0 * ld);
  const long long ld2 = ld >> 1;
  const double2 z = make_double2(0.0, 0.0);
  double s0 = 0.0, t0 = 0.0, s1 = 0.0, t1 = 0.0;
  auto live = [&](int i) { return tiles ? (skf[i] & bit) != 0 : k + 1 >= skf[i]; };
  int i = 0;
  for (; i + 3 < nr; i += 4, a += 4 * ld2) {
    const double2 a0 = live(i) ? __ldcs(a) : z, a1 = live(i + 1) ? __ldcs(a + ld2) : z,
                  a2 = live(i + 2) ? __ldcs(a + 2 * ld2) : z, a3 = live(i + 3) ? __ldcs(a + 3 * ld2) : z;
    const double* xr = T.x + T.r0 + i;
    const double x0 = xr[0], x1 = xr[1], x2 = xr[2], x3 = xr[3];
    s0 = fma(a0.x, x0, fma(a1.x, x1, s0));
    t0 = fma(a0.y, x0, fma(a1.y, x1, t0));
    s1 = fma(a2.x, x2, fma(a3.x, x3, s1));
    t1 = fma(a2.y, x2, fma(a3.y, x3, t1));
  }
  for (; i < nr; ++i, a += ld2) {
    const double2 a0 = live(i) ? __ldcs(a) : z;
    s0 = fma(a0.x, T.x[T.r0 + i], s0);
    t0 = fma(a0.y, T.x[T.r0 + i], t0);
  }
  T.y[k] = s0 + s1;
  if (k + 1 < T.c1) T.y[k + 1] = t0 + t1;
}

__global__ void __launch_bounds__(256, 6) gemv_t_kernel(const GemvTask* __restrict__ tasks) {
  const GemvTask T = tasks[blockIdx.x];
  const int k = T.c0 + 2 * threadIdx.x;  // c0 is even
  if (k >= T.c1) return;
  int i0 = T.r0;
  // lower triangular: column k starts at row k; A[k][k+1] is a stored zero
  if (T.tri) i0 = max(i0, k);
  const long long ld = T.lda;
  const double2* a = reinterpret_cast<const double2*>(T.A + k + (long long)i0 * ld);
  const long long ld2 = ld >> 1;
  double s0 = 0.0, t0 = 0.0, s1 = 0.0, t1 = 0.0;
  int i = i0;
  for (; i + 3 < T.r1; i += 4, a += 4 * ld2) {
    const double2 a0 = __ldcs(a), a1 = __ldcs(a + ld2), a2 = __ldcs(a + 2 * ld2), a3 = __ldcs(a + 3 * ld2);
    const double x0 = T.x[i], x1 = T.x[i + 1], x2 = T.x[i + 2], x3 = T.x[i + 3];
    s0 = fma(a0.x, x0, fma(a1.x, x1, s0));
    t0 = fma(a0.y, x0, fma(a1.y, x1, t0));
    s1 = fma(a2.x, x2, fma(a3.x, x3, s1));
    t1 = fma(a2.y, x2, fma(a3.y, x3, t1));
  }
  for (; i < T.r1; ++i, a += ld2) {
    const double2 a0 = __ldcs(a);
    s0 = fma(a0.x, T.x[i], s0);
    t0 = fma(a0.y, T.x[i], t0);
  }
  T.y[k] = s0 + s1;
  if (k + 1 < T.c1) T.y[k + 1] = t0 + t1;
}

// Mode N with the matrix rows staged by the bulk copy engine (long rows,
// >= 1536 entries on average: lpr code 64; shorter rows lose more to the
// per-CTA x staging and ring start-up than they gain).  Each warp walks its rows (or row pairs of a
// triangle, tri == 2) in chunks of GB_CH entries; lane 0 keeps GB_S chunks in
// flight in the warp's ring (one mbarrier per slot) while the warp reduces
// the previous chunk against x staged in shared memory.  A row's chunks
// accumulate into one per-lane sum; the warp reduction runs at the row's end.
constexpr int GB_CH = 256, GB_S = 4, GB_XCAP = 4096;
struct GbCursor {
  int n = 0, sub = 0, off = 0;  // row (or pair) counter of the warp, row of the pair, offset in the row
  bool fresh = true;            // off not yet moved past the row's leading all-zero chunks
};
// block-sparse rows (task.rmask, staged in shared memory per task row): the
// 256-column chunk at column col (a multiple of 32) holds no nonzero
constexpr int GB_MW = 16;  // mask words per row (K <= 16384)
__device__ __forceinline__ bool gb_zero_chunk(const uint32_t* smk, int mw, int lrow, int col) {
  const int t = col >> 5, w = t >> 5, sh = t & 31;
  const uint32_t* m = smk + lrow * mw;
  uint32_t bits = m[w] >> sh;
  if (sh > 24 && w + 1 < mw) bits |= m[w + 1] << (32 - sh);
  return (bits & 0xFFu) == 0u;
}
// skip all-zero chunks, keeping the row's last chunk (every row ends with a
// chunk, whose completion writes y[row])
__device__ __forceinline__ void gb_skip(const GemvTask& T, const uint32_t* smk, int row, int start, int len,
                                        int& off) {
  while (off + GB_CH < len && gb_zero_chunk(smk, T.mwords, row - T.r0, start + off)) off += GB_CH;
}
// row index, its first column (even: 16-byte aligned; the leading zeros of a
// coupling row are skipped) and its length counted from there, for the
// cursor; false when the warp has no more rows
__device__ __forceinline__ bool gb_row(const GemvTask& T, const uint32_t* smk, int warp, GbCursor& c, int& row,
                                       int& start, int& len) {
  const int q = T.r0 + warp + 8 * c.n;
  if (q >= T.r1) return false;
  start = 0;
  if (T.tri == 2) {
    row = c.sub ? T.c1 - 1 - q : q;
    len = row + 1;
  } else {
    row = q;
    len = T.tri ? min(T.c1, q + 1) : T.c1;
    if (T.kfirst) start = min(T.kfirst[row], len) & (smk ? ~31 : ~1);  // tile-aligned with masks
    len -= start;
    if (smk && c.fresh) gb_skip(T, smk, row, start, len, c.off);
  }
  c.fresh = false;
  return true;
}
__device__ __forceinline__ void gb_advance(const GemvTask& T, const uint32_t* smk, int warp, GbCursor& c,
                                           int start, int len, int row) {
  c.off += GB_CH;
  if (c.off < len) {
    if (smk && !T.tri) gb_skip(T, smk, row, start, len, c.off);
    return;
  }
  c.off = 0;
  c.fresh = true;
  if (T.tri == 2 && c.sub == 0 && T.c1 - 1 - (T.r0 + warp + 8 * c.n) != T.r0 + warp + 8 * c.n) {
    c.sub = 1;
    return;
  }
  c.sub = 0;
  ++c.n;
}
__global__ void __launch_bounds__(256, 2) gemv_n_bulk_kernel(const GemvTask* __restrict__ tasks) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar[8 * GB_S];
  const GemvTask T = tasks[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wring = sm + warp * GB_S * GB_CH;
  double* xs = sm + 8 * GB_S * GB_CH;
  uint64_t* wbar = bar + warp * GB_S;
  const uint32_t* smk = nullptr;  // (block-sparse rows: gemv_n_bulk_sparse_kernel)
  GbCursor pc;  // producer cursor (lane 0)
  auto issue = [&](int slot) -> bool {
    int row, start, len;
    if (!gb_row(T, smk, warp, pc, row, start, len)) return false;
    if (len > 0) {
      const int cl = min(GB_CH, len - pc.off);
      const uint32_t bytes = (uint32_t)((cl + 1) & ~1) * 8u;  // even count: 16-byte multiple (ld even)
      ptx::mbar_expect_tx(&wbar[slot], bytes);
      ptx::bulk_g2s(wring + slot * GB_CH, T.A + (long long)row * T.lda + start + pc.off, bytes, &wbar[slot]);
    } else {
      ptx::mbar_arrive(&wbar[slot]);  // an all-zero row: an empty chunk
    }
    gb_advance(T, smk, warp, pc, start, len, row);
    return true;
  };
  if (lane == 0) {
    for (int s = 0; s < GB_S; ++s) ptx::mbar_init(&wbar[s], 1);
    ptx::mbar_init_fence();
    for (int s = 0; s < GB_S; ++s)
      if (!issue(s)) break;
  }
  const bool sx = T.c1 <= GB_XCAP;
  for (int i = threadIdx.x; i < T.c1 && sx; i += 256) xs[i] = T.x[i];
  __syncthreads();
  const double* xv = sx ? xs : T.x;
  GbCursor cc;  // consumer cursor
  double acc = 0.0;
  for (int it = 0;; ++it) {
    int row, start, len;
    if (!gb_row(T, smk, warp, cc, row, start, len)) break;
    const int slot = it % GB_S;
    const int off = cc.off, cl = min(GB_CH, len - off);
    ptx::mbar_wait(&wbar[slot], (it / GB_S) & 1);
    const double* ch = wring + slot * GB_CH;
    const double* xo = xv + start + off;
#pragma unroll
    for (int t = 0; t < GB_CH / 64; ++t) {
      const int j = 64 * t + 2 * lane;
      if (j < cl) {
        const double2 g = *reinterpret_cast<const double2*>(ch + j);
        acc = fma(g.x, xo[j], acc);
        if (j + 1 < cl) acc = fma(g.y, xo[j + 1], acc);
      }
    }
    __syncwarp();
    if (lane == 0) issue(slot);
    if (off + GB_CH >= len) {  // row complete
      double s = acc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) T.y[row] = s;
      acc = 0.0;
    }
    gb_advance(T, smk, warp, cc, start, len, row);
  }
}

// Mode N over block-sparse rows (couplings E, masked L^{-1} rows: task.kfirst,
// task.rmask) with the rows staged by the bulk copy engine.  All-zero
// 32-column tiles are skipped at tile granularity: a chunk runs from the next
// nonzero tile to the last nonzero tile among the 8 tiles starting there (one
// bulk copy of 256 B .. 2 KB), so what is streamed is within a few percent of
// the nonzero tiles' bytes (cfg4 level 3: 2.78 GB against 2.57 GB nonzero and
// 3.74 GB with whole 256-column chunks).  Rows differ widely in length, so
// the warps of a CTA take rows from a shared counter instead of a fixed
// stride (a fixed assignment left warps idle behind the longest row), and the
// producer lane passes each slot's (row, column, count, last) to the consumer
// in shared memory next to the data.  A row is reduced by one warp in chunk
// order, so the sums do not depend on which warp takes it.
struct GbMeta {
  int row, col, cl, last;
};
__global__ void __launch_bounds__(256, 2) gemv_n_bulk_sparse_kernel(const GemvTask* __restrict__ tasks) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar[8 * GB_S];
  __shared__ GbMeta meta[8 * GB_S];
  __shared__ uint32_t smk[64 * GB_MW];
  __shared__ int next_row;
  const GemvTask T = tasks[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wring = sm + warp * GB_S * GB_CH;
  double* xs = sm + 8 * GB_S * GB_CH;
  uint64_t* wbar = bar + warp * GB_S;
  GbMeta* wmeta = meta + warp * GB_S;
  const int nr = T.r1 - T.r0, mw = T.mwords;
  const bool masked = T.rmask && nr <= 64 && mw <= GB_MW;
  if (masked)
    for (int i = threadIdx.x; i < nr * mw; i += 256) smk[i] = T.rmask[(size_t)T.r0 * mw + i];
  if (threadIdx.x == 0) next_row = 0;
  __syncthreads();
  // producer state (lane 0): the current row, its length, its tile count and
  // the next tile to read (-1: the row is finished, take another)
  int prow = -1, prlen = 0, pnt = 0, pnext = -1;
  // first tile >= t of row `row` holding a nonzero (-1: none left)
  auto next_tile = [&](int row, int t, int nt) -> int {
    if (t >= nt) return -1;
    if (!masked) return t;
    const uint32_t* m = smk + row * mw;
    for (int w = t >> 5; w < mw && 32 * w < nt; ++w) {
      uint32_t bits = m[w];
      if (w == (t >> 5)) bits &= 0xFFFFFFFFu << (t & 31);
      if (bits) {
        const int r = 32 * w + __ffs(bits) - 1;
        return r < nt ? r : -1;
      }
    }
    return -1;
  };
  // A chunk is the run from the next nonzero tile to the last nonzero tile
  // among the 8 tiles starting there: zero tiles are skipped at tile (256 B)
  // granularity, one bulk copy per chunk.
  auto issue = [&](int slot) {
    GbMeta& md = wmeta[slot];
    if (pnext < 0) {
      const int r = atomicAdd(&next_row, 1);
      if (r >= nr) {  // no rows left: a sentinel slot
        prow = -1;
        md.row = -1;
        ptx::mbar_arrive(&wbar[slot]);
        return;
      }
      prow = r;
      prlen = T.tri ? min(T.c1, T.r0 + r + 1) : T.c1;  // lower-triangular rows end at the diagonal
      pnt = (prlen + 31) >> 5;
      pnext = next_tile(r, T.kfirst ? min(T.kfirst[T.r0 + r], prlen) >> 5 : 0, pnt);
      if (pnext < 0) {  // an all-zero row: an empty chunk that writes y[row] = 0
        md.row = prow;
        md.col = 0;
        md.cl = 0;
        md.last = 1;
        ptx::mbar_arrive(&wbar[slot]);
        return;
      }
    }
    const int t0 = pnext;
    int cnt = min(GB_CH / 32, pnt - t0);
    if (masked) {
      const uint32_t* m = smk + prow * mw;
      const int w = t0 >> 5, sh = t0 & 31;
      uint32_t bits = m[w] >> sh;
      if (sh > 24 && w + 1 < mw) bits |= m[w + 1] << (32 - sh);
      bits &= (1u << cnt) - 1u;  // bit 0 (tile t0) is set
      cnt = 32 - __clz(bits);
    }
    pnext = next_tile(prow, t0 + cnt, pnt);
    const int col = 32 * t0;
    const int cl = min(32 * cnt, prlen - col);
    md.row = prow;
    md.col = col;
    md.cl = cl;
    md.last = pnext < 0;
    const uint32_t bytes = (uint32_t)((cl + 1) & ~1) * 8u;  // even count: 16-byte multiple (ld even)
    ptx::mbar_expect_tx(&wbar[slot], bytes);
    ptx::bulk_g2s(wring + slot * GB_CH, T.A + (long long)(T.r0 + prow) * T.lda + col, bytes, &wbar[slot]);
  };
  if (lane == 0) {
    for (int s = 0; s < GB_S; ++s) ptx::mbar_init(&wbar[s], 1);
    ptx::mbar_init_fence();
    for (int s = 0; s < GB_S; ++s) issue(s);
  }
  const bool sx = T.c1 <= GB_XCAP;
  for (int i = threadIdx.x; i < T.c1 && sx; i += 256) xs[i] = T.x[i];
  __syncthreads();
  const double* xv = sx ? xs : T.x;
  double acc = 0.0;
  for (int it = 0;; ++it) {
    const int slot = it % GB_S;
    ptx::mbar_wait(&wbar[slot], (it / GB_S) & 1);
    const GbMeta md = wmeta[slot];
    if (md.row < 0) break;
    const double* ch = wring + slot * GB_CH;
    const double* xo = xv + md.col;
#pragma unroll
    for (int t = 0; t < GB_CH / 64; ++t) {
      const int j = 64 * t + 2 * lane;
      if (j < md.cl) {
        const double2 g = *reinterpret_cast<const double2*>(ch + j);
        acc = fma(g.x, xo[j], acc);
        if (j + 1 < md.cl) acc = fma(g.y, xo[j + 1], acc);
      }
    }
    __syncwarp();
    if (lane == 0) issue(slot);
    if (md.last) {  // row complete
      double sum = acc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) T.y[T.r0 + md.row] = sum;
      acc = 0.0;
    }
  }
}

// Mode N over block-sparse rows, tile lists (the default for masked rows):
// one warp per row; the row's nonzero 32-column tiles are compacted into a
// per-warp list in shared memory (from the row's tile mask: popcount prefix
// over the mask words, one lane per word), and the warp then streams only
// those tiles, a half warp per tile (16 lanes x 16 B = one 256-byte tile), 4
// loads in flight per lane, evict-first.  Every load that is issued fetches
// nonzero data, so the bytes in flight per SM do not drop with the rows'
// density (the bulk-copy ring above issues one copy per chunk and a chunk
// shrinks with the density: 4.2 TB/s on the cfg4 level-3 couplings against
// 6.2 TB/s of the transposed sweep over the same tiles).  Fixed lane
// assignment and iteration order: the sums do not depend on scheduling.
constexpr int GTL_CAP = 512;  // tiles per row (K <= 16384, mwords <= 16)
__global__ void __launch_bounds__(256, 6) gemv_n_tiles_kernel(const GemvTask* __restrict__ tasks) {
  __shared__ uint16_t tl[8][GTL_CAP];
  const GemvTask T = tasks[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, l16 = lane & 15;
  const int mw = T.mwords;
  const bool listed = T.rmask && mw <= GTL_CAP / 32;
  uint16_t* wl = tl[warp];
  const double* __restrict__ x = T.x;
  for (int row = T.r0 + warp; row < T.r1; row += 8) {  // warp-uniform
    const int rlen = T.tri ? min(T.c1, row + 1) : T.c1;
    const int nt = (rlen + 31) >> 5;
    int total, tfirst = 0;
    if (listed) {
      uint32_t word = 0;
      if (lane < mw && 32 * lane < nt) {
        word = T.rmask[(size_t)row * mw + lane];
        if (nt - 32 * lane < 32) word &= (1u << (nt - 32 * lane)) - 1u;
      }
      const int cnt = __popc(word);
      int pre = cnt;  // inclusive prefix over the lanes (mask words)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += v;
      }
      total = __shfl_sync(0xffffffffu, pre, 31);
      int at = pre - cnt;
      __syncwarp();  // the previous row's list has been read
      while (word) {
        wl[at++] = (uint16_t)(32 * lane + __ffs(word) - 1);
        word &= word - 1;
      }
      __syncwarp();
    } else {
      tfirst = T.kfirst ? min(T.kfirst[row], rlen) >> 5 : 0;
      total = nt - tfirst;
    }
    const double2* a = reinterpret_cast<const double2*>(T.A + (long long)row * T.lda) + l16;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int j0 = half; j0 < total; j0 += 8) {
      int c[4];
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + 2 * u;
        c[u] = -1;
        v[u] = make_double2(0.0, 0.0);
        if (j < total) {
          const int t = listed ? (int)wl[j] : tfirst + j;
          const int col = 32 * t + 2 * l16;
          if (col < rlen) {
            c[u] = col;
            v[u] = __ldcs(a + 16 * t);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (c[u] >= 0) {
          double acc = u == 0 ? s0 : (u == 1 ? s1 : (u == 2 ? s2 : s3));
          acc = fma(v[u].x, x[c[u]], acc);
          if (c[u] + 1 < rlen) acc = fma(v[u].y, x[c[u] + 1], acc);
          if (u == 0) s0 = acc;
          else if (u == 1) s1 = acc;
          else if (u == 2) s2 = acc;
          else s3 = acc;
        }
      }
    }
    double sum = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) T.y[row] = sum;
  }
}

cudaError_t launch_gemv(const GemvTask* d_tasks, int ntasks, int mode, cudaStream_t s, int lpr) {
  if (ntasks <= 0) return cudaSuccess;
  count_launch();
  static const int bulk = getenv("SGF_GEMV_BULK") ? atoi(getenv("SGF_GEMV_BULK")) : 1;
  if ((mode == 0 || mode == 3) && lpr == 64 && bulk) {
    const size_t smem = ((size_t)8 * GB_S * GB_CH + GB_XCAP) * sizeof(double);
    static FuncAttrs fa, fa_sp;
    static const int sparse_ring = getenv("SGF_GEMV_SPARSE_RING") ? atoi(getenv("SGF_GEMV_SPARSE_RING")) : 0;
    if (mode == 3 && !sparse_ring) {  // block-sparse rows: per-row tile lists
      gemv_n_tiles_kernel<<<ntasks, 256, 0, s>>>(d_tasks);
      return cudaGetLastError();
    }
    if (mode == 3) {  // the bulk-copy ring over block-sparse rows
      cudaError_t e = ensure_smem(gemv_n_bulk_sparse_kernel, smem, fa_sp);
      if (e != cudaSuccess) return e;
      gemv_n_bulk_sparse_kernel<<<ntasks, 256, smem, s>>>(d_tasks);
      return cudaGetLastError();
    }
    cudaError_t e = ensure_smem(gemv_n_bulk_kernel, smem, fa);
    if (e != cudaSuccess) return e;
    gemv_n_bulk_kernel<<<ntasks, 256, smem, s>>>(d_tasks);
    return cudaGetLastError();
  }
  if (lpr == 64) lpr = 32;
  if (mode == 0) {
    if (lpr == 8) gemv_n_kernel<8><<<ntasks, 256, 0, s>>>(d_tasks);
    else if (lpr == 16) gemv_n_kernel<16><<<ntasks, 256, 0, s>>>(d_tasks);
    else gemv_n_kernel<32><<<ntasks, 256, 0, s>>>(d_tasks);
  } else if (mode == 3) {  // mode N, block-sparse rows (task.kfirst / task.rmask)
    if (lpr == 8) gemv_n_kernel<8, true><<<ntasks, 256, 0, s>>>(d_tasks);
    else if (lpr == 16) gemv_n_kernel<16, true><<<ntasks, 256, 0, s>>>(d_tasks);
    else gemv_n_kernel<32, true><<<ntasks, 256, 0, s>>>(d_tasks);
  } else if (mode == 2) {  // transposed, rows with leading zeros (task.kfirst, <= GT_MAXROWS rows)
    gemv_t_lead_kernel<<<ntasks, 256, 0, s>>>(d_tasks);
  } else {
    gemv_t_kernel<<<ntasks, 256, 0, s>>>(d_tasks);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Symmetric GEMV from the lower triangle, one CTA per matrix (m <= 64*Q).
// Warp w takes the row pairs (p, m-1-p), p = w (mod 8): the two rows hold
// m+1 entries together, so every pair issues the same Q+1 16-byte loads per
// lane at once.  Lane l owns the column pairs 64q + 2l + {0,1}; slot s of a
// pair reads column block q = s of row p, or q = Q-s of row m-1-p (the two
// ranges never collide), so the column accumulators are indexed at compile
// time and stay in registers.  Each stored entry is read once and used
// twice: G_ij x_j into the row sum of i (warp reduction), G_ij x_i into the
// lane's column sums of j (strictly lower part).  The 8 warps' column sums
// are added in fixed order through shared memory at the end.
// ---------------------------------------------------------------------------
#ifndef SYMV_MINB
#define SYMV_MINB 2
#endif
template <int Q>
__global__ void __launch_bounds__(256, SYMV_MINB) symv_kernel(const SymvTask* __restrict__ tasks) {
  extern __shared__ double sm[];
  constexpr int MP = 64 * Q;
  const SymvTask T = tasks[blockIdx.x];
  const int m = T.m;
  double* xs = sm;
  double* yr = sm + MP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < MP; i += 256) xs[i] = i < m ? T.x[i] : 0.0;
  __syncthreads();
  double c0[Q], c1[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) c0[q] = c1[q] = 0.0;
  const int npairs = (m + 1) / 2;
  for (int p = warp; p < npairs; p += 8) {
    const int ra = p, rb = m - 1 - p;  // rb == ra for the middle row of an odd m
    const int qa = (ra >> 6) + 1, qb = (rb == ra) ? 0 : (rb >> 6) + 1;
    const double* rowa = T.G + (long long)ra * T.ld;
    const double* rowb = T.G + (long long)rb * T.ld;
    double2 g[Q + 1];
#pragma unroll
    for (int s = 0; s <= Q; ++s) {
      const bool isa = s < qa;
      const int q = isa ? s : Q - s;
      const int j = 64 * q + 2 * lane;
      const bool ok = isa ? (j <= ra) : (q < qb && j <= rb);
      g[s] = ok ? __ldcs(reinterpret_cast<const double2*>((isa ? rowa : rowb) + j)) : make_double2(0.0, 0.0);
    }
    const double xa = xs[ra], xb = xs[rb];
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int s = 0; s <= Q; ++s) {
      if (s < qa) {
        if (s < Q) {
          const int j = 64 * s + 2 * lane;
          if (j <= ra) {
            const double g0 = g[s].x, g1 = (j + 1 <= ra) ? g[s].y : 0.0;  // G[i][i+1] is not stored
            sa = fma(g0, xs[j], fma(g1, xs[j + 1], sa));
            if (j < ra) c0[s] = fma(g0, xa, c0[s]);
            if (j + 1 < ra) c1[s] = fma(g1, xa, c1[s]);
          }
        }
      } else if (s >= 1 && Q - s < qb) {
        constexpr int dummy = 0;
        (void)dummy;
        const int q = Q - s;
        const int j = 64 * q + 2 * lane;
        if (j <= rb) {
          const double g0 = g[s].x, g1 = (j + 1 <= rb) ? g[s].y : 0.0;
          sb = fma(g0, xs[j], fma(g1, xs[j + 1], sb));
          if (j < rb) c0[Q - s] = fma(g0, xb, c0[Q - s]);
          if (j + 1 < rb) c1[Q - s] = fma(g1, xb, c1[Q - s]);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
      yr[ra] = sa;
      if (rb != ra) yr[rb] = sb;
    }
  }
  double* cp = sm + 2 * MP + warp * MP;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    cp[64 * q + 2 * lane] = c0[q];
    cp[64 * q + 2 * lane + 1] = c1[q];
  }
  __syncthreads();
  const double* cpa = sm + 2 * MP;
  for (int j = threadIdx.x; j < m; j += 256) {
    double c = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += cpa[w * MP + j];
    const double v = yr[j] + c;
    T.y[j] = T.base ? fma(T.sign, v, T.base[j]) : T.sign * v;
  }
}

// Same arithmetic (bitwise identical results), rows staged by the bulk copy
// engine: every warp owns a ring of S pair slots in shared memory and its
// lane 0 keeps S row pairs (two cp.async.bulk each, one mbarrier per slot)
// in flight while the warp reduces the previous pair from shared memory.
// With no operand registers the kernel fits 3 CTAs per SM at Q = 8, S = 2
// (~200 KB of G in flight per SM, against ~70 KB issued by the register
// version, whose loads also wait behind each pair's reduction).
template <int Q, int S>
__global__ void __launch_bounds__(256, 3) symv_bulk_kernel(const SymvTask* __restrict__ tasks, double* __restrict__ v) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar[8 * S];
  constexpr int MP = 64 * Q;
  constexpr int SLOT = MP + 2;  // doubles per pair: row a (even length) then row b
  const SymvTask T = tasks[blockIdx.x];
  const int m = T.m;
  const long long ld = T.ld;
  double* xs = sm;
  double* yr = sm + MP;
  double* ring = sm + 2 * MP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wring = ring + warp * S * SLOT;
  uint64_t* wbar = bar + warp * S;
  const int npairs = (m + 1) / 2;
  auto issue = [&](int p, int s) {
    const int ra = p, rb = m - 1 - p;
    const uint32_t na = (uint32_t)((ra + 2) & ~1), nb = (rb == ra) ? 0u : (uint32_t)((rb + 2) & ~1);
    ptx::mbar_expect_tx(&wbar[s], (na + nb) * 8u);
    ptx::bulk_g2s(wring + s * SLOT, T.G + (long long)ra * ld, na * 8u, &wbar[s]);
    if (nb) ptx::bulk_g2s(wring + s * SLOT + na, T.G + (long long)rb * ld, nb * 8u, &wbar[s]);
  };
  if (lane == 0) {
    for (int s = 0; s < S; ++s) ptx::mbar_init(&wbar[s], 1);
    ptx::mbar_init_fence();
    for (int s = 0; s < S; ++s)
      if (warp + 8 * s < npairs) issue(warp + 8 * s, s);
  }
  for (int i = threadIdx.x; i < MP; i += 256) xs[i] = i < m ? ((v && T.gather_x) ? v[T.idx[i]] : T.x[i]) : 0.0;
  __syncthreads();
  double c0[Q], c1[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) c0[q] = c1[q] = 0.0;
  int it = 0;
  for (int p = warp; p < npairs; p += 8, ++it) {
    const int s = it % S;
    const int ra = p, rb = m - 1 - p;
    const int qa = (ra >> 6) + 1, qb = (rb == ra) ? 0 : (rb >> 6) + 1;
    const double* rowa = wring + s * SLOT;
    const double* rowb = rowa + ((ra + 2) & ~1);
    ptx::mbar_wait(&wbar[s], (it / S) & 1);
    const double xa = xs[ra], xb = xs[rb];
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int t = 0; t <= Q; ++t) {
      if (t < qa) {
        if (t < Q) {
          const int j = 64 * t + 2 * lane;
          if (j <= ra) {
            const double2 g = *reinterpret_cast<const double2*>(rowa + j);
            const double g0 = g.x, g1 = (j + 1 <= ra) ? g.y : 0.0;
            sa = fma(g0, xs[j], fma(g1, xs[j + 1], sa));
            if (j < ra) c0[t] = fma(g0, xa, c0[t]);
            if (j + 1 < ra) c1[t] = fma(g1, xa, c1[t]);
          }
        }
      } else if (t >= 1 && Q - t < qb) {
        const int q = Q - t;
        const int j = 64 * q + 2 * lane;
        if (j <= rb) {
          const double2 g = *reinterpret_cast<const double2*>(rowb + j);
          const double g0 = g.x, g1 = (j + 1 <= rb) ? g.y : 0.0;
          sb = fma(g0, xs[j], fma(g1, xs[j + 1], sb));
          if (j < rb) c0[q] = fma(g0, xb, c0[q]);
          if (j + 1 < rb) c1[q] = fma(g1, xb, c1[q]);
        }
      }
    }
    __syncwarp();  // every lane has read the slot
    if (lane == 0 && p + 8 * S < npairs) issue(p + 8 * S, s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
      yr[ra] = sa;
      if (rb != ra) yr[rb] = sb;
    }
  }
  __syncthreads();  // the column partials reuse the ring
  double* cp = ring + warp * MP;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    cp[64 * q + 2 * lane] = c0[q];
    cp[64 * q + 2 * lane + 1] = c1[q];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < m; j += 256) {
    double c = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) c += ring[w * MP + j];
    const double r = yr[j] + c;
    if (v) {  // fused: base from and result to the full vector (this node's unknowns only)
      const int u = T.idx[j];
      v[u] = T.base ? fma(T.sign, r, v[u]) : T.sign * r;
    } else {
      T.y[j] = T.base ? fma(T.sign, r, T.base[j]) : T.sign * r;
    }
  }
}

template <int Q, int S>
static cudaError_t symv_bulk_q(const SymvTask* d_tasks, int ntasks, cudaStream_t s, double* v = nullptr) {
  // ring (8 warps x S slots) also holds the 8 x MP column partials at the end
  const size_t ring = (size_t)8 * std::max(S * (64 * Q + 2), 64 * Q);
  const size_t smem = (2 * (size_t)64 * Q + ring) * sizeof(double);
  static FuncAttrs fa;
  cudaError_t e = ensure_smem(symv_bulk_kernel<Q, S>, smem, fa);
  if (e != cudaSuccess) return e;
  count_launch(); symv_bulk_kernel<Q, S><<<ntasks, 256, smem, s>>>(d_tasks, v);
  return cudaGetLastError();
}

template <int Q>
static cudaError_t symv_q(const SymvTask* d_tasks, int ntasks, cudaStream_t s) {
  const size_t smem = (size_t)10 * 64 * Q * sizeof(double);
  static FuncAttrs fa;
  cudaError_t e = ensure_smem(symv_kernel<Q>, smem, fa);
  if (e != cudaSuccess) return e;
  count_launch(); symv_kernel<Q><<<ntasks, 256, smem, s>>>(d_tasks);
  return cudaGetLastError();
}

static int symv_variant() {
  static const int variant = getenv("SGF_SYMV") ? atoi(getenv("SGF_SYMV")) : 1;
  return variant;
}

bool symv_fused_ok(int max_m) { return symv_variant() == 1 && max_m <= 768; }

cudaError_t launch_symv_fused(const SymvTask* d_tasks, int ntasks, int max_m, double* v, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  if (max_m <= 128) return symv_bulk_q<2, 4>(d_tasks, ntasks, s, v);
  if (max_m <= 256) return symv_bulk_q<4, 3>(d_tasks, ntasks, s, v);
  if (max_m <= 512) return symv_bulk_q<8, 2>(d_tasks, ntasks, s, v);
  if (max_m <= 768) return symv_bulk_q<12, 2>(d_tasks, ntasks, s, v);
  return cudaErrorInvalidValue;
}

cudaError_t launch_symv(const SymvTask* d_tasks, int ntasks, int max_m, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  if (symv_variant() == 1) {
    if (max_m <= 128) return symv_bulk_q<2, 4>(d_tasks, ntasks, s);
    if (max_m <= 256) return symv_bulk_q<4, 3>(d_tasks, ntasks, s);
    if (max_m <= 512) return symv_bulk_q<8, 2>(d_tasks, ntasks, s);
    if (max_m <= 768) return symv_bulk_q<12, 2>(d_tasks, ntasks, s);
  }
  if (max_m <= 128) return symv_q<2>(d_tasks, ntasks, s);
  if (max_m <= 256) return symv_q<4>(d_tasks, ntasks, s);
  if (max_m <= 512) return symv_q<8>(d_tasks, ntasks, s);
  if (max_m <= 768) return symv_q<12>(d_tasks, ntasks, s);
  if (max_m <= 1024) return symv_q<16>(d_tasks, ntasks, s);
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Level-1 groups through the banded Cholesky factor.  A lexicographic 8^3
// interior has bandwidth 64, so in 64 x 64 blocks L is block bidiagonal:
// diagonal blocks L_pp and sub-diagonal blocks S_p = L_{p,p-1}, which hold
// nonzeros only at column >= row (bandwidth <= 64).  The diagonal blocks of
// X = L^{-1} are the inverses of the L_pp, so
//   forward   w_p = X_pp (x_p - S_p w_{p-1}),            p = 0 .. nb-1
//   backward  v_p = X_pp^T (w_p - S_{p+1}^T v_{p+1}),    p = nb-1 .. 0
// gives v = L^{-T} L^{-1} x = G x from 2 x 15 block products per 512-unknown
// node: ~0.6 MB streamed (16-column granularity on the triangles) instead of
// the 1.05 MB of G's lower triangle.  One CTA per node; the vector lives in
// shared memory.  Row products: thread (row, quarter) reads 16 entries of its
// row with 16-byte loads, 4-lane shuffle reduction.  Transposed products:
// thread (column, row quarter) reads 16 rows of its column (a warp reads 256
// contiguous bytes per row), partials summed in fixed order through shared
// memory.  A block's entries are requested before the barrier that publishes
// the previous product (their addresses do not depend on the solve).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 4) l1_band_kernel(const SymvTask* __restrict__ tasks, double* __restrict__ v) {
  __shared__ __align__(16) double xs[L1B_MAXM];
  __shared__ __align__(16) double tv[64];
  __shared__ double part[4][64];
  const SymvTask T = tasks[blockIdx.x];
  const int m = T.m, tid = threadIdx.x;
  const long long ld = T.ld;
  const int nb = (m + 63) >> 6;
  for (int i = tid; i < 64 * nb; i += 256) xs[i] = i < m ? ((v && T.gather_x) ? v[T.idx[i]] : T.x[i]) : 0.0;
  __syncthreads();
  const int r = tid >> 2, qd = tid & 3;   // row products: row, column quarter
  const int cc = tid & 63, rq = tid >> 6;  // transposed products: column, row quarter
  double a[16];
  // thread (r, qd) loads the 16-byte words 4k + qd (k = 0..7) of row r of a
  // row-major block -- the four threads of a row read 64 contiguous bytes per
  // instruction and their shared-memory operands do not collide -- and only
  // the words that touch columns [lo, hi] (zeros elsewhere)
  auto load_row = [&](const double* B, int lo, int hi) {
    const double2* src = reinterpret_cast<const double2*>(B + (long long)r * ld) + qd;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c0 = 8 * k + 2 * qd;
      double2 t = make_double2(0.0, 0.0);
      if (c0 + 1 >= lo && c0 <= hi) t = __ldcs(src + 4 * k);
      a[2 * k] = t.x;
      a[2 * k + 1] = t.y;
    }
  };
  // sum over the thread's words of a[] * vec[columns <= cmax]
  auto dot_row = [&](const double* vec, int cmax) {
    const double2* w2 = reinterpret_cast<const double2*>(vec) + qd;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c0 = 8 * k + 2 * qd;
      const double2 w = w2[4 * k];
      if (c0 <= cmax) acc = fma(a[2 * k], w.x, acc);
      if (c0 + 1 <= cmax) acc = fma(a[2 * k + 1], w.y, acc);
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    return acc;
  };
  // thread (cc, rq) loads B[16rq .. 16rq+15][cc], rows in [lo, hi] only
  auto load_col = [&](const double* B, int lo, int hi) {
    const double* src = B + (long long)(16 * rq) * ld + cc;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int row = 16 * rq + j;
      a[j] = (row >= lo && row <= hi) ? __ldcs(src) : 0.0;
      src += ld;
    }
  };
  // ---- forward: L w = x ----
  for (int p = 0; p < nb; ++p) {
    const int rows = min(64, m - 64 * p);
    if (p > 0) {
      // t = x_p - S_p w_{p-1}: row r of S_p holds nonzeros at columns >= r
      load_row(T.L + (long long)(64 * p) * ld + 64 * (p - 1), r < rows ? r : 64, 63);
      const double acc = dot_row(xs + 64 * (p - 1), 63);
      if (qd == 0 && r < rows) tv[r] = xs[64 * p + r] - acc;
    } else if (tid < rows) {
      tv[tid] = xs[tid];
    }
    // w_p = X_pp t: lower triangle, row r uses columns <= r
    load_row(T.X + (long long)(64 * p) * ld + 64 * p, 0, r < rows ? r : -1);
    __syncthreads();
    {
      const double acc = dot_row(tv, r);
      if (qd == 0 && r < rows) xs[64 * p + r] = acc;
    }
    __syncthreads();
  }
  // ---- backward: L^T v = w ----
  for (int p = nb - 1; p >= 0; --p) {
    const int rows = min(64, m - 64 * p);
    if (p < nb - 1) {
      // u = w_p - S_{p+1}^T v_{p+1}: column cc of S_{p+1} holds nonzeros at rows <= cc
      const int rows1 = min(64, m - 64 * (p + 1));
      load_col(T.L + (long long)(64 * (p + 1)) * ld + 64 * p, 0, min(cc, rows1 - 1));
      const double* vv = xs + 64 * (p + 1) + 16 * rq;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 16; ++j) acc = fma(a[j], vv[j], acc);
      part[rq][cc] = acc;
      __syncthreads();
      if (tid < rows) tv[tid] = xs[64 * p + tid] - (((part[0][tid] + part[1][tid]) + part[2][tid]) + part[3][tid]);
    } else if (tid < rows) {
      tv[tid] = xs[64 * p + tid];
    }
    // v_p = X_pp^T u: column cc uses rows >= cc (< rows)
    load_col(T.X + (long long)(64 * p) * ld + 64 * p, cc < rows ? cc : 64, rows - 1);
    __syncthreads();
    {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int row = 16 * rq + j;
        if (row >= cc && row < rows) acc = fma(a[j], tv[row], acc);
      }
      part[rq][cc] = acc;
    }
    __syncthreads();
    if (tid < rows) xs[64 * p + tid] = ((part[0][tid] + part[1][tid]) + part[2][tid]) + part[3][tid];
    __syncthreads();
  }
  for (int j = tid; j < m; j += 256) {
    const double rr = xs[j];
    if (v) {  // fused: base from and result to the full vector (this node's unknowns only)
      const int u = T.idx[j];
      v[u] = T.base ? fma(T.sign, rr, v[u]) : T.sign * rr;
    } else {
      T.y[j] = T.base ? fma(T.sign, rr, T.base[j]) : T.sign * rr;
    }
  }
}

cudaError_t launch_l1_band(const SymvTask* d_tasks, int ntasks, double* v, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  count_launch();
  l1_band_kernel<<<ntasks, 256, 0, s>>>(d_tasks, v);  // (5 or 6 CTAs per SM: no faster; 6 spills)
  return cudaGetLastError();
}

// short sparse rows (level-1 couplings: 1-3 entries per row), thread per row
__global__ void sub_spmv_kernel(int nrows, const int* __restrict__ rid, const int* __restrict__ rp,
                                const int* __restrict__ ci, const double* __restrict__ v, double* __restrict__ x,
                                double* __restrict__ out, int mode) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int e = rp[r]; e < rp[r + 1]; ++e) s = fma(v[e], x[ci[e]], s);
    if (mode == 0) x[rid[r]] -= s;
    else out[r] = s;
  }
}

cudaError_t launch_sub_spmv(int nrows, const int* rid, const int* rp, const int* ci, const double* v, double* x,
                            double* out, int mode, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  int blocks = (nrows + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  count_launch(); sub_spmv_kernel<<<blocks, 256, 0, s>>>(nrows, rid, rp, ci, v, x, out, mode);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// out[o] = sign_base*base[o] - sum_{q<nrb} part[poff + q*stride + k]  for the
// flat segment layout described by RedSeg (one CTA-chunk per 256 entries).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) reduce_parts_kernel(const RedSeg* __restrict__ segs, double* __restrict__ v) {
  const RedSeg R = segs[blockIdx.y];
  const int k = blockIdx.x * 256 + threadIdx.x;
  if (k >= R.n) return;
  double s = 0.0;
  for (int q = 0; q < R.nrb; ++q) s += R.part[(long long)q * R.stride + k];
  const double b = R.base ? R.base[k] : 0.0;
  if (v && R.idx) v[R.idx[k]] = b + R.sign * s;  // fused scatter into the full vector
  else R.out[k] = b + R.sign * s;
}

cudaError_t launch_reduce_parts(const void* d_segs, int nseg, int max_n, cudaStream_t s, double* v) {
  if (nseg <= 0 || max_n <= 0) return cudaSuccess;
  dim3 grid((max_n + 255) / 256, nseg);
  count_launch(); reduce_parts_kernel<<<grid, 256, 0, s>>>((const RedSeg*)d_segs, v);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// gathers / scatters over int32 index lists
// ---------------------------------------------------------------------------
__global__ void gather_kernel(const double* __restrict__ x, const int* __restrict__ idx, double* __restrict__ out,
                              long long n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    out[e] = x[idx[e]];
}
__global__ void scatter_kernel(const double* __restrict__ v, const int* __restrict__ idx, double* __restrict__ x,
                               long long n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    x[idx[e]] = v[e];
}
// x[tgt[u]] -= t[pos[j]] (add = 0) or += (add = 1) for j in [ptr[u], ptr[u+1])
// in order (ascending factor)
__global__ void combine_kernel(double* __restrict__ x, const int* __restrict__ tgt, const long long* __restrict__ ptr,
                               const long long* __restrict__ pos, const double* __restrict__ t, long long nt,
                               int add) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < nt; u += (long long)gridDim.x * blockDim.x) {
    double v = x[tgt[u]];
    if (add)
      for (long long j = ptr[u]; j < ptr[u + 1]; ++j) v += t[pos[j]];
    else
      for (long long j = ptr[u]; j < ptr[u + 1]; ++j) v -= t[pos[j]];
    x[tgt[u]] = v;
  }
}

static inline unsigned grid_for(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (unsigned)b;
}

cudaError_t launch_gather(const double* x, const int* idx, double* out, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch(); gather_kernel<<<grid_for(n), 256, 0, s>>>(x, idx, out, n);
  return cudaGetLastError();
}
cudaError_t launch_scatter(const double* v, const int* idx, double* x, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  count_launch(); scatter_kernel<<<grid_for(n), 256, 0, s>>>(v, idx, x, n);
  return cudaGetLastError();
}
cudaError_t launch_combine(double* x, const int* tgt, const long long* ptr, const long long* pos, const double* t,
                           long long nt, cudaStream_t s, int add) {
  if (nt <= 0) return cudaSuccess;
  count_launch(); combine_kernel<<<grid_for(nt), 256, 0, s>>>(x, tgt, ptr, pos, t, nt, add);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// PCG vector kernels (reference krylov.py:34-102).  Dots use a fixed grid and
// a fixed-order final reduction: bitwise reproducible.
// ---------------------------------------------------------------------------
constexpr int RED_BLOCKS = 296;
// Partial buffer of the PCG reductions (PCG_PART doubles, runtime.h): block
// partials, and at PCG_CNT_OFF the arrival counter of the in-kernel final
// reduction (zero between launches: the finishing block resets it).
constexpr int RED_MAX = PCG_CNT_OFF;  // most partials a reducing launch may write

// CSR SpMV y = A x (b == nullptr) or y = b - A x.  One warp per 32
// consecutive rows: the warp streams the rows' contiguous nonzero range in
// chunks of 256 with fully coalesced, independent loads (8 per lane in flight),
// stages the products v[e] * x[ci[e]] in shared memory, and every lane then
// sums its own row in storage order -- the sequential order of the reference's
// CSR product (scipy), so the result does not depend on the launch shape.
constexpr int SPMV_CH = 256;
constexpr int SPMV_WARPS = 8;
__device__ void block_partial_finish(double v, double* part, double* out, int slot);
// DOT: also x.y (p'Ap of PCG) -- every lane adds x[row] * y[row] of its rows,
// block partials and the final sum in fixed order (block_partial_finish).
template <class RP, bool DOT = false>
__global__ void __launch_bounds__(256, 4) spmv_kernel(int n, const RP* __restrict__ rp, const int* __restrict__ ci,
                                                   const double* __restrict__ v, const double* __restrict__ x,
                                                   double* __restrict__ y, const double* __restrict__ b,
                                                   double* __restrict__ part = nullptr, double* __restrict__ out = nullptr,
                                                   int slot = 0) {
  __shared__ double prod[SPMV_WARPS][SPMV_CH];
  double dacc = 0.0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* pw = prod[w];
  const long long nwarps = (long long)gridDim.x * SPMV_WARPS;
  for (long long r0 = ((long long)blockIdx.x * SPMV_WARPS + w) * 32; r0 < n; r0 += nwarps * 32) {
    const long long row = r0 + lane;
    const int last = (int)min(31LL, n - 1 - r0);  // last valid lane
    long long rs = 0, re = 0;
    if (row < n) {
      rs = (long long)rp[row];
      re = (long long)rp[row + 1];
    }
    const long long e0 = __shfl_sync(0xffffffffu, rs, 0);
    const long long e1 = __shfl_sync(0xffffffffu, re, last);
    double s = 0.0;
    for (long long cs = e0; cs < e1; cs += SPMV_CH) {
      const int cnt = (int)min((long long)SPMV_CH, e1 - cs);
      int cj[SPMV_CH / 32];
      double vj[SPMV_CH / 32];
#pragma unroll
      for (int j = 0; j < SPMV_CH / 32; ++j) {
        const int k = lane + 32 * j;
        if (k < cnt) {
          cj[j] = __ldcs(ci + cs + k);
          vj[j] = __ldcs(v + cs + k);
        }
      }
#pragma unroll
      for (int j = 0; j < SPMV_CH / 32; ++j) {
        const int k = lane + 32 * j;
        if (k < cnt) pw[k] = vj[j] * __ldg(x + cj[j]);
      }
      __syncwarp();
      const long long a = max(rs, cs), z = min(re, cs + cnt);
      for (long long e = a; e < z; ++e) s += pw[e - cs];
      __syncwarp();
    }
    if (row < n) {
      y[row] = b ? b[row] - s : s;
      if (DOT) dacc = fma(x[row], s, dacc);
    }
  }
  if (DOT) block_partial_finish(dacc, part, out, slot);
}

__global__ void rowptr32_kernel(const long long* __restrict__ rp, int* __restrict__ out, long long n1) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n1; i += (long long)gridDim.x * blockDim.x)
    out[i] = (int)rp[i];
}

cudaError_t launch_rowptr32(const long long* rp, int* out, long long n1, cudaStream_t s) {
  if (n1 <= 0) return cudaSuccess;
  long long blocks = std::min<long long>((n1 + 255) / 256, 148 * 16);
  count_launch(); rowptr32_kernel<<<(unsigned)blocks, 256, 0, s>>>(rp, out, n1);
  return cudaGetLastError();
}

cudaError_t launch_spmv(int n, const long long* rp, const int* rp32, const int* ci, const double* v, const double* x,
                        double* y, const double* b, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long warps = ((long long)n + 31) / 32;
  long long blocks = (warps + SPMV_WARPS - 1) / SPMV_WARPS;
  if (blocks > 148 * 4) blocks = 148 * 4;  // 4 resident CTAs per SM (64 regs), grid-stride beyond
  count_launch();
  if (rp32) spmv_kernel<int><<<(unsigned)blocks, 256, 0, s>>>(n, rp32, ci, v, x, y, b);
  else spmv_kernel<long long><<<(unsigned)blocks, 256, 0, s>>>(n, rp, ci, v, x, y, b);
  return cudaGetLastError();
}

// y = A x and out[slot] = x'y in one launch (the p'Ap of a PCG iteration)
cudaError_t launch_spmv_dot(int n, const long long* rp, const int* rp32, const int* ci, const double* v,
                            const double* x, double* y, double* part, double* out, int slot, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long warps = ((long long)n + 31) / 32;
  long long blocks = (warps + SPMV_WARPS - 1) / SPMV_WARPS;
  if (blocks > 148 * 4) blocks = 148 * 4;
  if (blocks > RED_MAX) blocks = RED_MAX;
  count_launch();
  if (rp32) spmv_kernel<int, true><<<(unsigned)blocks, 256, 0, s>>>(n, rp32, ci, v, x, y, nullptr, part, out, slot);
  else spmv_kernel<long long, true><<<(unsigned)blocks, 256, 0, s>>>(n, rp, ci, v, x, y, nullptr, part, out, slot);
  return cudaGetLastError();
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block partial to part[blockIdx.x]; the block that arrives last (counter at
// part + PCG_CNT_OFF) adds all partials in index order into out[slot] and
// resets the counter -- the sum does not depend on which block that is.  One
// launch per reduction instead of a partial and a finishing launch.
__device__ void block_partial_finish(double v, double* part, double* out, int slot) {
  __shared__ double red[8];
  __shared__ double all[RED_MAX];
  __shared__ bool last;
  unsigned* counter = reinterpret_cast<unsigned*>(part + PCG_CNT_OFF);
  v = wsum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    part[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) all[i] = __ldcg(part + i);
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)gridDim.x; ++i) s += all[i];
    out[slot] = s;
    *counter = 0u;
  }
}

// a.b into out[slot]
__global__ void __launch_bounds__(256) dot_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n,
                                                  double* __restrict__ part, double* __restrict__ out, int slot) {
  double s = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) s = fma(a[i], b[i], s);
  block_partial_finish(s, part, out, slot);
}

// x += alpha p ; r -= alpha q ; ||r||^2 into out[slot]  with alpha = sc[rz]/sc[1]
__global__ void __launch_bounds__(256) xr_update_kernel(double* __restrict__ x, double* __restrict__ r,
                                                        const double* __restrict__ p, const double* __restrict__ q,
                                                        long long n, const double* __restrict__ sc,
                                                        double* __restrict__ part, double* __restrict__ out, int slot,
                                                        int rz) {
  const double alpha = sc[rz] / sc[1];
  double s = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  block_partial_finish(s, part, out, slot);
}

// p = z + beta p with beta = sc[num]/sc[den] (the new and the previous r'z)
__global__ void __launch_bounds__(256) p_update_kernel(double* __restrict__ p, const double* __restrict__ z, long long n,
                                                       const double* __restrict__ sc, int num, int den) {
  const double beta = sc[num] / sc[den];
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) p[i] = z[i] + beta * p[i];
}

// out = b - out (the residual of a callback operator's product)
__global__ void __launch_bounds__(256) residual_kernel(const double* __restrict__ b, double* __restrict__ out,
                                                       long long n) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) out[i] = b[i] - out[i];
}

cudaError_t launch_residual(const double* b, double* out, long long n, cudaStream_t s) {
  count_launch(); residual_kernel<<<RED_BLOCKS, 256, 0, s>>>(b, out, n);
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* a, const double* b, long long n, double* part, double* out, int slot,
                       cudaStream_t s) {
  count_launch(); dot_kernel<<<RED_BLOCKS, 256, 0, s>>>(a, b, n, part, out, slot);
  return cudaGetLastError();
}
cudaError_t launch_xr_update(double* x, double* r, const double* p, const double* q, long long n, const double* sc,
                             double* part, double* out, int slot, cudaStream_t s, int rz) {
  count_launch(); xr_update_kernel<<<RED_BLOCKS, 256, 0, s>>>(x, r, p, q, n, sc, part, out, slot, rz);
  return cudaGetLastError();
}
cudaError_t launch_p_update(double* p, const double* z, long long n, const double* sc, cudaStream_t s, int num,
                            int den) {
  count_launch(); p_update_kernel<<<RED_BLOCKS, 256, 0, s>>>(p, z, n, sc, num, den);
  return cudaGetLastError();
}

}  // namespace sgf
