// Householder QR with column-norm pivoting, truncated at the numerical rank.
//
// Restates the pivot/reflector rules of the reference `pivoted_qr`
// (densela.py:149-217):
//   pivot      = first argmax of the downdated squared column norms (lowest
//                index on exact ties), or the replayed column (parity mode);
//   stop       when the pivot norm^2 <= floor^2 or ||x|| <= floor,
//                floor = eps * max(max|A|, 1);
//   reflector  sign = -sign(x0) (-1 for x0 == 0), u1 = x0 - sign*||x||,
//              w = x / u1 (w0 = 1), tau = -sign*u1/||x||, R_kk = sign*||x||;
//   downdate   norm2_j = max(norm2_j - R_kj^2, 0), recomputed from the
//              column below row k when norm2_j <= eps * ref2_j.
// The reference runs every step and counts rank = #{|R_ii| > tol |R_00|}
// (full_steps = 1 does the same).  The first r steps of a pivoted QR do not
// depend on later ones and |R_ii| is non-increasing, so stopping at the
// first |R_kk| <= tol |R_00| (the default) yields the same rank, pivots, R_1
// and Q_1 while skipping min(m,c) - r steps.  The reflectors past the rank
// only choose the orthonormal completion Q_2, which the reference itself
// determines by rounding (its columns past the numerical rank are noise):
// apply_inverse depends on Q_2 Q_2^T = I - Q_1 Q_1^T only, and
// apply_half_inverse's dropped coordinates match the reference's up to that
// rotation (tests/test_gpu_parity.py::test_half_inverse_invariants).
// Low-rank mode (forced rank r, factorization.py:331-339) runs exactly r steps.
//
// One CTA per compressed node; the m x c panel (column major) stays in
// global memory / L2, the current reflector lives in shared memory.
#include <cfloat>
#include <cmath>
#include <cooperative_groups.h>
#include <cstdlib>
#include <map>

#include "common.h"

namespace sgf {

constexpr int QR_THREADS = 512;
constexpr int QR_WARPS = QR_THREADS / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double s = (l < QR_WARPS) ? red[l] : 0.0;
    s = warp_sum(s);
    if (l == 0) red[QR_WARPS] = s;
  }
  __syncthreads();
  return red[QR_WARPS];
}

__device__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double s = (l < QR_WARPS) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (l == 0) red[QR_WARPS] = s;
  }
  __syncthreads();
  return red[QR_WARPS];
}

// first index of the maximum of nrm2[k..c)
__device__ int block_argmax(const double* nrm2, int k, int c, double* redv, int* redi) {
  double bv = -1.0;
  int bi = c;
  for (int j = k + threadIdx.x; j < c; j += blockDim.x) {
    double v = nrm2[j];
    if (v > bv) { bv = v; bi = j; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) { redv[w] = bv; redi[w] = bi; }
  __syncthreads();
  if (w == 0) {
    bv = (l < QR_WARPS) ? redv[l] : -1.0;
    bi = (l < QR_WARPS) ? redi[l] : c;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (l == 0) redi[QR_WARPS] = bi;
  }
  __syncthreads();
  return redi[QR_WARPS];
}

__global__ void __launch_bounds__(QR_THREADS) qrcp_kernel(const QrTask* __restrict__ tasks) {
  extern __shared__ double v[];  // m
  __shared__ double red[QR_WARPS + 1];
  __shared__ double redv[QR_WARPS + 1];
  __shared__ int redi[QR_WARPS + 1];
  __shared__ int s_piv;
  const QrTask T = tasks[blockIdx.x];
  const int m = T.m, c = T.c, kmax = min(m, c);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* N = T.Nm;
  const double eps = DBL_EPSILON;

  for (int j = warp; j < c; j += QR_WARPS) {
    const double* col = N + (long long)j * m;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s = fma(col[i], col[i], s);
    s = warp_sum(s);
    if (lane == 0) { T.nrm2[j] = s; T.ref2[j] = s; T.perm[j] = j; }
  }
  double amax = 0.0;
  for (long long e = tid; e < (long long)m * c; e += QR_THREADS) amax = fmax(amax, fabs(N[e]));
  amax = block_max(amax, red);
  const double floor_ = eps * fmax(amax, 1.0);
  const double floor2 = floor_ * floor_;
  __syncthreads();

  const int limit = (T.forced_rank >= 0) ? min(T.forced_rank, kmax) : kmax;
  int steps = 0, rank = 0;
  double r00 = 0.0;
  for (int k = 0; k < limit; ++k) {
    int piv;
    if (T.replay && k < T.nreplay) {
      if (tid == 0) s_piv = -1;
      __syncthreads();
      const int want = T.replay[k];
      for (int j = k + tid; j < c; j += QR_THREADS)
        if (T.perm[j] == want) s_piv = j;
      __syncthreads();
      piv = s_piv;
      if (piv < 0) piv = block_argmax(T.nrm2, k, c, redv, redi);  // malformed replay: fall back
    } else {
      piv = block_argmax(T.nrm2, k, c, redv, redi);
    }
    if (T.nrm2[piv] <= floor2) break;
    if (piv != k) {
      double* a = N + (long long)k * m;
      double* b = N + (long long)piv * m;
      for (int i = tid; i < m; i += QR_THREADS) { double tmp = a[i]; a[i] = b[i]; b[i] = tmp; }
      __syncthreads();
      if (tid == 0) {
        double t2 = T.nrm2[k]; T.nrm2[k] = T.nrm2[piv]; T.nrm2[piv] = t2;
        t2 = T.ref2[k]; T.ref2[k] = T.ref2[piv]; T.ref2[piv] = t2;
        int ti = T.perm[k]; T.perm[k] = T.perm[piv]; T.perm[piv] = ti;
      }
    }
    __syncthreads();
    double* xk = N + (long long)k * m;
    double ss = 0.0;
    for (int i = k + tid; i < m; i += QR_THREADS) ss = fma(xk[i], xk[i], ss);
    const double xn = sqrt(block_sum(ss, red));
    if (xn <= floor_) break;
    if (k == 0) r00 = xn;
    if (xn > T.tol * r00) ++rank;
    else if (T.forced_rank < 0 && !T.full_steps) break;  // rank reached
    const double x0 = xk[k];
    const double sgn = (x0 != 0.0) ? -copysign(1.0, x0) : -1.0;
    const double u1 = x0 - sgn * xn;
    const double tau = -sgn * u1 / xn;
    for (int i = k + tid; i < m; i += QR_THREADS) v[i - k] = (i == k) ? 1.0 : xk[i] / u1;
    __syncthreads();
    const int len = m - k;
    for (int j = k + 1 + warp; j < c; j += QR_WARPS) {
      double* col = N + (long long)j * m + k;
      double s = 0.0;
      for (int i = lane; i < len; i += 32) s = fma(v[i], col[i], s);
      s = warp_sum(s);
      const double ts = tau * s;
      double fresh = 0.0;
      for (int i = lane; i < len; i += 32) {
        double nv = fma(-ts, v[i], col[i]);
        col[i] = nv;
        if (i > 0) fresh = fma(nv, nv, fresh);
      }
      fresh = warp_sum(fresh);
      if (lane == 0) {
        const double rkj = col[0];
        double nn = fmax(T.nrm2[j] - rkj * rkj, 0.0);
        if (nn <= eps * T.ref2[j]) {
          nn = fresh;
          T.ref2[j] = fmax(fresh, floor2);
        }
        T.nrm2[j] = nn;
      }
    }
    __syncthreads();
    for (int i = k + 1 + tid; i < m; i += QR_THREADS) xk[i] = v[i - k];
    if (tid == 0) { xk[k] = sgn * xn; T.tau[k] = tau; }
    __syncthreads();
    steps = k + 1;
  }
  if (T.forced_rank >= 0) rank = min(T.forced_rank, m);
  if (tid == 0) { *T.out_rank = rank; *T.out_steps = steps; }
}

// ---------------------------------------------------------------------------
// Cluster variant: one thread-block cluster of QC CTAs per node.  CTA q owns
// the panel positions j == q (mod QC) (norms, updates); every CTA recomputes
// the reflector from the pivot column redundantly (identical arithmetic =>
// identical results).  Columns are never moved during the factorization:
// every CTA keeps the same position -> column map in shared memory and applies
// the pivot swap to it locally, and norms are kept per column.  A CTA's
// candidate for step k+1 depends only on its own updates of step k, so one
// cluster barrier per step suffices (candidates of k+1 and the updates of k
// become visible together); the pivot column of step k is written back by its
// owner after that barrier.  At the end the columns are put in position order
// through a scratch panel.  Same arithmetic rules as qrcp_kernel above.
// ---------------------------------------------------------------------------
// QC CTAs per cluster (16: non-portable size, allowed at launch), QCT threads
// per CTA.  A step's column updates are latency-bound loads from L2 (one warp
// per column, two passes), so the threads per node set the step time: 1024
// threads per CTA leave each warp 1-2 columns of a 600-1200 column panel per
// step (256 threads: 5-10 columns per warp, ~100 us per step at m = 1300).
template <int QCW>
__device__ double cblock_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < QCW; ++i) s += red[i];  // fixed order, same in every CTA
  return s;
}

template <int QC, int QCT>
__global__ void __cluster_dims__(QC, 1, 1) __launch_bounds__(QCT)
    qrcp_cluster_kernel(const QrTask* __restrict__ tasks) {
  constexpr int QCW = QCT / 32;
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double v[];  // m reflector entries, then c column ids
  __shared__ double red[QCW];
  // candidates double-buffered by step parity: a fast CTA publishes step k+1
  // while a slow one may still read step k
  __shared__ double cand_v[2];
  __shared__ int cand_i[2];
  __shared__ double s_amax;
  __shared__ double wv[QCW];
  __shared__ int wi[QCW];
  const int q = (int)cluster.block_rank();
  const QrTask T = tasks[blockIdx.x / QC];
  const int m = T.m, c = T.c, kmax = min(m, c);
  int* col_of = reinterpret_cast<int*>(v + m);  // position -> column
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* N = T.Nm;
  const double eps = DBL_EPSILON;

  for (int j = tid; j < c; j += QCT) col_of[j] = j;
  // initial norms of owned columns, local max |A|
  double amax = 0.0;
  for (int j = q + QC * warp; j < c; j += QC * QCW) {
    const double* col = N + (long long)j * m;
    double s = 0.0, mx = 0.0;
    for (int i = lane; i < m; i += 32) {
      s = fma(col[i], col[i], s);
      mx = fmax(mx, fabs(col[i]));
    }
    s = warp_sum(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    amax = fmax(amax, mx);
    if (lane == 0) { T.nrm2[j] = s; T.ref2[j] = s; }
  }
  if (lane == 0) red[warp] = amax;
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int i = 0; i < QCW; ++i) mx = fmax(mx, red[i]);
    s_amax = mx;
  }
  cluster.sync();
  {
    double mx = 0.0;
    for (int r = 0; r < QC; ++r) mx = fmax(mx, *cluster.map_shared_rank(&s_amax, r));
    amax = mx;
  }
  const double floor_ = eps * fmax(amax, 1.0);
  const double floor2 = floor_ * floor_;

  // this CTA's pivot candidate for step k over its positions >= k (first max
  // by position, or the replayed column)
  auto local_candidate = [&](int k) {
    const bool rep = T.replay && k < T.nreplay;
    double bv = rep ? 0.0 : -1.0;
    int bi = c;
    for (int j = k + ((q - k) % QC + QC) % QC + QC * tid; j < c; j += QC * QCT) {
      const int cj = col_of[j];
      if (rep) {
        if (cj == T.replay[k]) { bv = 1.0; bi = j; }
      } else {
        const double x = T.nrm2[cj];
        if (x > bv) { bv = x; bi = j; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { wv[warp] = bv; wi[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b = wv[0];
      int i0 = wi[0];
      for (int w = 1; w < QCW; ++w)
        if (wv[w] > b || (wv[w] == b && wi[w] < i0)) { b = wv[w]; i0 = wi[w]; }
      cand_v[k & 1] = b;
      cand_i[k & 1] = i0;
    }
  };

  const int limit = (T.forced_rank >= 0) ? min(T.forced_rank, kmax) : kmax;
  int steps = 0, rank = 0;
  double r00 = 0.0;
  int pend_col = -1, pend_k = -1;  // pivot column whose final values this CTA still has to store
  double pend_r = 0.0;
  __syncthreads();
  if (limit > 0) local_candidate(0);
  for (int k = 0; k < limit; ++k) {
    cluster.sync();  // candidates of k and every update of step k-1 visible
    // store the previous step's pivot column (everyone has read it)
    if (pend_col >= 0) {
      double* col = N + (long long)pend_col * m;
      for (int i = pend_k + 1 + tid; i < m; i += QCT) col[i] = v[i - pend_k];
      if (tid == 0) col[pend_k] = pend_r;
      pend_col = -1;
    }
    int piv = c;
    {
      double b = -2.0;
      for (int r = 0; r < QC; ++r) {
        const double ov = *cluster.map_shared_rank(&cand_v[k & 1], r);
        const int oi = *cluster.map_shared_rank(&cand_i[k & 1], r);
        if (oi >= c) continue;
        if (ov > b || (ov == b && oi < piv)) { b = ov; piv = oi; }
      }
    }
    if (piv >= c) break;  // malformed replay
    if (T.nrm2[col_of[piv]] <= floor2) break;
    __syncthreads();  // everyone has read col_of / v of the previous step
    if (tid == 0 && piv != k) {
      const int t2 = col_of[k];
      col_of[k] = col_of[piv];
      col_of[piv] = t2;
    }
    __syncthreads();
    const int ck = col_of[k];
    const double* xk = N + (long long)ck * m;
    double ss = 0.0;
    for (int i = k + tid; i < m; i += QCT) ss = fma(xk[i], xk[i], ss);
    const double xn = sqrt(cblock_sum<QCW>(ss, red));
    if (xn <= floor_) break;
    if (k == 0) r00 = xn;
    if (xn > T.tol * r00) ++rank;
    else if (T.forced_rank < 0 && !T.full_steps) break;
    const double x0 = xk[k];
    const double sgn = (x0 != 0.0) ? -copysign(1.0, x0) : -1.0;
    const double u1 = x0 - sgn * xn;
    const double tau = -sgn * u1 / xn;
    for (int i = k + tid; i < m; i += QCT) v[i - k] = (i == k) ? 1.0 : xk[i] / u1;
    __syncthreads();
    const int len = m - k;
    for (int j = k + 1 + ((q - k - 1) % QC + QC) % QC + QC * warp; j < c; j += QC * QCW) {
      const int cj = col_of[j];
      double* col = N + (long long)cj * m + k;
      // both passes keep 8 loads of the column in flight per lane (the column
      // comes from L2: one load per trip cost a memory latency per 32 rows);
      // the accumulation order is the plain loop's
      double s = 0.0;
      int i = lane;
      for (; i + 224 < len; i += 256) {
        double cv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) cv[u] = col[i + 32 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) s = fma(v[i + 32 * u], cv[u], s);
      }
      if (i < len) {  // the last, partial batch
        double cv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) cv[u] = (i + 32 * u < len) ? col[i + 32 * u] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i + 32 * u < len) s = fma(v[i + 32 * u], cv[u], s);
      }
      s = warp_sum(s);
      const double ts = tau * s;
      double fresh = 0.0;
      i = lane;
      for (; i + 224 < len; i += 256) {
        double cv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) cv[u] = col[i + 32 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double nv = fma(-ts, v[i + 32 * u], cv[u]);
          col[i + 32 * u] = nv;
          if (i + 32 * u > 0) fresh = fma(nv, nv, fresh);
        }
      }
      if (i < len) {
        double cv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) cv[u] = (i + 32 * u < len) ? col[i + 32 * u] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i + 32 * u < len) {
            const double nv = fma(-ts, v[i + 32 * u], cv[u]);
            col[i + 32 * u] = nv;
            if (i + 32 * u > 0) fresh = fma(nv, nv, fresh);
          }
      }
      fresh = warp_sum(fresh);
      if (lane == 0) {
        const double rkj = col[0];
        double nn = fmax(T.nrm2[cj] - rkj * rkj, 0.0);
        if (nn <= eps * T.ref2[cj]) {
          nn = fresh;
          T.ref2[cj] = fmax(fresh, floor2);
        }
        T.nrm2[cj] = nn;
      }
    }
    if (k % QC == q) {
      pend_col = ck;
      pend_k = k;
      pend_r = sgn * xn;
      if (tid == 0) T.tau[k] = tau;
    }
    steps = k + 1;
    __syncthreads();  // this CTA's norms of step k written
    if (k + 1 < limit) local_candidate(k + 1);
  }
  cluster.sync();  // every CTA is done reading the last pivot column
  if (pend_col >= 0) {
    double* col = N + (long long)pend_col * m;
    for (int i = pend_k + 1 + tid; i < m; i += QCT) col[i] = v[i - pend_k];
    if (tid == 0) col[pend_k] = pend_r;
  }
  cluster.sync();
  // columns into position order through the scratch panel, permutation out
  for (int j = q; j < c; j += QC) {
    const double* src = N + (long long)col_of[j] * m;
    double* dst = T.tmp + (long long)j * m;
    for (int i = tid; i < m; i += QCT) dst[i] = src[i];
  }
  if (q == 0)
    for (int j = tid; j < c; j += QCT) T.perm[j] = col_of[j];
  cluster.sync();
  for (int j = q; j < c; j += QC) {
    const double* src = T.tmp + (long long)j * m;
    double* dst = N + (long long)j * m;
    for (int i = tid; i < m; i += QCT) dst[i] = src[i];
  }
  if (q == 0 && tid == 0) {
    *T.out_rank = (T.forced_rank >= 0) ? min(T.forced_rank, m) : rank;
    *T.out_steps = steps;
  }
  cluster.sync();  // keep every CTA's shared memory alive for remote reads
}

// ---------------------------------------------------------------------------
// Shared-memory resident variant (the panels of the compression levels fit a
// 16-CTA cluster: m x c <= 1225 x 184 at 128^3 -> ~118 KB per CTA).  CTA q
// holds the ORIGINAL columns cj == q (mod QC) in its shared memory for the
// whole factorization, so a step touches no global memory, and a step costs
// ONE cluster barrier:
//   B   cluster barrier: the updates and candidates of step k-1 are final.
//       A candidate carries the column's downdated norm^2 (the pivot rule),
//       its exact norm^2 below row k (from the previous update's sweep) and
//       its row-k entry, so every CTA picks the pivot (first maximum by
//       position, or the replayed column), applies the position swap to its
//       copy of the position <-> column maps and forms the reflector scalars
//       (sign, u1, tau, R_kk) itself -- identical inputs, identical values.
//       Every CTA then reads the pivot column from the owner (DSMEM) scaled
//       by 1/u1 as the reflector, updates its unpivoted columns (dot, axpy,
//       norm downdate, exact norm^2 below row k+1) and forms its candidate
//       for step k+1.  The owner rewrites the pivot column as R_kk + the
//       reflector after the NEXT barrier (nobody reads it remotely again).
// Per-column arithmetic and reduction orders are those of the kernels above
// (lane-strided FMA chains + warp_sum).  At the end every CTA writes its
// columns to their final positions in N.
// ---------------------------------------------------------------------------
struct QsCand {
  double v;    // comparison value (downdated norm^2, or 1 for the replayed column)
  double n2;   // the column's downdated norm^2
  double xn2;  // the column's exact norm^2 below row k
  double x0;   // the column's row-k entry
  int pos;     // position (c: none)
};
constexpr int QST = 384;          // threads of the shared-memory variant: one warp per owned column
constexpr int QSW = QST / 32;
constexpr int QS_VCH = 4;         // reflector copy: remote loads in flight per thread
template <int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(QST)
    qrcp_smem_kernel(const QrTask* __restrict__ tasks, int cpc) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double qs[];
  __shared__ double red[QSW];
  __shared__ QsCand cand[2];
  __shared__ QsCand sel;
  __shared__ int sel_pc;
  __shared__ double s_amax;
  __shared__ double wv[QSW];
  __shared__ int wi[QSW], wl[QSW];
  const int q = (int)cluster.block_rank();
  const QrTask T = tasks[blockIdx.x / CS];
  const int m = T.m, c = T.c, kmax = min(m, c);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double eps = DBL_EPSILON;
  // layout: cpc owned columns (m each) | local reflector (m) | nrm2, ref2, fn2 (cpc each)
  //         | col_of (c) | pos_of (c) | done (cpc)
  const int mp = (m + 1) & ~1;  // column stride: every buffer 16-byte aligned
  double* cols = qs;
  double* vloc = cols + (size_t)cpc * mp;
  double* nrm2 = vloc + mp;
  double* ref2 = nrm2 + cpc;
  double* fn2 = ref2 + cpc;
  int* col_of = reinterpret_cast<int*>(fn2 + cpc);
  int* pos_of = col_of + c;
  int* done = pos_of + c;
  const int nown = (c > q) ? (c - q + CS - 1) / CS : 0;  // owned columns q, q+CS, ...
  for (int j = tid; j < c; j += QST) {
    col_of[j] = j;
    pos_of[j] = j;
  }
  for (int l = tid; l < nown; l += QST) done[l] = 0;
  for (int l = 0; l < nown; ++l) {
    const double* src = T.Nm + (long long)(q + CS * l) * m;
    double* dst = cols + (size_t)l * mp;
    for (int i = tid; i < m; i += QST) dst[i] = src[i];
  }
  __syncthreads();
  double amax = 0.0;
  for (int l = warp; l < nown; l += QSW) {
    const double* col = cols + (size_t)l * mp;
    double s = 0.0, mx = 0.0;
    for (int i = lane; i < m; i += 32) {
      s = fma(col[i], col[i], s);
      mx = fmax(mx, fabs(col[i]));
    }
    s = warp_sum(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    amax = fmax(amax, mx);
    if (lane == 0) { nrm2[l] = s; ref2[l] = s; fn2[l] = s; }
  }
  if (lane == 0) red[warp] = amax;
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int i = 0; i < QSW; ++i) mx = fmax(mx, red[i]);
    s_amax = mx;
  }
  cluster.sync();
  {
    double mx = 0.0;
    for (int r = 0; r < CS; ++r) mx = fmax(mx, *cluster.map_shared_rank(&s_amax, r));
    amax = mx;
  }
  const double floor_ = eps * fmax(amax, 1.0);
  const double floor2 = floor_ * floor_;

  // this CTA's candidate for step k over its unpivoted columns: first maximum by position
  auto local_candidate = [&](int k) {
    const bool rep = T.replay && k < T.nreplay;
    double bv = rep ? 0.0 : -1.0;
    int bp = c, bl = -1;
    for (int l = tid; l < nown; l += QST) {
      if (done[l]) continue;
      const int cj = q + CS * l, pj = pos_of[cj];
      if (rep) {
        if (cj == T.replay[k]) { bv = 1.0; bp = pj; bl = l; }
      } else {
        const double x = nrm2[l];
        if (x > bv || (x == bv && pj < bp)) { bv = x; bp = pj; bl = l; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bl = ol; }
    }
    if (lane == 0) { wv[warp] = bv; wi[warp] = bp; wl[warp] = bl; }
    __syncthreads();
    if (tid == 0) {
      double b = wv[0];
      int p0 = wi[0], l0 = wl[0];
      for (int w = 1; w < QSW; ++w)
        if (wv[w] > b || (wv[w] == b && wi[w] < p0)) { b = wv[w]; p0 = wi[w]; l0 = wl[w]; }
      QsCand r{b, 0.0, 0.0, 0.0, p0};
      if (l0 >= 0) {
        r.n2 = nrm2[l0];
        r.xn2 = fn2[l0];
        r.x0 = cols[(size_t)l0 * mp + k];
      }
      cand[k & 1] = r;
    }
  };

  const int limit = (T.forced_rank >= 0) ? min(T.forced_rank, kmax) : kmax;
  int steps = 0, rank = 0;
  double r00 = 0.0;
  // the previous pivot column, rewritten as R_kk + reflector after the next barrier
  int p_lp = -1, p_k = 0;
  double p_u1 = 1.0, p_rkk = 0.0;
  auto flush_pivot = [&]() {
    if (p_lp < 0) return;
    double* xk = cols + (size_t)p_lp * mp;
    for (int i = p_k + 1 + tid; i < m; i += QST) xk[i] = xk[i] / p_u1;
    if (tid == 0) xk[p_k] = p_rkk;
    p_lp = -1;
  };
  if (limit > 0) local_candidate(0);
  for (int k = 0; k < limit; ++k) {
    cluster.sync();  // candidates of k, every update of k-1; nobody reads the previous pivot column
    if (warp == 0) {   // lane r < CS fetches CTA r's candidate; (value, position) order is total
      QsCand o{-2.0, 0.0, 0.0, 0.0, c};
      if (lane < CS) {
        o = *cluster.map_shared_rank(&cand[k & 1], lane);
        if (o.pos >= c) o.v = -2.0;
      }
      double bv = o.v;
      int bp = o.pos, bl = lane;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, d);
        const int op = __shfl_xor_sync(0xffffffffu, bp, d);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, d);
        if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bl = ol; }
      }
      const double n2 = __shfl_sync(0xffffffffu, o.n2, bl);
      const double xn2 = __shfl_sync(0xffffffffu, o.xn2, bl);
      const double x0 = __shfl_sync(0xffffffffu, o.x0, bl);
      if (lane == 0) {
        const int pp = bp < c && bv > -2.0 ? bp : c;
        sel = QsCand{bv, n2, xn2, x0, pp};
        if (pp < c && n2 > floor2) {
          const int pc = col_of[pp];
          sel_pc = pc;
          if (pp != k) {  // position swap k <-> pp
            const int ck = col_of[k];
            col_of[k] = pc;
            col_of[pp] = ck;
            pos_of[pc] = k;
            pos_of[ck] = pp;
          }
        }
      }
    } else {
      flush_pivot();
    }
    __syncthreads();
    if (warp == 0) flush_pivot();
    const int pp = sel.pos;
    if (pp >= c) break;  // malformed replay
    if (sel.n2 <= floor2) break;
    const int pc = sel_pc;
    const int owner = pc % CS, lp = pc / CS;
    const double xn = sqrt(sel.xn2);
    if (xn <= floor_) break;
    const double r0 = (k == 0) ? xn : r00;
    if (T.forced_rank < 0 && !T.full_steps && !(xn > T.tol * r0)) break;
    const double x0 = sel.x0;
    const double sgn = (x0 != 0.0) ? -copysign(1.0, x0) : -1.0;
    const double u1 = x0 - sgn * xn;
    const double tau = -sgn * u1 / xn;
    if (k == 0) r00 = xn;
    if (xn > T.tol * r00) ++rank;
    const int len = m - k;
    {  // remote pivot column / u1 -> local reflector, the loads all in flight before the stores
      const double* rx = cluster.map_shared_rank(cols + (size_t)lp * mp + k, owner);
      double t[QS_VCH];
#pragma unroll
      for (int u = 0; u < QS_VCH; ++u)
        if (tid + QST * u < len) t[u] = rx[tid + QST * u];
#pragma unroll
      for (int u = 0; u < QS_VCH; ++u) {
        const int i = tid + QST * u;
        if (i < len) vloc[i] = (i == 0) ? 1.0 : t[u] / u1;
      }
      for (int i = tid + QST * QS_VCH; i < len; i += QST) vloc[i] = rx[i] / u1;
    }
    if (owner == q) {
      if (tid == 0) {
        done[lp] = 1;
        T.tau[k] = tau;
      }
      p_lp = lp;
      p_k = k;
      p_u1 = u1;
      p_rkk = sgn * xn;
    }
    __syncthreads();
    for (int l = warp; l < nown; l += QSW) {
      if (done[l]) continue;
      double* col = cols + (size_t)l * mp + k;
      double s = 0.0;
      for (int i = lane; i < len; i += 32) s = fma(vloc[i], col[i], s);
      s = warp_sum(s);
      const double ts = tau * s;
      double fresh = 0.0;
      for (int i = lane; i < len; i += 32) {
        const double nv = fma(-ts, vloc[i], col[i]);
        col[i] = nv;
        if (i > 0) fresh = fma(nv, nv, fresh);
      }
      fresh = warp_sum(fresh);
      if (lane == 0) {
        const double rkj = col[0];
        double nn = fmax(nrm2[l] - rkj * rkj, 0.0);
        if (nn <= eps * ref2[l]) {
          nn = fresh;
          ref2[l] = fmax(fresh, floor2);
        }
        nrm2[l] = nn;
        fn2[l] = fresh;
      }
    }
    steps = k + 1;
    __syncthreads();  // norms of step k
    if (k + 1 < limit) local_candidate(k + 1);
  }
  cluster.sync();  // every CTA has read its last remote data; all inputs were loaded long ago
  flush_pivot();
  __syncthreads();
  // columns to their final positions, permutation out
  for (int l = 0; l < nown; ++l) {
    const int cj = q + CS * l;
    const double* src = cols + (size_t)l * mp;
    double* dst = T.Nm + (long long)pos_of[cj] * m;
    for (int i = tid; i < m; i += QST) dst[i] = src[i];
  }
  if (q == 0)
    for (int j = tid; j < c; j += QST) T.perm[j] = col_of[j];
  if (q == 0 && tid == 0) {
    *T.out_rank = (T.forced_rank >= 0) ? min(T.forced_rank, m) : rank;
    *T.out_steps = steps;
  }
  cluster.sync();  // keep every CTA's shared memory alive for remote reads
}

template <int CS>
static size_t qrcp_smem_bytes(int m, int c) {
  const size_t cpc = (size_t)(c + CS - 1) / CS, mp = (size_t)((m + 1) & ~1);
  return (cpc * mp + mp + 3 * cpc) * sizeof(double) + (2 * (size_t)c + cpc) * sizeof(int);
}

template <int CS>
static cudaError_t qr_configure(size_t sb) {
  static FuncAttrs fa;
  cudaError_t e = ensure_nonportable_cluster(qrcp_smem_kernel<CS>, fa);
  if (e != cudaSuccess) return e;
  return ensure_smem(qrcp_smem_kernel<CS>, sb, fa);
}

template <int CS>
static cudaError_t qr_launch_smem(const QrTask* d_tasks, int ntasks, size_t sb, int max_c, cudaStream_t s) {
  cudaError_t e = qr_configure<CS>(sb);
  if (e != cudaSuccess) return e;
  count_launch();
  qrcp_smem_kernel<CS><<<ntasks * CS, QST, sb, s>>>(d_tasks, (max_c + CS - 1) / CS);
  return cudaGetLastError();
}

// resident clusters of the shared-memory QR for a cluster size and shared
// memory per CTA (cached: the occupancy query is a driver call)
template <int CS>
static int qr_active(size_t sb) {
  if (qr_configure<CS>(sb) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS * 64);
  cfg.blockDim = dim3(QST);
  cfg.dynamicSmemBytes = sb;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = CS;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, qrcp_smem_kernel<CS>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

static int qr_active_clusters(int cs, size_t sb) {
  static std::map<std::pair<int, size_t>, int> cache;
  const size_t key_sb = (sb + 4095) / 4096 * 4096;
  auto it = cache.find({cs, key_sb});
  if (it != cache.end()) return it->second;
  int n = cs == 16 ? qr_active<16>(key_sb) : cs == 12 ? qr_active<12>(key_sb) : cs == 10 ? qr_active<10>(key_sb)
                                                                                           : qr_active<8>(key_sb);
  cache[{cs, key_sb}] = n;
  return n;
}

template <int QC, int QCT>
static cudaError_t qr_cluster_configure(size_t smem) {
  static FuncAttrs fa;
  cudaError_t e = QC > 8 ? ensure_nonportable_cluster(qrcp_cluster_kernel<QC, QCT>, fa) : cudaSuccess;
  if (e == cudaSuccess) e = ensure_smem(qrcp_cluster_kernel<QC, QCT>, smem, fa);
  return e;
}

template <int QC, int QCT>
static cudaError_t qr_launch_cluster(const QrTask* d_tasks, int ntasks, size_t smem, cudaStream_t s) {
  cudaError_t e = qr_cluster_configure<QC, QCT>(smem);
  if (e != cudaSuccess) return e;
  qrcp_cluster_kernel<QC, QCT><<<ntasks * QC, QCT, smem, s>>>(d_tasks);
  return cudaGetLastError();
}

cudaError_t launch_qrcp(const QrTask* d_tasks, int ntasks, int max_m, cudaStream_t s, int max_c) {
  if (ntasks <= 0) return cudaSuccess;
  size_t smem = (size_t)max_m * sizeof(double) + (size_t)max_c * sizeof(int);
  static FuncAttrs fa_single;
  {
    cudaError_t e = ensure_smem(qrcp_kernel, smem, fa_single);
    if (e != cudaSuccess) return e;
  }
  static int single = getenv("SGF_QR_SINGLE_CTA") ? 1 : 0;
  static int smem_ok = getenv("SGF_QR_SMEM") ? atoi(getenv("SGF_QR_SMEM")) : 1;
  // Cluster size: the panel must fit the cluster's shared memory, and the
  // wave's nodes run in rounds of (resident clusters); pick the size with the
  // fewest rounds (16-CTA clusters: at most 7 resident on the GPCs), ties to
  // the larger cluster (fewer columns per warp).
  constexpr size_t SMEM_CAP = (size_t)220 << 10;
  if (!single && smem_ok) {
    int best_cs = 0, best_rounds = 1 << 30;
    size_t best_sb = 0;
    const int cands[4] = {16, 12, 10, 8};
    for (int cs : cands) {
      if (smem_ok > 1 && cs != smem_ok) continue;  // SGF_QR_SMEM=<size> forces a cluster size
      const size_t sb = cs == 16 ? qrcp_smem_bytes<16>(max_m, max_c)
                        : cs == 12 ? qrcp_smem_bytes<12>(max_m, max_c)
                        : cs == 10 ? qrcp_smem_bytes<10>(max_m, max_c)
                                   : qrcp_smem_bytes<8>(max_m, max_c);
      if (sb > SMEM_CAP) continue;
      const int act = qr_active_clusters(cs, sb);
      if (act <= 0) continue;
      const int rounds = (ntasks + act - 1) / act;
      if (rounds < best_rounds) {
        best_rounds = rounds;
        best_cs = cs;
        best_sb = sb;
      }
    }
    if (best_cs == 16) return qr_launch_smem<16>(d_tasks, ntasks, best_sb, max_c, s);
    if (best_cs == 12) return qr_launch_smem<12>(d_tasks, ntasks, best_sb, max_c, s);
    if (best_cs == 10) return qr_launch_smem<10>(d_tasks, ntasks, best_sb, max_c, s);
    if (best_cs == 8) return qr_launch_smem<8>(d_tasks, ntasks, best_sb, max_c, s);
  }
  count_launch();
  if (single) {
    qrcp_kernel<<<ntasks, QR_THREADS, smem, s>>>(d_tasks);
    return cudaGetLastError();
  }
  // panel in global memory / L2: 16-CTA clusters of 1024 threads (cfg5's level-3
  // waves of 4-12 nodes, m ~ 1300 x 650 columns: 88 ms; 12 / 10 / 8 CTAs per
  // node 97 / 105 / 122 ms although fewer of the 16-CTA clusters are resident;
  // 16 x 256 threads 159 ms).  SGF_QR_CL=<size * 10000 + threads>: another variant.
  static const int cl = getenv("SGF_QR_CL") ? atoi(getenv("SGF_QR_CL")) : 161024;
  switch (cl) {
    case 160256: return qr_launch_cluster<16, 256>(d_tasks, ntasks, smem, s);
    case 81024: return qr_launch_cluster<8, 1024>(d_tasks, ntasks, smem, s);
    default: return qr_launch_cluster<16, 1024>(d_tasks, ntasks, smem, s);
  }
}

// ---------------------------------------------------------------------------
// Finish: explicit reflectors V (m x s, unit lower trapezoid, column major),
// the compact-WY factor T (s x s upper, row major) with
// H_0 ... H_{s-1} = I - V T V^T, and Q1 = H_0...H_{s-1} [I_r; 0] (m x r,
// column major).  Q = H_0 ... H_{s-1} is the orthogonal completion used for
// the compression factor; its first r columns are the reference's Q_1.
// ---------------------------------------------------------------------------
// phase 0: V (one CTA-stripe per node); phase 1: T from G = V^T V (computed by
// the GEMM kernel between the two phases).  Q1 is never formed: every
// product with Q (inverse operator, basis update) goes through V and T.
__global__ void __launch_bounds__(QR_THREADS) qr_extract_v_kernel(const QrFinishTask* __restrict__ tasks) {
  const QrFinishTask F = tasks[blockIdx.y];
  const int m = F.m, s = *F.steps;
  for (long long e = blockIdx.x * (long long)QR_THREADS + threadIdx.x; e < (long long)m * s;
       e += (long long)gridDim.x * QR_THREADS) {
    const int k = (int)(e / m), i = (int)(e % m);
    F.V[e] = (i < k) ? 0.0 : (i == k ? 1.0 : F.Nm[(long long)k * m + i]);
  }
}

// T recurrence (LAPACK larft, forward, columnwise) with T's upper triangle
// (packed rows) and column k of G in shared memory: each step reads only
// shared memory after one staged column (the global-memory form re-read T and
// G every step).  Same summation order.
__global__ void __launch_bounds__(QR_THREADS) qr_larft_kernel(const QrFinishTask* __restrict__ tasks) {
  extern __shared__ double tsm[];
  const QrFinishTask F = tasks[blockIdx.x];
  const int s = *F.steps;
  const int tid = threadIdx.x;
  const double* G = F.G;  // s x s, G[a][b] = v_a . v_b
  double* gk = tsm;       // column k of G
  double* tp = tsm + s;   // packed upper T: row a holds T[a][a..s)
  auto off = [s](int a) { return (long long)a * (2LL * s - a + 1) / 2; };
  for (int k = 0; k < s; ++k) {
    for (int b = tid; b < k; b += QR_THREADS) gk[b] = G[(long long)b * s + k];
    const double tk = F.tau[k];
    __syncthreads();
    // T[a][k] = -tau_k sum_{a<=b<k} T[a][b] G[b][k], a < k   (T upper)
    for (int a = tid; a < k; a += QR_THREADS) {
      const double* ta = tp + off(a) - a;  // ta[b] = T[a][b]
      double acc = 0.0;
      for (int b = a; b < k; ++b) acc = fma(ta[b], gk[b], acc);
      const double t = -tk * acc;
      tp[off(a) + (k - a)] = t;
      F.Tm[(long long)a * s + k] = t;
    }
    if (tid == 0) {
      tp[off(k)] = tk;
      F.Tm[(long long)k * s + k] = tk;
    }
    for (int a = k + 1 + tid; a < s; a += QR_THREADS) F.Tm[(long long)a * s + k] = 0.0;
    __syncthreads();
  }
}

// global-memory form for reflector counts whose T does not fit shared memory
__global__ void __launch_bounds__(QR_THREADS) qr_larft_global_kernel(const QrFinishTask* __restrict__ tasks) {
  const QrFinishTask F = tasks[blockIdx.x];
  const int s = *F.steps;
  const int tid = threadIdx.x;
  const double* G = F.G;
  for (int k = 0; k < s; ++k) {
    const double tk = F.tau[k];
    for (int a = tid; a < k; a += QR_THREADS) {
      double acc = 0.0;
      for (int b = a; b < k; ++b) acc = fma(F.Tm[(long long)a * s + b], G[b * s + k], acc);
      F.Tm[(long long)a * s + k] = -tk * acc;
    }
    if (tid == 0) F.Tm[(long long)k * s + k] = tk;
    for (int a = k + 1 + tid; a < s; a += QR_THREADS) F.Tm[(long long)a * s + k] = 0.0;
    __syncthreads();
  }
}

cudaError_t launch_qr_finish(const void* d_tasks, int ntasks, int phase, cudaStream_t s, int max_s) {
  if (ntasks <= 0) return cudaSuccess;
  count_launch();
  if (phase == 0) {
    qr_extract_v_kernel<<<dim3(16, ntasks), QR_THREADS, 0, s>>>((const QrFinishTask*)d_tasks);
  } else {
    const size_t smem = ((size_t)max_s + (size_t)max_s * (max_s + 1) / 2) * sizeof(double);
    if (smem > (size_t)220 << 10) {  // s > 232
      qr_larft_global_kernel<<<ntasks, QR_THREADS, 0, s>>>((const QrFinishTask*)d_tasks);
      return cudaGetLastError();
    }
    static FuncAttrs fa;
    cudaError_t e = ensure_smem(qr_larft_kernel, smem, fa);
    if (e != cudaSuccess) return e;
    qr_larft_kernel<<<ntasks, QR_THREADS, smem, s>>>((const QrFinishTask*)d_tasks);
  }
  return cudaGetLastError();
}

}  // namespace sgf
