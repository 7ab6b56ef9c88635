// Shared definitions of the sgf native library (B200 / sm_100a).
//
// Data layout conventions
//   * every dense block is row-major with an explicit leading dimension;
//     kernels address operands through (row stride, col stride) pairs so a
//     stored block (a,b) can be read as itself or as its transpose without
//     a copy (the reference keeps only blocks i <= j, blockmatrix.py:14-83);
//   * triangular matrices (L, L^{-1}) are stored as full squares with exact
//     zeros in the unused triangle, so K-range limits are optimisations only.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace sgf {

// ---- kernel function attributes (per device) ----------------------------------
// cudaFuncSetAttribute applies to the current device only, so a process with
// contexts on several GPUs must configure each one.  A FuncAttrs instance
// (one static per kernel) remembers, per device ordinal, the largest dynamic
// shared-memory size already set and whether non-portable cluster sizes were
// enabled.  The entry points select the context's device before launching.
struct FuncAttrs {
  std::atomic<int> smem[64];
  std::atomic<unsigned long long> nonportable;
  FuncAttrs() : nonportable(0) {
    for (auto& v : smem) v.store(0, std::memory_order_relaxed);
  }
};
template <class K>
inline cudaError_t ensure_smem(K kern, size_t bytes, FuncAttrs& fa) {
  int d = 0;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return e;
  std::atomic<int>& cur = fa.smem[d & 63];
  if ((int)bytes <= cur.load(std::memory_order_acquire)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  int seen = cur.load(std::memory_order_relaxed);
  while (seen < (int)bytes && !cur.compare_exchange_weak(seen, (int)bytes)) {
  }
  return cudaSuccess;
}
template <class K>
inline cudaError_t ensure_nonportable_cluster(K kern, FuncAttrs& fa) {
  int d = 0;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (d & 63);
  if (fa.nonportable.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) fa.nonportable.fetch_or(bit);
  return e;
}

// ---- batched FP64 GEMM (DMMA) ------------------------------------------------
// C(i,j) = beta*C(i,j) + alpha * sum_seg sum_{k in seg range} A(i,k) * B(j,k)
// A(i,k) = A[i*a_rs + k*a_ks],  B(j,k) = B[j*b_rs + k*b_ks]
enum : int {
  SEG_KLIM_M = 1,    // k < m0 + BM   (A lower triangular in (i,k))
  SEG_KLIM_N = 2,    // k < n0 + BN   (B lower triangular in (j,k))
  SEG_KSTART_M = 4,  // k >= m0       (A upper triangular in (i,k))
  SEG_KSTART_N = 8,  // k >= n0       (B upper triangular in (j,k))
};

struct GemmSeg {
  const double* A;
  const double* B;
  long long a_rs, a_ks;
  long long b_rs, b_ks;
  int K;
  int flags;
  // optional (single-segment tasks): one byte per 64 x 16 tile of A (row tile
  // i / 64, K chunk k / 16; a_nzk chunks per row tile), nonzero where the tile
  // holds a nonzero: K steps over all-zero A tiles are skipped (exact zeros)
  const uint8_t* a_nz = nullptr;
  int a_nzk = 0;
};
// nonzero flags of the 64 x 16 tiles of strided views (gemm_dmma.cu), one per job
struct NzFlagJob {
  const double* p;
  long long rs, cs;
  int rows, cols;
  uint8_t* out;  // (rows / 64 rounded up) x (cols / 16 rounded up)
};
cudaError_t launch_nz_flags64(const NzFlagJob* d_jobs, const long long* d_tile_prefix, int njobs, long long ntiles,
                              cudaStream_t s);

struct GemmTask {
  double* C;
  long long c_rs, c_cs;
  int M, N;      // extents of C (bounds for the tile)
  int m0, n0;    // tile origin (set per tile from its GemmTile record)
  int seg0, nseg;
  double alpha, beta;
};
// one output tile of a product: the product's GemmTask and the tile's
// coordinates in units of the launch's tile shape (8 bytes per tile: the
// host writes one record per tile instead of a whole task)
struct GemmTile {
  uint32_t desc;
  uint16_t mt, nt;
};

// ---- Cholesky of diagonal tiles ------------------------------------------------
// Factor the nb x nb (nb <= 64) diagonal tile W[k0:k1, k0:k1] (row-major,
// ld) in place, write its inverse to Dinv (64x64, ld 64), and flag
// breakdown (pivot <= floor or non-finite) into status[node].
struct DiagTask {
  double* W;        // node matrix base (row-major m x m, ld = m)
  double* Dinv;     // 64 x 64 scratch for this node's current panel
  int ld;
  int k0, nb;
  const double* floor;  // device: CHOL_PIVOT_RTOL * max(diag(A_BB), 0)
  int node;         // index into the status array
};

// ---- 2-D block copies ------------------------------------------------------------
struct CopyTask {
  const double* src;
  double* dst;
  long long s_rs, s_cs;
  long long d_rs, d_cs;
  int rows, cols;
  int lower = 0;  // 1: copy the lower triangle (col <= row), write zeros above it
};

// ---- column-pivoted QR (truncated at the rank) ------------------------------------
struct QrTask {
  double* Nm;          // m x c column-major (ld = m); overwritten with R and reflectors
  double* tau;         // >= min(m,c)
  double* nrm2;        // c scratch
  double* ref2;        // c scratch
  int* perm;           // c, output permutation
  const int* replay;   // optional: pivot column (original index) per step, or null
  int nreplay;
  int m, c;
  int forced_rank;     // >= 0: low-rank mode (run exactly this many steps)
  int full_steps;      // 1: run every step up to the zero-column floor, as the reference does
                       //    (rank = #{|R_kk| > tol |R_00|}); 0: stop at the rank
  double tol;
  int* out_rank;       // -> rank
  int* out_steps;      // -> reflectors computed
  double* tmp;         // m x c scratch panel (cluster variant: final column reorder)
};

// ---- FP64 GEMM emulated on the INT8 tensor cores (ozaki.cu) ------------------------
// split an R x K FP64 operand (x[r*rs + k*cs]) into exponents + 8 int8 slices,
// padded to Rp x Kp (multiples of 128 and 32)
struct OzSplitJob {
  const double* x;
  long long rs, cs;
  int R, K, Rp, Kp;
  int8_t* out;
  int* exps;
  uint8_t* nz;  // optional: nz[(r / 128) * (Kp / 32) + k / 32] = 1 where the 128 x 32 tile has a nonzero
  int* kfirst;  // optional: per row r < R, the first column k with x(r, k) != 0 (K when none)
  uint32_t* rmask;  // optional: per row r < R, mwords words; bit t: columns [32t, 32t+32) hold a nonzero
                    // value (must be zeroed beforehand when the warp kernel runs)
  int mwords;
};
// one product term C += alpha * A B^T of split operands (rows of A = rows of C)
struct OzSeg {
  const int8_t* a;
  const int8_t* b;
  const int* ea;
  const int* eb;
  int a_rp, b_rp;
  int nk;  // K tiles of 32
  double alpha;
  const uint8_t* a_nz;  // optional nonzero flags of A's 128 x 32 tiles (row tile-major, nk per row tile):
                        // all-zero K tiles are skipped (their products are exact zeros)
  const uint8_t* b_nz;  // same for B (its K padding equals A's)
};
// one 128 x 128 output tile: C = beta*C + sum of its segments (in order)
struct OzTask {
  double* C;
  long long c_rs, c_cs;
  int M, N, m0, n0;
  int seg0, nseg;
  double beta;
  int klim;    // K tiles used by this tile end before klim (triangular operands), >= nk when unlimited
  int kstart;  // ... and start at kstart
};
cudaError_t launch_oz_split(const OzSplitJob* d_jobs, const long long* d_group_prefix, int njobs,
                            long long total_groups, cudaStream_t s, bool all_rowc = false);
// row-contiguous operands (oz_split_rows_ok): groups of
// oz_split_rows_per_cta(max Kp) rows per CTA (the prefix counts those groups), rows staged once
bool oz_split_rows_ok(const OzSplitJob& j);
int oz_split_rows_per_cta(int max_kp);
cudaError_t launch_oz_split_rows(const OzSplitJob* d_jobs, const long long* d_group_prefix, int njobs,
                                 long long total_groups, int max_kp, cudaStream_t s);
cudaError_t launch_oz_gemm(const OzTask* d_tasks, int ntasks, const OzSeg* d_segs, cudaStream_t s);

// ---- apply / GEMV -----------------------------------------------------------------
// mode 0 (N): y[i] = sum_{k in [kb,ke)} A[i*lda + k] * x[k]  for rows i in [r0, r1)
// mode 1 (T): part[k] = sum_{i in [r0,r1)} A[i*lda + k] * x[i]  for k in [c0, c1)
struct GemvTask {
  const double* A;
  long long lda;
  const double* x;
  double* y;
  int r0, r1;
  int c0, c1;
  int tri;             // 1: lower-triangular A (row i uses k <= i); 2 (mode N): rows in pairs
                       //    (p, c1-1-p) for pair indices p in [r0, r1)
  const int* kfirst = nullptr;  // optional (tri == 0): row i is zero in columns < kfirst[i] (skipped)
  const uint32_t* rmask = nullptr;  // optional (tri == 0): row i's 32-column tiles holding a nonzero
  int mwords = 0;                   // (mwords words per row; all-zero tiles are skipped)
};

// partial buffer of the PCG reductions (doubles) and the offset of its arrival counter (runtime.h launch_dot)
constexpr int PCG_PART = 1024, PCG_CNT_OFF = 1000;

struct TriTask { double* p; int m; int ld; };

// y = base + sign * G x for a symmetric m x m G whose lower triangle is
// stored (row-major, ld); base may be null (then y = sign * G x)
struct SymvTask {
  const double* G;
  long long ld;
  const double* x;
  const double* base;
  double* y;
  int m;
  double sign;
  const int* idx = nullptr;  // the node's unknowns in the full vector (fused gather/scatter, see launch_symv)
  int gather_x = 0;          // fused: x = v[idx] (else x as given)
  // banded form (launch_l1_band): G x = L^{-T} (L^{-1} x) by block substitution with the
  // Cholesky factor L (bandwidth <= 64) and the inverted diagonal blocks of L^{-1}
  const double* L = nullptr;
  const double* X = nullptr;
};

struct QrFinishTask {
  const double* Nm;   // m x c panel holding the reflectors below the diagonal
  const double* tau;
  const int* steps;   // device scalar
  const int* rank;    // device scalar
  double* V;          // m x cap_s
  double* Tm;         // cap_s x cap_s
  double* Q1;         // m x cap_r
  double* G;          // cap_s x cap_s scratch (reflector Gram matrix)
  int m;
};

// CSR -> level-1 block scatter parameters (dense_kernels.cu)
struct CsrScatter {
  const long long* indptr;
  const int* indices;
  const double* values;
  const int* owner;
  const int* local;
  const int* size;           // per cell
  const long long* diag_off;
  const int* up_ptr;         // per cell: coupled cells b > a, ascending
  const int* up_cell;
  const long long* up_off;
  double* base;
  long long n;
  const int* cell_rank;      // sharded: owning rank per cell (-1 shared), nullptr = all entries
  int my_rank;
};

// out[k] = base[k] + sign * sum_{q<nrb} part[q*stride + k], k < n
struct RedSeg {
  const double* part;
  const double* base;   // may be null (then 0)
  double* out;
  int n;
  int nrb;
  int stride;
  double sign;
  const int* idx = nullptr;  // fused scatter: with a full vector v, the result goes to v[idx[k]] instead of out[k]
};

}  // namespace sgf

// kernel launchers (defined in the .cu files)
namespace sgf {
// number of kernels launched by the library (all launchers increment it)
extern unsigned long long g_kernel_launches;
inline void count_launch(unsigned long long k = 1) { g_kernel_launches += k; }

cudaError_t launch_gemm(const GemmTask* d_descs, const GemmTile* d_tiles, int ntiles, const GemmSeg* d_segs, int big_tiles,
                        cudaStream_t s);
cudaError_t launch_fill_identity(double* const* d_ptrs, const int* d_sizes, int n, cudaStream_t s);
struct ZeroRange {
  uint8_t* p;
  size_t bytes;
};
cudaError_t launch_zero_ranges(const ZeroRange* d_ranges, int n, cudaStream_t s);
cudaError_t launch_scatter_values(const double* vals, const long long* dst, long long nnz, double* base,
                                  cudaStream_t s);
// lpr: lanes per row of the mode-N kernel (8, 16 or 32)
cudaError_t launch_gemv(const GemvTask* d_tasks, int ntasks, int mode, cudaStream_t s, int lpr = 32);
// level-1 eliminations with sparse couplings (l1_sparse.cu)
constexpr int L1_KMAX = 6;  // nonzeros per coupling row (CSR rows of <= 7 entries)
struct L1RowTask {  // one coupling block, stored srows x scols row-major; A_NB = stored (trans = 0) or its transpose
  const double* p;
  int srows, scols, trans;
  long long rl0;  // row-list index of A_NB row 0
};
struct L1ETask {  // the E rows of one interior: E (c x m, ld lde) from the row lists [rl0, rl0 + c) and X = L^{-1}
  const double* X;
  long long ldx;
  double* E;
  long long lde;
  int m, c;
  long long rl0;
};
struct L1Contrib {
  long long rl_a, rl_b;  // row-list indices of the target's row 0 / column 0 in this interior's lists
  const double* G;       // A_BB^{-1}, lower triangle
  long long ldg;
};
struct L1SchurTask {  // rows [r0, r0+64) of target C (rows x cols), C -= sum of contributors [c0, c0+nc)
  double* C;
  long long ldc;
  int r0, rows, cols, diag, c0, nc;
};
cudaError_t launch_l1_rows(const L1RowTask* d_tasks, int ntasks, int* rl_n, int* rl_k, double* rl_a, int* overflow,
                           cudaStream_t s);
cudaError_t launch_l1_e(const L1ETask* d_tasks, int ntasks, int max_m, int max_c, const int* rl_n, const int* rl_k,
                        const double* rl_a, cudaStream_t s);
inline bool l1_e_fits(int max_m, int max_c) {  // shared memory of launch_l1_e
  return 16.0 * (max_m | 1) * 8 + (double)max_c * (L1_KMAX * 12 + 4) <= 220.0 * 1024;
}
cudaError_t launch_l1_schur(const L1SchurTask* d_tasks, int ntasks, const L1Contrib* d_contrib, const int* rl_n,
                            const int* rl_k, const double* rl_a, cudaStream_t s);
cudaError_t launch_symv(const SymvTask* d_tasks, int ntasks, int max_m, cudaStream_t s);
// fused form on a full vector v: x = v[idx] (gather_x) or the task's x, base = v[idx] when the
// task has a base, result written to v[idx]; false when the selected kernel has no fused form
bool symv_fused_ok(int max_m);
cudaError_t launch_symv_fused(const SymvTask* d_tasks, int ntasks, int max_m, double* v, cudaStream_t s);
// the same operation through the banded Cholesky factor (tasks carry L and X; m <= L1B_MAXM)
constexpr int L1B_MAXM = 1024;
cudaError_t launch_l1_band(const SymvTask* d_tasks, int ntasks, double* v, cudaStream_t s);
// sparse rows: mode 0: x[rid[r]] -= sum_e v[e] x[ci[e]];  mode 1: out[r] = sum_e v[e] x[ci[e]]
cudaError_t launch_sub_spmv(int nrows, const int* rid, const int* rp, const int* ci, const double* v, double* x,
                            double* out, int mode, cudaStream_t s);
cudaError_t launch_zero_tiles(const double* p, long long rs, long long cs, int rows, int cols, int tr, int tk,
                              unsigned long long* counters, cudaStream_t s);
cudaError_t launch_max_diag(const double* const* d_ptrs, const int* d_sizes, const int* d_ld, int n,
                            double* d_out, cudaStream_t s);
}  // namespace sgf
