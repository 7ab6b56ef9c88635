/*
 * sgf.h -- C ABI of the B200-native factorize -> apply -> PCG path of the
 * polynomial-preserving hierarchical factorization (arXiv 1907.03406).
 *
 * Plain pointers and sizes only; no torch / CUDA C++ types cross the
 * boundary (the stream is passed as an opaque pointer).  Every entry point
 * returns an sgf_status; sgf_last_error() returns the message of the last
 * failure on a context.  Status codes map one-to-one onto the reference's
 * exception taxonomy (errors.py:4-50):
 *   SGF_NOT_SPD       -> NotSPDError              (densela.py:106-110)
 *   SGF_SHAPE         -> ShapeMismatchError       (factorization.py:235-239)
 *   SGF_INDEFINITE    -> IndefiniteDetectedError  (krylov.py:62-63,71-72,90-91)
 *   SGF_INVALID_ARG   -> ValueError               (factorization.py:427-440)
 *   SGF_TRACE         -> RuntimeError (rank-trace divergence, factorization.py:497-509,543-549)
 *   SGF_NON_SYMMETRIC -> NonSymmetricPatternError (blockmatrix.py:109-113)
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/polyprec/):
 *   sgf_factorize          factorization.py:410-573  factorize(problem, scheme, degree, b,
 *                                                    skip_levels, compression, mode, rank_tol,
 *                                                    rank_trace)
 *   sgf_apply              factorization.py:241-271  Preconditioner.apply_inverse /
 *                                                    apply_half_inverse(_t) / apply_operator
 *   sgf_pcg                krylov.py:34-102          pcg(matvec, b, precond, tol, maxit,
 *                                                    true_residual_every)
 *   sgf_precond_stats_json factorization.py:551-567  Preconditioner.stats
 *   sgf_precond_rank_trace factorization.py:73-109   Preconditioner.rank_trace
 *   sgf_precond_factor_*   factorization.py:112-213  factor attributes (.idx .L .Q .retained
 *                                                    .node .couplings)
 *   sgf_factor_apply       factorization.py:126-209  factor .solve_forward / .solve_transpose /
 *                                                    .mult_transpose / .mult_forward
 *   sgf_pcg_ops            krylov.py:28-102          pcg with callable / @-able operators
 *   sgf_potrf_batched      densela.py:87-116         cholesky(A)
 *   sgf_trsm_batched       densela.py:119-146        tri_solve(chol, B, mode)
 *   sgf_qrcp_batched       densela.py:149-217        pivoted_qr(A, rank_tol, full_q)
 *   sgf_gemm               densela.py:79-84          matmul(a, b)
 */
#ifndef SGF_H
#define SGF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SGF_OK = 0,
  SGF_NOT_SPD = 1,
  SGF_SHAPE = 2,
  SGF_INDEFINITE = 3,
  SGF_INVALID_ARG = 4,
  SGF_TRACE = 5,
  SGF_CUDA = 6,
  SGF_OOM = 7,
  SGF_NON_SYMMETRIC = 8
} sgf_status;

/* cell kinds (partition.py:17 KIND_NAMES, plus the general family) */
enum { SGF_KIND_CELL0 = 0, SGF_KIND_CELL1 = 1, SGF_KIND_CELL2 = 2, SGF_KIND_CELL3 = 3, SGF_KIND_GENERAL = 4 };
/* modes (factorization.py:33) */
enum { SGF_MODE_POLYNOMIAL = 0, SGF_MODE_LOWRANK = 1, SGF_MODE_EXACT = 2 };
/* apply operations (factorization.py:241-271) */
enum { SGF_APPLY_INVERSE = 0, SGF_APPLY_HALF_INVERSE = 1, SGF_APPLY_HALF_INVERSE_T = 2, SGF_APPLY_OPERATOR = 3 };
/* factor types (factorization.py:112-213) */
enum { SGF_FACTOR_ELIMINATION = 0, SGF_FACTOR_COMPRESSION = 1, SGF_FACTOR_DENSE = 2 };

typedef struct sgf_ctx sgf_ctx;
typedef struct sgf_precond sgf_precond;
typedef struct sgf_csr sgf_csr;

/* What one rank contributes to the trailing matrix at the end of the
   sharded local phase (see sgf_factor_args.exchange). */
typedef struct {
  int64_t nblocks;          /* live trailing-matrix blocks: the same sorted list on every rank */
  int64_t nsend;            /* blocks holding nonzero data on this rank */
  const int32_t* send_idx;  /* host [nsend]: their positions in the block list */
  const int32_t* send_meta; /* host [4*nsend]: node a, node b, rank of a, rank of b (-1 = top separator) */
  const double* send_buf;   /* device: the blocks' entries packed in send_idx order */
  int64_t send_len;         /* doubles in send_buf */
  void* accum;              /* rank 0: handle for sgf_exchange_accumulate */
} sgf_exchange;

typedef struct {
  /* matrix: CSR pattern on the host, values on host or device */
  int64_t n;
  int64_t nnz;
  const int64_t* indptr;    /* host, n+1 */
  const int32_t* indices;   /* host, nnz */
  const double* values;     /* nnz; device pointer when values_on_device != 0 */
  int values_on_device;
  /* polynomial basis Pi (host, n x pi_cols row-major), basis.py:38-62 */
  int pi_cols;
  const double* phi;
  /* partition hierarchy (partition.py:179-217): nlevels levels */
  int nlevels;
  const int32_t* level_ncells;     /* [nlevels] */
  const int8_t* cell_kind;         /* concatenated over levels, SGF_KIND_* */
  const int8_t* cell_interior;     /* concatenated over levels, 1 = interior role */
  const int64_t* father;           /* concatenated over levels 0..nlevels-2: child -> father */
  const int64_t* l1_ptr;           /* [level_ncells[0]+1]: level-1 cell unknown lists */
  const int64_t* l1_unknowns;      /* [n] component-major unknown ids per cell, ascending cell id */
  /* options (factorization.py:410-412) */
  int compress_kind_mask;          /* bit k: kind k is compressed (COMPRESS_KINDS :37-42) */
  int raw_kind_mask;               /* bit k: couplings to kind k enter unfiltered (UNFILTERED_KINDS :47) */
  int skip_levels;
  int compression;
  int mode;                        /* SGF_MODE_* */
  double rank_tol;
  /* low-rank replay: (level, node, rank) triples of a polynomial run */
  int n_trace;
  const int32_t* trace;
  /* QR pivot replay (parity mode): one permutation per compression in
     reference execution order; replay_ptr has n_replay+1 entries */
  int n_replay;
  const int64_t* replay_ptr;
  const int32_t* replay_perm;
  /* alternative to phi: build Pi natively from vertex coordinates (host,
     n_vertices x 3) with basis.py:38-62's rule (degree 0/1/2, components
     1/3); used when phi == NULL */
  const double* coords;
  int64_t n_vertices;
  int degree;
  int components;
  /* sharding across ranks, one process per GPU; shard_count
     <= 1 disables it.  Every rank runs the same symbolic factorization; a
     rank computes only the eliminations of the level-1 cells it owns
     (cell_rank[c] == shard_rank; -1 marks top-separator cells, whose blocks
     belong to rank 0) for the eliminations of levels 1..shard_stop_level.
     Then `exchange` is called once on every rank with the trailing-matrix
     blocks this rank holds nonzero data for (its own cells' blocks and its
     partial Schur sums of shared blocks, packed); the callback must deliver
     every other rank's contribution to rank 0, which adds them in ascending
     rank order with sgf_exchange_accumulate before returning, and continues
     with the remaining levels while the other ranks stop. */
  int shard_rank;
  int shard_count;
  const int32_t* cell_rank;
  int shard_stop_level;
  int (*exchange)(void* user, const sgf_exchange* x);
  void* exchange_user;
} sgf_factor_args;

typedef struct {
  int iterations;
  int converged;
  double final_rel_residual;
  double wall_time;          /* seconds, device-timed */
  int history_len;
} sgf_pcg_report;

int sgf_create(sgf_ctx** ctx, int device);
int sgf_destroy(sgf_ctx* ctx);
const char* sgf_last_error(const sgf_ctx* ctx);
/* the stream all work of the context runs on (cudaStream_t as void*) */
void* sgf_stream(sgf_ctx* ctx);
int sgf_sync(sgf_ctx* ctx);
/* returns the device memory the library caches for reuse (freed arena chunks
   of this context's device) to the driver, e.g. before another process on
   the same GPU needs it; live factors and matrices are untouched */
int sgf_trim(sgf_ctx* ctx);

int sgf_factorize(sgf_ctx* ctx, const sgf_factor_args* args, sgf_precond** out);
int sgf_precond_free(sgf_precond* p);
int64_t sgf_precond_n(const sgf_precond* p);
const char* sgf_precond_stats_json(const sgf_precond* p);
int sgf_precond_rank_trace(const sgf_precond* p, int32_t* out, int cap);  /* returns #entries */
int sgf_precond_num_factors(const sgf_precond* p);

/* Measurement helper (bench.py's apply roofline; no reference counterpart):
 * bytes per sweep of the stored couplings E and of the L^{-1} triangles that
 * carry tile masks, out[0] dense (c*m*8, and m(m+1)/2*8) and out[1] in the
 * 32-column tiles that hold a nonzero -- the part the apply kernels stream
 * (all-zero tiles are skipped; apply.cpp).  Synchronises. */
int sgf_precond_coupling_bytes(const sgf_precond* p, double* out);
/* the same restricted to the factors of one level (level >= 1; 0: all) */
int sgf_precond_coupling_bytes_level(const sgf_precond* p, int level, double* out);
/* diagnostic: E bytes of a level under the forward sweeps' skipping
   granularities (out[6]: dense, nonzero tiles, from the first nonzero tile,
   256-column chunks, chunks trimmed to their nonzero span, nonzero-tile runs) */
int sgf_precond_coupling_bytes_detail(const sgf_precond* p, int level, double* out);
/* info[0..7] = type, node, m (idx size), c (coupling rows), retained, level, reflectors, QR columns */
int sgf_precond_factor_info(const sgf_precond* p, int k, int64_t* info);
/* what: 0 idx (int64 m), 1 L (m*m), 2 couplings E (c*m), 3 coupling idx (int64 c),
         4 Q (m*m, compression), 5 inverse operator (m*m: L^-1, or Q^T L^-1), 6 QR perm (int64) */
int sgf_precond_factor_copy(const sgf_precond* p, int k, int what, void* host_out, int64_t cap_bytes);

/* y = op(x); x,y device pointers when on_device != 0 else host.  Never
   mutates x (factorization.py:235-239 copies). */
int sgf_apply(sgf_precond* p, int op, const double* x, double* y, int on_device);

/* Rank 0 inside its exchange callback: add another rank's packed blocks
   (positions idx[0..n) of the block list, entries packed in that order;
   `packed` is a device pointer) into the trailing matrix. */
int sgf_exchange_accumulate(void* accum, const int32_t* idx, int64_t n, const double* packed);

/* Sharded preconditioners: factors [0, n_local) belong to the rank's local
   phase, [n_local, n) to the top part (rank 0).  n_local_unknowns = unknowns
   eliminated by the local factors; n_top = unknowns still active when the
   local phase ended (identical on every rank).  A single-GPU preconditioner
   has n_local = all factors and n_top = 0. */
int sgf_precond_shard_info(const sgf_precond* p, int64_t* n_local_factors, int64_t* n_local_unknowns,
                           int64_t* n_top);
/* which: 0 local eliminated unknowns, 1 top unknowns (int64) */
int sgf_precond_shard_set(const sgf_precond* p, int which, int64_t* out, int64_t cap);
/* In-place partial sweeps on a device n-vector: part 0 forward over the
   local factors, 1 forward then backward over the top factors, 2 backward
   over the local factors.  Parts 0, 1, 2 in sequence = apply_inverse. */
int sgf_apply_part(sgf_precond* p, int part, double* y);
/* The sharded apply_inverse on distributed vectors (entries owned by this
   rank: its local unknowns, plus the top unknowns on rank 0; others zero),
   in three stages around the caller's collectives on top_buf (n_top):
     stage 0: y = x; local forward sweeps; top_buf = y[top] - x[top]
              -> caller sums top_buf onto rank 0
     stage 1 (rank 0): y[top] = x[top] + top_buf; top sweeps; top_buf = y[top]
              -> caller broadcasts top_buf
     stage 2: y[top] = top_buf; local backward sweeps; non-owned entries of
              y zeroed when mask != 0
   Device pointers; x is not modified. */
int sgf_apply_shard(sgf_precond* p, int stage, const double* x, double* y, double* top_buf, int mask);
/* Device vector helpers on the context stream: out[i] = x[idx[i]] and
   y[idx[i]] = v[i] (int32 device indices). */
int sgf_vec_gather(sgf_ctx* ctx, const double* x, const int32_t* idx, double* out, int64_t n);
int sgf_vec_scatter(sgf_ctx* ctx, const double* v, const int32_t* idx, double* y, int64_t n);

int sgf_csr_create(sgf_ctx* ctx, int64_t n, int64_t nnz, const int64_t* indptr, const int32_t* indices,
                   const double* values, int on_device, sgf_csr** out);
int sgf_csr_free(sgf_csr* a);
int sgf_spmv(sgf_csr* a, const double* x, double* y, int on_device);

/* PCG with the reference recurrence; precond may be NULL (identity).
   history must hold maxit + 2 doubles. */
int sgf_pcg(sgf_ctx* ctx, sgf_csr* a, sgf_precond* p, const double* b, double* x, double tol, int maxit,
            int true_residual_every, int on_device, sgf_pcg_report* rep, double* history);

/* PCG whose preconditioner is a callback on device n-vectors (out = M^-1 in,
   enqueued on the context stream; nonzero return = failure); used by the
   sharded solve, where M^-1 includes collectives. */
typedef int (*sgf_precond_fn)(void* user, const double* in, double* out);
int sgf_pcg_cb(sgf_ctx* ctx, sgf_csr* a, sgf_precond_fn fn, void* user, const double* b, double* x, double tol,
               int maxit, int true_residual_every, int on_device, sgf_pcg_report* rep, double* history);

/* PCG over general operators (krylov.py:28-31 _as_linop: matvec / precond
   may be matrices, `@`-able objects or callables).  Exactly one of `a` (a
   device CSR) and `mv` (out = A in on device n-vectors, enqueued on the
   context stream; nonzero return = failure) is given; at most one of `p`
   and `pf`.  The recurrence, dots and vector updates run on the device as
   in sgf_pcg; only the callbacks run wherever the caller put them. */
typedef int (*sgf_matvec_fn)(void* user, const double* in, double* out);
int sgf_pcg_ops(sgf_ctx* ctx, int64_t n, sgf_csr* a, sgf_matvec_fn mv, void* mv_user, sgf_precond* p,
                sgf_precond_fn pf, void* pf_user, const double* b, double* x, double tol, int maxit,
                int true_residual_every, int on_device, sgf_pcg_report* rep, double* history);

/* Distributed PCG (the sharded solve): every vector is a full-length device
   vector holding this rank's owned entries (zero elsewhere); `mv` computes
   the owned rows of A in (after its own halo exchange), `pf` the sharded
   preconditioner, and `reduce` sums nvals host doubles in place across the
   ranks (same order on every rank, so every rank takes the same branches).
   Same recurrence and report as sgf_pcg. */
typedef int (*sgf_reduce_fn)(void* user, double* vals, int nvals);
int sgf_pcg_dist(sgf_ctx* ctx, int64_t n, sgf_matvec_fn mv, void* mv_user, sgf_precond_fn pf, void* pf_user,
                 sgf_reduce_fn reduce, void* reduce_user, const double* b, double* x, double tol, int maxit,
                 int true_residual_every, sgf_pcg_report* rep, double* history);

/* Stream-ordered copy on the context stream (host or device pointers,
   cudaMemcpyDefault), synchronised before returning. */
int sgf_memcpy(sgf_ctx* ctx, void* dst, const void* src, int64_t bytes);
/* Make the context stream wait for all work enqueued so far on `stream`
   (a cudaStream_t, e.g. torch's current stream) before its next launch. */
int sgf_stream_wait(sgf_ctx* ctx, void* stream);

/* One factor's operation, in place on an n-vector (device pointer when
   on_device != 0, else host): op 0 solve_forward, 1 solve_transpose,
   2 mult_transpose, 3 mult_forward (factorization.py:126-148, 173-183,
   199-209: EliminationFactor / CompressionFactor / DenseFactor methods). */
enum { SGF_SOLVE_FORWARD = 0, SGF_SOLVE_TRANSPOSE = 1, SGF_MULT_TRANSPOSE = 2, SGF_MULT_FORWARD = 3 };
int sgf_factor_apply(sgf_precond* p, int k, int op, double* x, int on_device);

/* Per-primitive entry points (densela.py:79-217).  Matrices are row-major
   DEVICE buffers; the per-matrix size / leading-dimension / pointer arrays
   and the outputs status / rank are HOST arrays of `batch` entries.
   sgf_potrf_batched  cholesky (densela.py:87-116): L_b lower with zeros
     above; status_b = SGF_INVALID_ARG (NaN/Inf, densela.py:43-49),
     SGF_NON_SYMMETRIC (max|A-A^T| > 1e-12 max|A|, :97-104), SGF_NOT_SPD
     (pivot <= 1e-14 max diag, :105-110; pivot_index / pivot_value report it)
   sgf_trsm_batched   tri_solve (densela.py:119-146): mode 0 X = L^-1 B
     (m x nrhs), 1 X = L^-T B, 2 X = B L^-T (nrhs x m)
   sgf_qrcp_batched   pivoted_qr (densela.py:149-217): A (m x c) ->
     perm (c, int32), R (min(m,c) x c upper trapezoid), Q (m x min(m,c), or
     m x m when full_q), rank = #{|R_ii| > rank_tol |R_00|}; steps = the
     Householder reflections performed
   sgf_gemm           matmul (densela.py:79-84): C = alpha A B + beta C,
     A m x k, B k x n */
int sgf_potrf_batched(sgf_ctx* ctx, int batch, const int32_t* m, const double* const* A, const int32_t* lda,
                      double* const* L, const int32_t* ldl, int32_t* status, int32_t* pivot_index,
                      double* pivot_value);
int sgf_trsm_batched(sgf_ctx* ctx, int batch, const int32_t* m, const int32_t* nrhs, const int32_t* mode,
                     const double* const* L, const int32_t* ldl, const double* const* B, const int32_t* ldb,
                     double* const* X, const int32_t* ldx);
int sgf_qrcp_batched(sgf_ctx* ctx, int batch, const int32_t* m, const int32_t* c, const double* const* A,
                     const int32_t* lda, double rank_tol, int full_q, double* const* Q, double* const* R,
                     int32_t* const* perm, int32_t* rank, int32_t* steps);
int sgf_gemm(sgf_ctx* ctx, int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
             double beta, double* C, int ldc);

/* Host helper (partition.py:142-199, 232-242 for the level-1 cells): unknown
   ids grouped by cell (cells in id order, vertices ascending, components
   major within a cell) and the per-cell pointer, for a nested/general grid
   level given per axis the index extent [lo, hi] of every label.  Cell id =
   (rank_x * ty + rank_y) * tz + rank_z. */
int sgf_cell_unknowns(int nx, int ny, int nz, int tx, int ty, int tz, const int64_t* lox, const int64_t* hix,
                      const int64_t* loy, const int64_t* hiy, const int64_t* loz, const int64_t* hiz, int components,
                      int64_t* out_ptr, int64_t* out_unknowns);

/* instrumentation (no reference counterpart): kernels launched so far, and
   per-kernel-class CUDA-event timing.  Classes: 0 GEMM on DMMA (work = flops),
   1 GEMV (bytes), 2 SpMV (bytes), 3 QR, 4 diagonal Cholesky, 5 copies (bytes),
   6 vector ops, 7 FP64 products on the INT8 tensor cores (FP64 flops),
   8 their operand splits (bytes).  out[3*cls + 0..2] = milliseconds, work,
   launches. */
uint64_t sgf_kernel_launches(void);
int sgf_profile_enable(int on);
int sgf_profile_read(double* out, int cap);

#ifdef __cplusplus
}
#endif
#endif
