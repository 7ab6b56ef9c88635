// Device-resident preconditioner: the ordered elementary factors of the
// reference (factorization.py:112-213) plus the level-batched apply plan.
#pragma once
#include <array>
#include <deque>
#include <functional>
#include <memory>

#include "runtime.h"

namespace sgf {

struct Factor {
  int type = 0;   // SGF_FACTOR_*
  int node = -1;
  int level = 0;  // 1-based level of the factorization pass (dense: levels+1)
  int m = 0, c = 0, r = 0, steps = 0;
  int ld = 0;                 // leading dimension of L, inv and E (pad_ld(m))
  std::vector<int64_t> idx;   // node actives at factor time
  std::vector<int64_t> nidx;  // elimination: stacked neighbour actives (sorted neighbour order)
  double* L = nullptr;        // m x m lower (row-major)
  double* inv = nullptr;      // m x m: L^{-1} (elim/dense) or Q^T L^{-1} (compression)
  double* E = nullptr;        // c x m couplings E_N = A_NB L^{-T}, stacked
  int* ekfirst = nullptr;     // per row of E: first nonzero column (leading zeros: E = A_NB L^{-T} with
                              // L^{-T} upper triangular keeps the leading zero columns of A_NB's rows)
  uint32_t* emask = nullptr;  // per row of E: bit t = 32-column tile t holds a nonzero (emw words per row;
  int emw = 0;                // E is block-sparse: zero runs at the interior's pieces, not only leading)
  int* xkfirst = nullptr;     // the same for the rows of L^{-1} (when its operand split recorded them:
  uint32_t* xmask = nullptr;  // the emulated levels), emw words per row
  int xmw = 0;
  double* V = nullptr;        // m x steps reflectors (column-major, unit lower trapezoid)
  double* Tw = nullptr;       // steps x steps compact-WY factor (row-major, upper)
  double* LQ = nullptr;       // compression: L Q (m x m, ld), formed on first apply_operator
  double* G = nullptr;        // level-1 elimination: A_BB^{-1} = L^{-T} L^{-1} (lower triangle, ld)
  int bw = -1;                // level-1 elimination: lower bandwidth of A_BB (and of L) in the node's order
  std::vector<int32_t> perm;  // compression: QR column permutation (first `steps` meaningful)
  int* perm_dev = nullptr;    // device copy until the end-of-factorization readback
  int ncols = 0;              // compression: columns of the rank basis N
};

// Level-1 couplings A_NB of the level-1 eliminations, which are still the
// original sparse matrix entries: apply_inverse uses them with G = A_BB^{-1}
// instead of streaming the dense E = A_NB L^{-T} twice (see apply.cpp).
struct L1Couplings {
  bool ready = false;
  int nb = 0;                  // rows: level-1 interior unknowns, in factor order
  int* b_rp = nullptr;         // [nb+1]
  int* b_ci = nullptr;         // neighbour unknown ids
  double* b_v = nullptr;
  int nf = 0;                  // rows: neighbour unknowns coupled to those interiors
  int* f_rid = nullptr;        // [nf] their ids
  int* f_rp = nullptr;         // [nf+1]
  int* f_ci = nullptr;         // interior unknown ids
  double* f_v = nullptr;
};

struct ApplyPlan;
void destroy_plan(ApplyPlan* p);
ApplyPlan* build_plan(class Precond* P);
void plan_extend(class Precond* P, size_t begin, size_t end);  // add groups of factors [begin, end)
// same, reading the factors only through the given (stable) pointers: safe to
// run on a worker thread while the driver keeps appending factors
void plan_extend_ptrs(class Precond* P, size_t begin, const std::vector<const Factor*>& fs);
void plan_finish(class Precond* P);
void plan_init(class Precond* P);

class Precond {
 public:
  Ctx* ctx = nullptr;
  int64_t n = 0;
  std::deque<Factor> factors;  // deque: stable element addresses while appending
  std::string stats;
  std::vector<int32_t> trace;  // (level, node, rank) triples
  Arena store;
  ApplyPlan* plan = nullptr;
  // sharding: factors [0, n_local) are the rank's local phase; top_idx are
  // the unknowns active when it ended (empty on a single GPU)
  L1Couplings l1;
  // level-1 couplings E = A_NB L^{-T} of the sparse level-1 path are formed
  // on first use (apply_inverse and the Schur updates never read them; the
  // half sweeps, apply_operator and the host factor views do): the row lists
  // and the task list are kept until then (materialize_l1_e)
  struct L1EPending {
    bool pending = false;
    std::vector<L1ETask> tasks;
    int max_m = 0, max_c = 0;
    int* rl_n = nullptr;
    int* rl_k = nullptr;
    double* rl_a = nullptr;
  } l1e;
  bool sharded = false;
  size_t n_local = 0;
  std::vector<int64_t> top_idx;
  // sharded: per exchange {blocks sent, bytes sent, blocks in the list, bytes of the whole list}
  std::vector<std::array<int64_t, 4>> exchange_log;
  // sharded apply (sgf_apply_shard): device top indices and owned-entry flags, built on first use
  int shard_rank = 0;
  int* d_top = nullptr;
  unsigned char* d_owned = nullptr;
  size_t local_count() const { return sharded ? n_local : factors.size(); }
  ~Precond() {
    if (plan) destroy_plan(plan);
  }
};

// the trailing-matrix contribution of one rank at the end of the sharded local phase
struct ShardExchange {
  cudaStream_t st = nullptr;
  Arena* scratch = nullptr;
  std::vector<double*> ptrs;     // every live block, key order
  std::vector<long long> counts;
  long long total = 0;           // bytes of all blocks
  std::vector<int32_t> send_idx;
  std::vector<int32_t> send_meta;
  double* send_buf = nullptr;
  long long send_len = 0;
};
void exchange_accumulate(ShardExchange* X, const int32_t* idx, int64_t n, const double* packed);

Precond* factorize(Ctx& ctx, const sgf_factor_args& a);
void materialize_l1_e(Precond* P);  // form the pending level-1 couplings E (stream ordered)
void apply_op(Precond* P, int op, const double* d_x, double* d_y);
void apply_part(Precond* P, int part, double* d_y);

struct Csr {
  Ctx* ctx = nullptr;
  int64_t n = 0, nnz = 0;
  long long* rp = nullptr;
  int* rp32 = nullptr;  // int32 row pointers when nnz fits (the SpMV reads these)
  int* ci = nullptr;
  double* v = nullptr;
  Arena mem;
  double* ws = nullptr;   // PCG workspace (4n + 520), one solve at a time per matrix
  double* hsc = nullptr;  // pinned scalars read back by the PCG
  ~Csr() {
    if (hsc) cudaFreeHost(hsc);
  }
};
void spmv(Csr* A, const double* d_x, double* d_y, const double* d_b);
// preconditioner: out = M^-1 in on device vectors (empty = identity)
using PrecFn = std::function<void(const double*, double*)>;
// operator: out = A in on device vectors (empty = A's own CSR SpMV)
using MatFn = std::function<void(const double*, double*)>;
// A owns the PCG workspace; with an operator callback its CSR arrays may be
// absent (only A->n is used)
void pcg(Ctx& ctx, Csr* A, const MatFn& Aop, const PrecFn& M, const double* d_b, double* d_x, double tol, int maxit,
         int true_every, sgf_pcg_report* rep, double* history);
// sums host doubles in place across the ranks of a sharded solve
using ReduceFn = std::function<void(double*, int)>;
void pcg_dist(Ctx& ctx, int64_t n, const MatFn& Aop, const PrecFn& M, const ReduceFn& reduce, const double* d_b,
              double* d_x, double tol, int maxit, int true_every, sgf_pcg_report* rep, double* history);
void apply_shard(Precond* P, int stage, const double* x, double* y, double* top_buf, int mask);

}  // namespace sgf
