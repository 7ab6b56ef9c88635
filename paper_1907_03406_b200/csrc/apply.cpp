// Level-batched preconditioner application and device PCG.
//
// apply_inverse = W^{-T} W^{-1} x (reference factorization.py:255-262).
// Factors of one (level, kind) group touch disjoint node index sets and
// commute inside the sweeps, so each group is one batched
// phase: gathers of the group's unknowns, batched GEMVs over the stored
// matrices, scatters back.  Elimination forward sweeps update shared
// separator unknowns x_N -= E_N z_B; the plan's combine list applies those
// in ascending factor order, exactly the reference's sequence.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <thread>
#include <utility>

#include "precond.h"

namespace sgf {

namespace {
constexpr int GN_ROWS = 64;   // rows per gemv_n CTA
constexpr int GT_ROWS = 256;  // rows per gemv_t partial
constexpr int GT_COLS = 512;  // columns per gemv_t CTA (2 per thread)
}  // namespace

struct Group {
  int type = 0;
  long long nm = 0, nc = 0;  // sum of m, sum of c
  int* idx = nullptr;
  int* nidx = nullptr;
  GemvTask* fwd1 = nullptr;
  int nf1 = 0;
  GemvTask* fwd2 = nullptr;
  int nf2 = 0;
  int* tgt = nullptr;
  long long* tptr = nullptr;
  long long* tpos = nullptr;
  long long ntgt = 0;
  GemvTask* bwd1 = nullptr;
  int nb1 = 0;
  int b1_mode = 1;  // 2: every task carries the rows' leading-zero offsets (gemv_t_lead_kernel)
  int f2_mode = 0;  // 3: the couplings' rows are block-sparse (task.kfirst / task.rmask)
  int f1_mode = 0, b2_mode = 1;  // 3 / 2: L^{-1}'s rows carry tile masks
  RedSeg* red1 = nullptr;
  int nred1 = 0, maxn1 = 0;
  GemvTask* bwd2 = nullptr;
  int nb2 = 0;
  RedSeg* red2 = nullptr;
  int nred2 = 0, maxn2 = 0;
  double bytes_f1 = 0, bytes_f2 = 0, bytes_b1 = 0, bytes_b2 = 0;  // matrix bytes streamed
  double *xb = nullptr, *zb = nullptr, *acc = nullptr, *xn = nullptr, *t = nullptr, *part = nullptr;  // workspaces
  size_t f0 = 0, f1 = 0;  // factor range
  int gn_rows = GN_ROWS, gt_rows = GT_ROWS;  // finer row blocks for groups of few large matrices
  int lpr1 = 32, lpr2 = 32;                   // mode-N lanes per row (inverse, couplings)
  // level-1 eliminations in apply_inverse: G = A_BB^{-1} with the sparse couplings
  bool sym = false;
  bool band = false;          // ... through the banded Cholesky factor (launch_l1_band)
  double bytes_band = 0;
  SymvTask* sym_f = nullptr;  // zb = G xb
  SymvTask* sym_b = nullptr;  // zb = xb - G acc
  int nsym = 0, sym_maxm = 0;
  double bytes_sym = 0;
  // apply_operator task lists (built on first use)
  GemvTask *oT = nullptr, *oE = nullptr, *oL = nullptr;
  int noT = 0, noE = 0, noL = 0;
  RedSeg* oRed = nullptr;
  int noRed = 0;
  double bytes_oT = 0, bytes_oE = 0, bytes_oL = 0;
};

// lanes per row for mode-N rows of `len2` 16-byte words on average
// (64: rows of >= 1536 entries, streamed through the bulk-copy kernel)
static int lanes_for(double len2) { return len2 <= 48 ? 8 : (len2 <= 96 ? 16 : (len2 < 768 ? 32 : 64)); }

// algorithmic bytes of the matrix entries a GEMV task list reads
static double gemv_bytes(const std::vector<GemvTask>& v, int mode) {
  double b = 0.0;
  for (const auto& t : v) {
    if (!t.tri) {
      b += 8.0 * (t.r1 - t.r0) * (t.c1 - t.c0);
    } else if (t.tri == 2) {
      for (int p = t.r0; p < t.r1; ++p) b += 8.0 * ((p + 1) + (t.c1 - 1 - p == p ? 0 : t.c1 - p));
    } else if (mode == 0) {
      for (int i = t.r0; i < t.r1; ++i) b += 8.0 * std::max(0, std::min(t.c1, i + 1) - t.c0);
    } else {
      for (int k = t.c0; k < t.c1; ++k) b += 8.0 * std::max(0, t.r1 - std::max(t.r0, k));
    }
  }
  return b;
}

struct ApplyPlan {
  Arena mem;
  std::vector<Group> groups;
  double* work = nullptr;  // n-vector (apply in place)
  std::vector<int> tix;    // host scratch of the plan builder (released by plan_finish)
  bool op_ready = false;   // apply_operator tasks built
  long long n = 0;
  // CUDA graphs of the sweeps on `work` (index = op), captured on first use
  cudaGraphExec_t graph[3] = {nullptr, nullptr, nullptr};
  unsigned long long graph_launches[3] = {0, 0, 0};
  // task lists and index arrays are uploaded on the context's upload stream
  // (the plan worker runs beside the factorization); the sweeps run on `s`
  ApplyPlan(cudaStream_t s, cudaStream_t upload) : mem(upload, (size_t)64 << 20) { mem.use_plan_pool(s); }
  ~ApplyPlan() {
    for (auto& g : graph)
      if (g) cudaGraphExecDestroy(g);
  }
};

void destroy_plan(ApplyPlan* p) { delete p; }

// lower triangle in row pairs (p, rows-1-p): 32 pairs per task
static void add_gemv_tri_pairs(std::vector<GemvTask>& v, const double* A, long long lda, const double* x, double* y,
                               int rows) {
  const int np = (rows + 1) / 2;
  for (int p0 = 0; p0 < np; p0 += 32) {
    GemvTask t;
    t.A = A;
    t.lda = lda;
    t.x = x;
    t.y = y;
    t.r0 = p0;
    t.r1 = std::min(np, p0 + 32);
    t.c0 = 0;
    t.c1 = rows;
    t.tri = 2;
    v.push_back(t);
  }
}

static void add_gemv_n(std::vector<GemvTask>& v, const double* A, long long lda, const double* x, double* y, int rows,
                       int cols, int tri, int rows_per = GN_ROWS, const int* kfirst = nullptr,
                       const uint32_t* rmask = nullptr, int mwords = 0) {
  for (int r0 = 0; r0 < rows; r0 += rows_per) {
    GemvTask t;
    t.A = A;
    t.lda = lda;
    t.x = x;
    t.y = y;
    t.r0 = r0;
    t.r1 = std::min(rows, r0 + rows_per);
    t.c0 = 0;
    t.c1 = cols;
    t.tri = tri;
    t.kfirst = kfirst;
    t.rmask = rmask;
    t.mwords = mwords;
    v.push_back(t);
  }
}

// partials part[rb*cols + k] = sum_{i in rb} A[i,k] x[i]; returns #row blocks
static int add_gemv_t(std::vector<GemvTask>& v, const double* A, long long lda, const double* x, double* part,
                      int rows, int cols, int tri, int rows_per = GT_ROWS, const int* kfirst = nullptr,
                      const uint32_t* rmask = nullptr, int mwords = 0) {
  int nrb = 0;
  for (int r0 = 0; r0 < rows; r0 += rows_per, ++nrb)
    for (int c0 = 0; c0 < cols; c0 += GT_COLS) {
      GemvTask t;
      t.A = A;
      t.lda = lda;
      t.x = x;
      t.y = part + (long long)nrb * cols;
      t.r0 = r0;
      t.r1 = std::min(rows, r0 + rows_per);
      t.c0 = c0;
      t.c1 = std::min(cols, c0 + GT_COLS);
      t.tri = tri;
      t.kfirst = kfirst;
      t.rmask = rmask;
      t.mwords = mwords;
      v.push_back(t);
    }
  return nrb;
}

// Extend the plan with the groups of factors [begin, end).  Called by the
// factorization driver right after each level's kernels are enqueued, so this
// host work overlaps the device execution of the level.  Every group owns its
// workspace slices.
void plan_extend(Precond* P, size_t begin, size_t end) {
  std::vector<const Factor*> fs;
  for (size_t i = begin; i < end; ++i) fs.push_back(&P->factors[i]);
  plan_extend_ptrs(P, begin, fs);
}

void plan_init(Precond* P) {
  if (P->plan) return;
  P->plan = new ApplyPlan(P->ctx->stream, P->ctx->upload_stream);
  P->plan->n = P->n;
  P->plan->work = P->plan->mem.alloc(std::max<long long>(P->n, 1));
  P->plan->tix.assign(P->n, -1);
}

void plan_extend_ptrs(Precond* P, size_t begin, const std::vector<const Factor*>& fs) {
  HostTimer ht("plan_extend");
  plan_init(P);
  ApplyPlan* plan = P->plan;
  std::vector<int>& tix = plan->tix;
  // groups: consecutive factors of the same (level, type); indices local to fs
  std::vector<std::pair<size_t, size_t>> ranges;
  for (size_t i = 0; i < fs.size();) {
    size_t j = i + 1;
    while (j < fs.size() && fs[j]->type == fs[i]->type && fs[j]->level == fs[i]->level &&
           fs[i]->type != SGF_FACTOR_DENSE)
      ++j;
    ranges.push_back({i, j});
    i = j;
  }
  for (auto& rg : ranges) {
    Group g;
    g.type = fs[rg.first]->type;
    g.f0 = begin + rg.first;
    g.f1 = begin + rg.second;
    long long sm = 0, sc = 0, sp = 0, ntn = 0, ntt = 0;
    for (size_t i = rg.first; i < rg.second; ++i) {
      const Factor& f = *fs[i];
      const long long cb = (f.m + GT_COLS - 1) / GT_COLS;
      ntn += (f.m + GN_ROWS - 1) / GN_ROWS + (f.c + GN_ROWS - 1) / GN_ROWS;
      ntt += ((f.m + GT_ROWS - 1) / GT_ROWS + (f.c + GT_ROWS - 1) / GT_ROWS) * cb;
    }
    // a group of a few large matrices (top levels, final dense) would leave
    // most SMs idle: one row per warp for gemv_n, 32-row partials for gemv_t
    if (ntn < 4 * 148) g.gn_rows = 8;
    if (ntt < 4 * 148) g.gt_rows = 32;
    for (size_t i = rg.first; i < rg.second; ++i) {
      const Factor& f = *fs[i];
      sm += f.m;
      sc += f.c;
      const long long rbE = (f.c + g.gt_rows - 1) / g.gt_rows, rbL = (f.m + g.gt_rows - 1) / g.gt_rows;
      sp += (rbE + rbL) * f.m;  // apply_operator stacks both partial sets
    }
    g.xb = plan->mem.alloc(std::max(sm, 1LL));
    g.zb = plan->mem.alloc(std::max(sm, 1LL));
    g.acc = plan->mem.alloc(std::max(sm, 1LL));
    g.xn = plan->mem.alloc(std::max(sc, 1LL));
    g.t = plan->mem.alloc(std::max(sc, 1LL));
    g.part = plan->mem.alloc(std::max(sp, 1LL));
    std::vector<int> idx, nidx;
    std::vector<GemvTask> f1, f2, b1, b2;
    std::vector<RedSeg> r1, r2;
    long long om = 0, oc = 0, op = 0;
    std::vector<std::pair<int64_t, long long>> contrib;  // (unknown, t position) in factor order
    for (size_t i = rg.first; i < rg.second; ++i) {
      const Factor& f = *fs[i];
      for (auto u : f.idx) idx.push_back((int)u);
      const int tri = (g.type != SGF_FACTOR_COMPRESSION);
      if (f.xmask) {  // block-sparse L^{-1} rows: zero tiles skipped (rows taken dynamically)
        add_gemv_n(f1, f.inv, f.ld, g.xb + om, g.zb + om, f.m, f.m, 1, g.gn_rows, f.xkfirst, f.xmask, f.xmw);
      } else if (tri && g.gn_rows == GN_ROWS) {
        add_gemv_tri_pairs(f1, f.inv, f.ld, g.xb + om, g.zb + om, f.m);
      } else {
        add_gemv_n(f1, f.inv, f.ld, g.xb + om, g.zb + om, f.m, f.m, tri, g.gn_rows);
      }
      if (g.type == SGF_FACTOR_ELIMINATION) {
        for (auto u : f.nidx) nidx.push_back((int)u);
        if (f.c > 0) add_gemv_n(f2, f.E, f.ld, g.zb + om, g.t + oc, f.c, f.m, 0, g.gn_rows, f.ekfirst, f.emask, f.emw);
        for (int p = 0; p < f.c; ++p) contrib.push_back({f.nidx[p], oc + p});
        int nrb = f.c > 0 ? add_gemv_t(b1, f.E, f.ld, g.xn + oc, g.part + op, f.c, f.m, 0, g.gt_rows, f.ekfirst,
                                       f.emask, f.emw)
                          : 0;
        r1.push_back(RedSeg{g.part + op, g.xb + om, g.acc + om, f.m, nrb, f.m, -1.0});
        // second stage reuses the partial buffer after red1 consumed it (masked
        // L^{-1}: every row of the square with its tile mask; the zero upper
        // triangle is skipped by the mask)
        int nrb2 = f.xmask ? add_gemv_t(b2, f.inv, f.ld, g.acc + om, g.part + op, f.m, f.m, 0, g.gt_rows, f.xkfirst,
                                        f.xmask, f.xmw)
                           : add_gemv_t(b2, f.inv, f.ld, g.acc + om, g.part + op, f.m, f.m, 1, g.gt_rows);
        r2.push_back(RedSeg{g.part + op, nullptr, g.zb + om, f.m, nrb2, f.m, 1.0});
        op += std::max<long long>(nrb, nrb2) * f.m;
      } else {
        int nrb = add_gemv_t(b1, f.inv, f.ld, g.xb + om, g.part + op, f.m, f.m, tri, g.gt_rows);
        r1.push_back(RedSeg{g.part + op, nullptr, g.zb + om, f.m, nrb, f.m, 1.0});
        op += (long long)nrb * f.m;
      }
        g.maxn1 = std::max(g.maxn1, f.m);
      g.maxn2 = std::max(g.maxn2, f.m);
      om += f.m;
      oc += f.c;
    }
    g.nm = om;
    g.nc = oc;
    // level-1 eliminations with G and the coupling lists of the whole level
    bool sym = g.type == SGF_FACTOR_ELIMINATION && P->l1.ready && om == P->l1.nb;
    for (size_t i = rg.first; sym && i < rg.second; ++i) sym = fs[i]->G != nullptr && fs[i]->level == 1;
    g.idx = plan->mem.upload(idx);
    if (sym) {
      std::vector<SymvTask> tf, tb;
      long long o = 0;
      static const bool band_ok = !(getenv("SGF_L1_BAND") && atoi(getenv("SGF_L1_BAND")) == 0);
      g.band = band_ok;
      for (size_t i = rg.first; i < rg.second; ++i) {
        const Factor& f = *fs[i];
        g.band = g.band && f.bw >= 1 && f.bw <= 64 && f.m <= L1B_MAXM && f.L && f.inv;
        for (int p = 0; p * 64 < f.m; ++p) {  // entries of X_pp's triangle and of S_p's band, read twice
          const double rows = std::min(64, f.m - 64 * p);
          g.bytes_band += 2.0 * 8.0 * (rows * (rows + 1.0) / 2.0 + (p ? rows * 64.0 - rows * (rows - 1.0) / 2.0 : 0.0));
        }
        // unfused form: x/base/result in the group's gathered buffers; fused
        // form (launch_symv_fused): through idx on the full vector
        tf.push_back(SymvTask{f.G, f.ld, g.xb + o, nullptr, g.zb + o, f.m, 1.0, g.idx + o, 1});
        tb.push_back(SymvTask{f.G, f.ld, g.acc + o, g.xb + o, g.zb + o, f.m, -1.0, g.idx + o, 0});
        tf.back().L = tb.back().L = f.L;
        tf.back().X = tb.back().X = f.inv;
        g.sym_maxm = std::max(g.sym_maxm, f.m);
        g.bytes_sym += 4.0 * f.m * (f.m + 1.0);
        o += f.m;
      }
      g.sym = true;
      g.nsym = (int)tf.size();
      g.sym_f = plan->mem.upload(tf);
      g.sym_b = plan->mem.upload(tb);
    }
    g.nidx = plan->mem.upload(nidx);
    g.bytes_f1 = gemv_bytes(f1, 0);
    g.bytes_f2 = gemv_bytes(f2, 0);
    {
      long long r1n = 0, r2n = 0;
      for (size_t i = rg.first; i < rg.second; ++i) {
        r1n += fs[i]->m;
        r2n += fs[i]->c;
      }
      if (r1n) g.lpr1 = lanes_for(g.bytes_f1 / 16.0 / r1n);
      for (auto& t : f1)  // row pairs: the 32-lane kernel, or the bulk one for long pairs (2x the mean row)
        if (t.tri == 2) g.lpr1 = (r1n && lanes_for(2.0 * g.bytes_f1 / 16.0 / r1n) == 64) ? 64 : 32;
      if (r2n) g.lpr2 = lanes_for(g.bytes_f2 / 16.0 / r2n);
    }
    g.bytes_b1 = gemv_bytes(b1, 1);
    {  // (masked L^{-1} tasks run over the square; their dense work is the triangle)
      std::vector<GemvTask> tb(b2);
      for (auto& t : tb)
        if (t.rmask) t.tri = 1;
      g.bytes_b2 = gemv_bytes(tb, 1);
    }
    {  // masked triangular rows grow with the row index: longest tasks first, so the launch does not end on a
       // few CTAs holding the longest rows (tasks write disjoint rows: their order is free)
      bool masked_tri = !f1.empty();
      for (const auto& t : f1) masked_tri = masked_tri && t.rmask && t.tri == 1;
      if (masked_tri)
        std::stable_sort(f1.begin(), f1.end(), [](const GemvTask& a, const GemvTask& b) { return a.r1 > b.r1; });
    }
    g.fwd1 = plan->mem.upload(f1);
    g.nf1 = (int)f1.size();
    g.fwd2 = plan->mem.upload(f2);
    g.nf2 = (int)f2.size();
    g.bwd1 = plan->mem.upload(b1);
    g.nb1 = (int)b1.size();
    {
      bool lead = !b1.empty();
      for (const auto& t : b1) lead = lead && (t.kfirst || t.rmask) && t.r1 - t.r0 <= GT_ROWS;
      g.b1_mode = lead ? 2 : 1;
      bool sp = !f2.empty();
      for (const auto& t : f2) sp = sp && (t.kfirst || t.rmask);
      g.f2_mode = sp ? 3 : 0;
      bool s1 = !f1.empty(), s2 = !b2.empty();
      for (const auto& t : f1) s1 = s1 && t.rmask;
      for (const auto& t : b2) s2 = s2 && t.rmask && t.r1 - t.r0 <= GT_ROWS;
      g.f1_mode = s1 ? 3 : 0;
      g.b2_mode = s2 ? 2 : 1;
      if (s1) g.lpr1 = 64;  // the bulk-copy kernel with dynamic rows
    }
    g.bwd2 = plan->mem.upload(b2);
    g.nb2 = (int)b2.size();
    // the group's final reduction scatters straight into the full vector
    // (backward_group): its segments carry the nodes' index arrays
    for (auto& r : (g.type == SGF_FACTOR_ELIMINATION ? r2 : r1)) r.idx = g.idx + (r.out - g.zb);
    g.red1 = plan->mem.upload(r1);
    g.nred1 = (int)r1.size();
    g.red2 = plan->mem.upload(r2);
    g.nred2 = (int)r2.size();
    if (!contrib.empty()) {
      // bucket the contributions per target unknown, keeping factor order
      // inside a bucket (counting sort; tix is an n-sized scratch map).  The
      // passes are bound by random accesses into tix and the fill cursors, so
      // large levels split the unknowns into ranges, one host thread each: a
      // thread scans every contribution and handles those of its range (its
      // slice of tix stays in cache).  The order of the targets differs from
      // the serial one; the order inside a target -- the summation order of
      // combine_kernel -- does not.
      const int nth = contrib.size() > 400000 ? 4 : 1;
      const int64_t n_all = (int64_t)tix.size();
      struct Part {
        std::vector<int> tgt;
        std::vector<long long> ptr;  // counts, then offsets inside the part
        long long total = 0;
      };
      std::vector<Part> parts(nth);
      std::vector<long long> pos(contrib.size());
      auto range = [&](int t) { return std::make_pair(n_all * t / nth, n_all * (t + 1) / nth); };
      auto count_pass = [&](int t) {
        Part& pt = parts[t];
        const auto [lo, hi] = range(t);
        for (auto& c : contrib) {
          if (c.first < lo || c.first >= hi) continue;
          int& ti = tix[c.first];
          if (ti < 0) {
            ti = (int)pt.tgt.size();
            pt.tgt.push_back((int)c.first);
            pt.ptr.push_back(0);
          }
          ++pt.ptr[ti];
        }
        long long run = 0;
        for (auto& p : pt.ptr) {
          const long long k = p;
          p = run;
          run += k;
        }
        pt.total = run;
      };
      auto fill_pass = [&](int t, long long base) {
        Part& pt = parts[t];
        const auto [lo, hi] = range(t);
        std::vector<long long> fillp(pt.ptr);
        for (auto& c : contrib)
          if (c.first >= lo && c.first < hi) pos[base + fillp[tix[c.first]]++] = c.second;
        for (int u : pt.tgt) tix[u] = -1;
      };
      auto run_all = [&](auto&& fn) {
        std::vector<std::thread> th;
        for (int t = 1; t < nth; ++t) th.emplace_back(fn, t);
        fn(0);
        for (auto& x : th) x.join();
      };
      run_all(count_pass);
      std::vector<long long> base(nth + 1, 0);
      for (int t = 0; t < nth; ++t) base[t + 1] = base[t] + parts[t].total;
      run_all([&](int t) { fill_pass(t, base[t]); });
      std::vector<int> tgt;
      std::vector<long long> ptr;
      for (int t = 0; t < nth; ++t) {
        tgt.insert(tgt.end(), parts[t].tgt.begin(), parts[t].tgt.end());
        for (long long p : parts[t].ptr) ptr.push_back(base[t] + p);
      }
      ptr.push_back(base[nth]);
      g.ntgt = (long long)tgt.size();
      g.tgt = plan->mem.upload(tgt);
      g.tptr = plan->mem.upload(ptr);
      g.tpos = plan->mem.upload(pos);
    }
    plan->groups.push_back(g);
  }
}

// The context stream waits for everything enqueued so far on the upload
// stream: the plan's task lists are in place before a sweep reads them.
static void plan_sync_uploads(Precond* P) {
  Ctx* c = P->ctx;
  SGF_CUDA(cudaEventRecord(c->upload_ev, c->upload_stream));
  SGF_CUDA(cudaStreamWaitEvent(c->stream, c->upload_ev, 0));
}

ApplyPlan* build_plan(Precond* P) {
  plan_extend(P, 0, P->factors.size());
  plan_sync_uploads(P);
  return P->plan;
}

void plan_finish(Precond* P) {
  if (!P->plan) return;
  std::vector<int>().swap(P->plan->tix);
  plan_sync_uploads(P);
}

static void gemv(const GemvTask* t, int nt, int mode, double bytes, cudaStream_t st, int lpr = 32) {
  ProfScope ps(st, PROF_GEMV, bytes);
  SGF_CUDA(launch_gemv(t, nt, mode, st, lpr));
}

// level-1 group of apply_inverse: v = G x_B, x_N -= A_NB v (forward, v kept
// in x_B); y_B = v - G A_NB^T x_N (backward).  Equal to the reference's
// L^{-1} / E = A_NB L^{-T} sweeps since E^T = L^{-1} A_NB^T and G = L^{-T} L^{-1}.
static void symv(const SymvTask* t, int nt, int maxm, double bytes, cudaStream_t st) {
  ProfScope ps(st, PROF_GEMV, bytes);
  SGF_CUDA(launch_symv(t, nt, maxm, st));
}

// with the fused symv, the gather of x_B and the scatter of the result go
// through the nodes' index arrays inside the kernel (two launches fewer per sweep)
static void forward_group_sym(const L1Couplings& c, const Group& g, double* y, cudaStream_t st) {
  if (g.band) {
    ProfScope ps(st, PROF_GEMV, g.bytes_band);
    SGF_CUDA(launch_l1_band(g.sym_f, g.nsym, y, st));
  } else if (symv_fused_ok(g.sym_maxm)) {
    ProfScope ps(st, PROF_GEMV, g.bytes_sym);
    SGF_CUDA(launch_symv_fused(g.sym_f, g.nsym, g.sym_maxm, y, st));
  } else {
    SGF_CUDA(launch_gather(y, g.idx, g.xb, g.nm, st));
    symv(g.sym_f, g.nsym, g.sym_maxm, g.bytes_sym, st);
    SGF_CUDA(launch_scatter(g.zb, g.idx, y, g.nm, st));
  }
  SGF_CUDA(launch_sub_spmv(c.nf, c.f_rid, c.f_rp, c.f_ci, c.f_v, y, nullptr, 0, st));
}

static void backward_group_sym(const L1Couplings& c, const Group& g, double* y, cudaStream_t st) {
  SGF_CUDA(launch_sub_spmv(c.nb, nullptr, c.b_rp, c.b_ci, c.b_v, y, g.acc, 1, st));
  if (g.band) {
    ProfScope ps(st, PROF_GEMV, g.bytes_band);
    SGF_CUDA(launch_l1_band(g.sym_b, g.nsym, y, st));
  } else if (symv_fused_ok(g.sym_maxm)) {
    ProfScope ps(st, PROF_GEMV, g.bytes_sym);
    SGF_CUDA(launch_symv_fused(g.sym_b, g.nsym, g.sym_maxm, y, st));
  } else {
    SGF_CUDA(launch_gather(y, g.idx, g.xb, g.nm, st));
    symv(g.sym_b, g.nsym, g.sym_maxm, g.bytes_sym, st);
    SGF_CUDA(launch_scatter(g.zb, g.idx, y, g.nm, st));
  }
}

static void forward_group(ApplyPlan* pl, const Group& g, double* y, cudaStream_t st) {
  (void)pl;
  SGF_CUDA(launch_gather(y, g.idx, g.xb, g.nm, st));
  gemv(g.fwd1, g.nf1, g.f1_mode, g.bytes_f1, st, g.lpr1);
  if (g.type == SGF_FACTOR_ELIMINATION) gemv(g.fwd2, g.nf2, g.f2_mode, g.bytes_f2, st, g.lpr2);
  SGF_CUDA(launch_scatter(g.zb, g.idx, y, g.nm, st));
  if (g.type == SGF_FACTOR_ELIMINATION) SGF_CUDA(launch_combine(y, g.tgt, g.tptr, g.tpos, g.t, g.ntgt, st));
}

static void backward_group(ApplyPlan* pl, const Group& g, double* y, cudaStream_t st) {
  (void)pl;
  SGF_CUDA(launch_gather(y, g.idx, g.xb, g.nm, st));
  if (g.type == SGF_FACTOR_ELIMINATION) {
    SGF_CUDA(launch_gather(y, g.nidx, g.xn, g.nc, st));
    gemv(g.bwd1, g.nb1, g.b1_mode, g.bytes_b1, st);
    SGF_CUDA(launch_reduce_parts(g.red1, g.nred1, g.maxn1, st));
    gemv(g.bwd2, g.nb2, g.b2_mode, g.bytes_b2, st);
    SGF_CUDA(launch_reduce_parts(g.red2, g.nred2, g.maxn2, st, y));  // + scatter into y
  } else {
    gemv(g.bwd1, g.nb1, g.b1_mode, g.bytes_b1, st);
    SGF_CUDA(launch_reduce_parts(g.red1, g.nred1, g.maxn1, st, y));  // + scatter into y
  }
}

// y and x are device n-vectors; y may alias x
static void fwd(ApplyPlan* pl, const L1Couplings& c, const Group& g, bool full, double* y, cudaStream_t st) {
  if (full && g.sym) forward_group_sym(c, g, y, st);
  else forward_group(pl, g, y, st);
}
static void bwd(ApplyPlan* pl, const L1Couplings& c, const Group& g, bool full, double* y, cudaStream_t st) {
  if (full && g.sym) backward_group_sym(c, g, y, st);
  else backward_group(pl, g, y, st);
}

// `full`: both sweeps of apply_inverse run, so level-1 groups may use the
// G form (its intermediate x_B differs from the L^{-1} half sweep's)
static void sweeps(ApplyPlan* pl, const L1Couplings& c, int op, double* y, cudaStream_t st) {
  const bool full = op == SGF_APPLY_INVERSE;
  if (op == SGF_APPLY_INVERSE || op == SGF_APPLY_HALF_INVERSE)
    for (auto& g : pl->groups) fwd(pl, c, g, full, y, st);
  if (op == SGF_APPLY_INVERSE || op == SGF_APPLY_HALF_INVERSE_T)
    for (auto it = pl->groups.rbegin(); it != pl->groups.rend(); ++it) bwd(pl, c, *it, full, y, st);
}

// ---------------------------------------------------------------------------
// apply_operator = W W^T x (reference factorization.py:264-271): the
// mult_transpose sweep over the factors in order, then mult_forward in
// reverse (:144-148, 179-183, 205-209).  Compression factors need L Q, formed
// once on first use as L - (L V) T V^T.
// ---------------------------------------------------------------------------
static void prepare_operator(Precond* P) {
  ApplyPlan* pl = P->plan;
  if (pl->op_ready) return;
  cudaStream_t st = P->ctx->stream;
  Arena scratch(st);
  GemmBatch g1, g2, g3;
  CopyBatch cp;
  for (auto& f : P->factors) {
    if (f.type != SGF_FACTOR_COMPRESSION) continue;
    const int m = f.m, s = f.steps;
    f.LQ = P->store.alloc((size_t)m * f.ld);
    cp.add(f.L, f.ld, 1, f.LQ, f.ld, 1, m, m);
    if (!s) continue;
    double* P1 = scratch.alloc((size_t)m * s);
    double* P2 = scratch.alloc((size_t)m * s);
    g1.add(P1, s, 1, m, s, 1.0, 0.0, {seg(f.L, f.ld, 1, f.V, m, 1, m, SEG_KLIM_M)});
    g2.add(P2, s, 1, m, s, 1.0, 0.0, {seg(P1, s, 1, f.Tw, 1, s, s, SEG_KLIM_N)});  // T upper
    g3.add(f.LQ, f.ld, 1, m, m, -1.0, 1.0, {seg(P2, s, 1, f.V, 1, m, s)});
  }
  cp.launch(scratch, st);
  g1.launch(scratch, st);
  g2.launch(scratch, st);
  g3.launch(scratch, st);
  for (auto& g : pl->groups) {
    std::vector<GemvTask> t1, te, tl;
    std::vector<RedSeg> rr;
    long long om = 0, oc = 0, op = 0;
    for (size_t i = g.f0; i < g.f1; ++i) {
      const Factor& f = P->factors[i];
      const double* M = (f.type == SGF_FACTOR_COMPRESSION) ? f.LQ : f.L;
      const int tri = (f.type != SGF_FACTOR_COMPRESSION);
      // transpose pass: [L^T | (LQ)^T] x_B (+ E^T x_N), partial row blocks stacked
      int nrb = add_gemv_t(t1, M, f.ld, g.xb + om, g.part + op, f.m, f.m, tri, g.gt_rows);
      if (f.type == SGF_FACTOR_ELIMINATION && f.c > 0)
        nrb += add_gemv_t(t1, f.E, f.ld, g.xn + oc, g.part + op + (long long)nrb * f.m, f.c, f.m, 0, g.gt_rows);
      rr.push_back(RedSeg{g.part + op, nullptr, g.zb + om, f.m, nrb, f.m, 1.0});
      op += (long long)nrb * f.m;
      // forward pass: x_N += E x_B, x_B = [L | LQ] x_B
      if (f.type == SGF_FACTOR_ELIMINATION && f.c > 0)
        add_gemv_n(te, f.E, f.ld, g.xb + om, g.t + oc, f.c, f.m, 0, g.gn_rows);
      add_gemv_n(tl, M, f.ld, g.xb + om, g.zb + om, f.m, f.m, tri, g.gn_rows);
      om += f.m;
      oc += f.c;
    }
    g.oT = pl->mem.upload(t1);
    g.noT = (int)t1.size();
    g.oRed = pl->mem.upload(rr);
    g.noRed = (int)rr.size();
    g.oE = pl->mem.upload(te);
    g.noE = (int)te.size();
    g.oL = pl->mem.upload(tl);
    g.noL = (int)tl.size();
    g.bytes_oT = gemv_bytes(t1, 1);
    g.bytes_oE = gemv_bytes(te, 0);
    g.bytes_oL = gemv_bytes(tl, 0);
  }
  plan_sync_uploads(P);
  SGF_CUDA(cudaStreamSynchronize(st));
  pl->op_ready = true;
}

static void operator_sweeps(ApplyPlan* pl, double* y, cudaStream_t st) {
  for (auto& g : pl->groups) {  // mult_transpose, factor order
    SGF_CUDA(launch_gather(y, g.idx, g.xb, g.nm, st));
    if (g.type == SGF_FACTOR_ELIMINATION) SGF_CUDA(launch_gather(y, g.nidx, g.xn, g.nc, st));
    gemv(g.oT, g.noT, 1, g.bytes_oT, st);
    SGF_CUDA(launch_reduce_parts(g.oRed, g.noRed, g.maxn1, st));
    SGF_CUDA(launch_scatter(g.zb, g.idx, y, g.nm, st));
  }
  for (auto it = pl->groups.rbegin(); it != pl->groups.rend(); ++it) {  // mult_forward, reverse order
    const Group& g = *it;
    SGF_CUDA(launch_gather(y, g.idx, g.xb, g.nm, st));
    if (g.type == SGF_FACTOR_ELIMINATION) {
      gemv(g.oE, g.noE, 0, g.bytes_oE, st);
      SGF_CUDA(launch_combine(y, g.tgt, g.tptr, g.tpos, g.t, g.ntgt, st, 1));
    }
    gemv(g.oL, g.noL, 0, g.bytes_oL, st);
    SGF_CUDA(launch_scatter(g.zb, g.idx, y, g.nm, st));
  }
}

void apply_op(Precond* P, int op, const double* d_x, double* d_y) {
  cudaStream_t st = P->ctx->stream;
  ApplyPlan* pl = P->plan;
  if (op < 0 || op > 3) fail(SGF_INVALID_ARG, "unknown apply operation");
  if (P->sharded) fail(SGF_INVALID_ARG, "sharded preconditioner: apply through the collective sharded apply");
  if (op != SGF_APPLY_INVERSE) materialize_l1_e(P);  // the L^{-1}/E form reads the level-1 couplings
  if (op == SGF_APPLY_OPERATOR) {
    prepare_operator(P);
    if (d_y != d_x) SGF_CUDA(cudaMemcpyAsync(d_y, d_x, P->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    operator_sweeps(pl, d_y, st);
    return;
  }
  static const bool no_graph = getenv("SGF_NO_GRAPH") != nullptr;
  if (g_prof.on || no_graph) {  // per-kernel timing needs eager launches
    if (d_y != d_x) SGF_CUDA(cudaMemcpyAsync(d_y, d_x, P->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    sweeps(pl, P->l1, op, d_y, st);
    return;
  }
  // the whole sweep sequence (~100 launches) replays as one CUDA graph on
  // the plan's work vector
  if (!pl->graph[op]) {
    cudaGraph_t g;
    SGF_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const unsigned long long before = g_kernel_launches;
    sweeps(pl, P->l1, op, pl->work, st);
    SGF_CUDA(cudaStreamEndCapture(st, &g));
    pl->graph_launches[op] = g_kernel_launches - before;
    SGF_CUDA(cudaGraphInstantiate(&pl->graph[op], g, 0));
    cudaGraphDestroy(g);
  }
  SGF_CUDA(cudaMemcpyAsync(pl->work, d_x, P->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  SGF_CUDA(cudaGraphLaunch(pl->graph[op], st));
  count_launch(pl->graph_launches[op]);
  SGF_CUDA(cudaMemcpyAsync(d_y, pl->work, P->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
}

// Partial sweeps in place (the sharded apply, sharded.py): groups never
// straddle the local/top boundary because the plan is extended per level.
void apply_part(Precond* P, int part, double* y) {
  if (part < 0 || part > 2) fail(SGF_INVALID_ARG, "unknown apply part");
  cudaStream_t st = P->ctx->stream;
  ApplyPlan* pl = P->plan;
  const size_t nl = P->local_count();
  const L1Couplings& c = P->l1;
  if (part == 0) {
    for (auto& g : pl->groups)
      if (g.f1 <= nl) fwd(pl, c, g, true, y, st);
  } else if (part == 1) {
    for (auto& g : pl->groups)
      if (g.f0 >= nl) fwd(pl, c, g, true, y, st);
    for (auto it = pl->groups.rbegin(); it != pl->groups.rend(); ++it)
      if (it->f0 >= nl) bwd(pl, c, *it, true, y, st);
  } else {
    for (auto it = pl->groups.rbegin(); it != pl->groups.rend(); ++it)
      if (it->f1 <= nl) bwd(pl, c, *it, true, y, st);
  }
}

// The sharded apply_inverse on distributed vectors (sgf_apply_shard): the
// local sweeps, the top unknowns' exchange buffer and the ownership mask as
// native steps, so the caller only runs the collectives on top_buf.
void apply_shard(Precond* P, int stage, const double* x, double* y, double* top_buf, int mask) {
  cudaStream_t st = P->ctx->stream;
  const long long n = P->n, nt = (long long)P->top_idx.size();
  if (!P->d_top) {
    std::vector<int> t(P->top_idx.begin(), P->top_idx.end());
    std::vector<unsigned char> own(n, 0);
    for (size_t i = 0; i < P->local_count(); ++i)
      for (int64_t u : P->factors[i].idx) own[u] = 1;
    if (P->shard_rank == 0)
      for (int64_t u : P->top_idx) own[u] = 1;
    P->d_top = P->store.alloc_t<int>(std::max<long long>(nt, 1));
    P->d_owned = P->store.alloc_t<unsigned char>(std::max<long long>(n, 1));
    if (nt) SGF_CUDA(cudaMemcpyAsync(P->d_top, t.data(), nt * sizeof(int), cudaMemcpyHostToDevice, st));
    SGF_CUDA(cudaMemcpyAsync(P->d_owned, own.data(), n, cudaMemcpyHostToDevice, st));
    SGF_CUDA(cudaStreamSynchronize(st));
  }
  if (stage == 0) {
    if (y != x) SGF_CUDA(cudaMemcpyAsync(y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    apply_part(P, 0, y);
    SGF_CUDA(launch_gather_diff(y, x, P->d_top, top_buf, nt, st));
  } else if (stage == 1) {
    SGF_CUDA(launch_scatter_base(y, x, P->d_top, top_buf, nt, st));
    apply_part(P, 1, y);
    SGF_CUDA(launch_gather(y, P->d_top, top_buf, nt, st));
  } else if (stage == 2) {
    SGF_CUDA(launch_scatter_base(y, nullptr, P->d_top, top_buf, nt, st));
    apply_part(P, 2, y);
    if (mask) SGF_CUDA(launch_mask(y, P->d_owned, n, st));
  } else {
    fail(SGF_INVALID_ARG, "unknown apply stage");
  }
}

// ---------------------------------------------------------------------------
void spmv(Csr* A, const double* d_x, double* d_y, const double* d_b) {
  // values + int32 columns + row pointers + x + y (+ b)
  ProfScope ps(A->ctx->stream, PROF_SPMV,
               12.0 * A->nnz + (A->rp32 ? 4.0 : 8.0) * (A->n + 1) + (d_b ? 24.0 : 16.0) * A->n);
  SGF_CUDA(launch_spmv((int)A->n, A->rp, A->rp32, A->ci, A->v, d_x, d_y, d_b, A->ctx->stream));
}

// PCG with the reference recurrence (krylov.py:34-102): true-residual
// replacement every `true_every` iterations, confirmation of a tentative
// convergence with the true residual, history semantics identical.
void pcg(Ctx& ctx, Csr* A, const MatFn& Aop, const PrecFn& M, const double* d_b, double* d_x, double tol, int maxit,
         int true_every, sgf_pcg_report* rep, double* history) {
  cudaStream_t st = ctx.stream;
  const long long n = A->n;
  auto t0 = std::chrono::steady_clock::now();
  // workspace held by the matrix (allocated on its first solve): a solve
  // allocates nothing, so it never waits in cudaMalloc / cudaFreeHost
  const long long np = (n + 31) & ~31LL;  // 256-byte aligned vectors
  if (!A->ws) {
    A->ws = A->mem.alloc(4 * np + PCG_PART + 8);
    SGF_CUDA(cudaMallocHost((void**)&A->hsc, 8 * sizeof(double)));
  }
  double* r = A->ws;
  double* z = r + np;
  double* p = z + np;
  double* q = p + np;
  double* part = q + np;
  double* sc = part + PCG_PART;  // 0 / 2: r'z of this and of the next direction (alternating), 1 pAp, 3 rr, 4 bb
  SGF_CUDA(cudaMemsetAsync(part + PCG_CNT_OFF, 0, 2 * sizeof(double), st));  // the reductions' arrival counter
  double* hsc = A->hsc;
  // SGF_TRACE=5: host time spent waiting in each readback vs. issuing work
  static const bool trace5 = getenv("SGF_TRACE") && atoi(getenv("SGF_TRACE")) == 5;
  double t_wait = 0.0, t_issue = 0.0;
  auto tlast = std::chrono::steady_clock::now();
  auto readback = [&](int lo, int cnt) {
    SGF_CUDA(cudaMemcpyAsync(hsc + lo, sc + lo, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (trace5) {
      auto t1 = std::chrono::steady_clock::now();
      t_issue += std::chrono::duration<double, std::milli>(t1 - tlast).count();
      SGF_CUDA(cudaStreamSynchronize(st));
      tlast = std::chrono::steady_clock::now();
      t_wait += std::chrono::duration<double, std::milli>(tlast - t1).count();
    } else {
      SGF_CUDA(cudaStreamSynchronize(st));
    }
  };
  // out = A in, or out = b - A in when b is given
  auto matvec = [&](const double* in, double* out, const double* b) {
    if (Aop) {
      Aop(in, out);
      if (b) SGF_CUDA(launch_residual(b, out, n, st));
    } else {
      spmv(A, in, out, b);
    }
  };
  // q = A p and sc[1] = p'q: one launch for the device CSR (the SpMV kernel adds p[row] q[row] as it goes)
  auto matvec_dot = [&](const double* in, double* out) {
    if (Aop) {
      Aop(in, out);
      SGF_CUDA(launch_dot(in, out, n, part, sc, 1, st));
    } else {
      ProfScope ps(A->ctx->stream, PROF_SPMV, 12.0 * A->nnz + (A->rp32 ? 4.0 : 8.0) * (A->n + 1) + 16.0 * A->n);
      SGF_CUDA(launch_spmv_dot((int)A->n, A->rp, A->rp32, A->ci, A->v, in, out, part, sc, 1, A->ctx->stream));
    }
  };
  auto precond = [&](const double* in, double* out) {
    if (M) M(in, out);
    else SGF_CUDA(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  };
  int hl = 0;
  SGF_CUDA(launch_dot(d_b, d_b, n, part, sc, 4, st));
  readback(4, 1);
  const double bnorm = std::sqrt(hsc[4]);
  SGF_CUDA(cudaMemsetAsync(d_x, 0, n * sizeof(double), st));
  if (bnorm == 0.0) {
    history[hl++] = 0.0;
    rep->iterations = 0;
    rep->converged = 1;
    rep->final_rel_residual = 0.0;
    rep->history_len = hl;
    SGF_CUDA(cudaStreamSynchronize(st));
    rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return;
  }
  SGF_CUDA(cudaMemcpyAsync(r, d_b, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  history[hl++] = 1.0;
  precond(r, z);
  SGF_CUDA(launch_dot(r, z, n, part, sc, 0, st));
  readback(0, 1);
  if (hsc[0] <= 0.0) {
    char buf[96];
    snprintf(buf, sizeof buf, "initial r'Mr = %.3e is not positive", hsc[0]);
    fail(SGF_INDEFINITE, buf);
  }
  SGF_CUDA(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  bool converged = false;
  int it = 0;
  int rz = 0;  // slot of the current r'z; the next one goes to the other of {0, 2} (no scalar copy)
  while (it < maxit) {
    ++it;
    matvec_dot(p, q);
    SGF_CUDA(launch_xr_update(d_x, r, p, q, n, sc, part, sc, 3, st, rz));
    if (true_every > 0 && it % true_every == 0) {
      matvec(d_x, r, d_b);
      SGF_CUDA(launch_dot(r, r, n, part, sc, 3, st));
    }
    readback(1, 3);
    if (hsc[1] <= 0.0) {
      char buf[96];
      snprintf(buf, sizeof buf, "p'Ap = %.3e at iteration %d", hsc[1], it);
      fail(SGF_INDEFINITE, buf);
    }
    double rel = std::sqrt(hsc[3]) / bnorm;
    if (rel <= tol) {
      matvec(d_x, r, d_b);
      SGF_CUDA(launch_dot(r, r, n, part, sc, 3, st));
      readback(3, 1);
      rel = std::sqrt(hsc[3]) / bnorm;
      history[hl++] = rel;
      if (rel <= tol) {
        converged = true;
        break;
      }
    } else {
      history[hl++] = rel;
    }
    precond(r, z);
    const int rz_new = 2 - rz;
    SGF_CUDA(launch_dot(r, z, n, part, sc, rz_new, st));
    readback(rz_new, 1);
    if (hsc[rz_new] <= 0.0) {
      char buf[96];
      snprintf(buf, sizeof buf, "r'Mr = %.3e at iteration %d", hsc[rz_new], it);
      fail(SGF_INDEFINITE, buf);
    }
    SGF_CUDA(launch_p_update(p, z, n, sc, st, rz_new, rz));
    rz = rz_new;
  }
  matvec(d_x, r, d_b);
  SGF_CUDA(launch_dot(r, r, n, part, sc, 3, st));
  readback(3, 1);
  const double fin = std::sqrt(hsc[3]) / bnorm;
  if (trace5) fprintf(stderr, "[pcg] %d iterations: host issue %.2f ms, waiting %.2f ms\n", it, t_issue, t_wait);
  rep->iterations = it;
  rep->converged = (converged && fin <= tol) ? 1 : 0;
  rep->final_rel_residual = fin;
  rep->history_len = hl;
  rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Distributed PCG (the sharded solve, sgf_pcg_dist): the reference recurrence
// (krylov.py:34-102) on vectors holding this rank's owned entries.  Every
// inner product is a local partial (non-owned entries are zero) summed across
// the ranks by the caller's `reduce` before anything uses it, so the scalars
// -- and every branch -- are identical on all ranks.  A's owned rows come
// from the caller's operator (halo exchange + row-block SpMV), M^-1 from the
// sharded apply.
void pcg_dist(Ctx& ctx, int64_t n, const MatFn& Aop, const PrecFn& M, const ReduceFn& reduce, const double* d_b,
              double* d_x, double tol, int maxit, int true_every, sgf_pcg_report* rep, double* history) {
  cudaStream_t st = ctx.stream;
  auto t0 = std::chrono::steady_clock::now();
  Arena ws(st);
  const long long np = (n + 31) & ~31LL;
  double* r = ws.alloc(4 * np + PCG_PART + 8);
  double* z = r + np;
  double* p = z + np;
  double* q = p + np;
  double* part = q + np;
  double* sc = part + PCG_PART;  // 0 rz, 1 pAp, 2 rz_new, 3 rr, 4 bb
  SGF_CUDA(cudaMemsetAsync(part + PCG_CNT_OFF, 0, 2 * sizeof(double), st));  // the reductions' arrival counter
  double* hsc = nullptr;
  SGF_CUDA(cudaMallocHost((void**)&hsc, 8 * sizeof(double)));
  struct Pin {
    double* p;
    ~Pin() { cudaFreeHost(p); }
  } pin{hsc};
  // device scalar -> host, summed over the ranks, written back for the kernels
  auto global = [&](int slot) {
    SGF_CUDA(cudaMemcpyAsync(hsc + slot, sc + slot, sizeof(double), cudaMemcpyDeviceToHost, st));
    SGF_CUDA(cudaStreamSynchronize(st));
    reduce(hsc + slot, 1);
    SGF_CUDA(cudaMemcpyAsync(sc + slot, hsc + slot, sizeof(double), cudaMemcpyHostToDevice, st));
    return hsc[slot];
  };
  auto residual = [&]() {  // r = b - A x
    Aop(d_x, r);
    SGF_CUDA(launch_residual(d_b, r, n, st));
  };
  int hl = 0;
  SGF_CUDA(launch_dot(d_b, d_b, n, part, sc, 4, st));
  const double bnorm = std::sqrt(global(4));
  SGF_CUDA(cudaMemsetAsync(d_x, 0, n * sizeof(double), st));
  if (bnorm == 0.0) {
    history[hl++] = 0.0;
    rep->iterations = 0;
    rep->converged = 1;
    rep->final_rel_residual = 0.0;
    rep->history_len = hl;
    SGF_CUDA(cudaStreamSynchronize(st));
    rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return;
  }
  SGF_CUDA(cudaMemcpyAsync(r, d_b, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  history[hl++] = 1.0;
  M(r, z);
  SGF_CUDA(launch_dot(r, z, n, part, sc, 0, st));
  if (global(0) <= 0.0) {
    char buf[96];
    snprintf(buf, sizeof buf, "initial r'Mr = %.3e is not positive", hsc[0]);
    fail(SGF_INDEFINITE, buf);
  }
  SGF_CUDA(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  bool converged = false;
  int it = 0;
  while (it < maxit) {
    ++it;
    Aop(p, q);
    SGF_CUDA(launch_dot(p, q, n, part, sc, 1, st));
    const double pAp = global(1);
    if (pAp <= 0.0) {
      char buf[96];
      snprintf(buf, sizeof buf, "p'Ap = %.3e at iteration %d", pAp, it);
      fail(SGF_INDEFINITE, buf);
    }
    SGF_CUDA(launch_xr_update(d_x, r, p, q, n, sc, part, sc, 3, st));
    if (true_every > 0 && it % true_every == 0) {
      residual();
      SGF_CUDA(launch_dot(r, r, n, part, sc, 3, st));
    }
    double rel = std::sqrt(global(3)) / bnorm;
    if (rel <= tol) {
      residual();
      SGF_CUDA(launch_dot(r, r, n, part, sc, 3, st));
      rel = std::sqrt(global(3)) / bnorm;
      history[hl++] = rel;
      if (rel <= tol) {
        converged = true;
        break;
      }
    } else {
      history[hl++] = rel;
    }
    M(r, z);
    SGF_CUDA(launch_dot(r, z, n, part, sc, 2, st));
    const double rz_new = global(2);
    if (rz_new <= 0.0) {
      char buf[96];
      snprintf(buf, sizeof buf, "r'Mr = %.3e at iteration %d", rz_new, it);
      fail(SGF_INDEFINITE, buf);
    }
    SGF_CUDA(launch_p_update(p, z, n, sc, st));
    SGF_CUDA(cudaMemcpyAsync(sc, sc + 2, sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  residual();
  SGF_CUDA(launch_dot(r, r, n, part, sc, 3, st));
  const double fin = std::sqrt(global(3)) / bnorm;
  rep->iterations = it;
  rep->converged = (converged && fin <= tol) ? 1 : 0;
  rep->final_rel_residual = fin;
  rep->history_len = hl;
  SGF_CUDA(cudaStreamSynchronize(st));
  rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace sgf
