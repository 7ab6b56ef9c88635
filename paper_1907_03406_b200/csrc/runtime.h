// Host runtime of the sgf library: context, device arenas, block table,
// batched-launch builders.  The factorization driver (factorize.cpp), the
// apply plan (apply.cpp) and the C ABI (capi.cpp) build on this.
#pragma once
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "common.h"
#include "sgf.h"

namespace sgf {

struct Error {
  int status;
  std::string msg;
};

[[noreturn]] void fail(int status, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define SGF_CUDA(x) ::sgf::cuda_check((x), #x)

// extra launchers (defined in .cu files, not in common.h)
cudaError_t launch_diag_chol_ex(const DiagTask* d_tasks, int ntasks, int* d_status, double* d_pivval,
                                double* const* d_xdiag, const int* d_ldx, cudaStream_t s);
cudaError_t launch_copy_tiled(const CopyTask* d_tasks, const long long* d_prefix, int ntasks, long long ntiles,
                              cudaStream_t s);
cudaError_t launch_zero_upper(const void* d_tasks, const long long* d_prefix, int ntasks, long long ntiles,
                              cudaStream_t s);
cudaError_t launch_qrcp(const QrTask* d_tasks, int ntasks, int max_m, cudaStream_t s, int max_c = 0);
cudaError_t launch_csr_scatter(const void* params, cudaStream_t s);
cudaError_t launch_sym_check(long long n, const long long* ip, const int* ix, const double* v,
                             unsigned long long* out, cudaStream_t s);
cudaError_t launch_qr_finish(const void* d_tasks, int ntasks, int phase, cudaStream_t s, int max_s = 0);
cudaError_t launch_reduce_parts(const void* d_segs, int nseg, int max_n, cudaStream_t s, double* v = nullptr);
cudaError_t launch_gather(const double* x, const int* idx, double* out, long long n, cudaStream_t s);
cudaError_t launch_scatter(const double* v, const int* idx, double* x, long long n, cudaStream_t s);
cudaError_t launch_combine(double* x, const int* tgt, const long long* ptr, const long long* pos, const double* t,
                           long long nt, cudaStream_t s, int add = 0);
cudaError_t launch_spmv(int n, const long long* rp, const int* rp32, const int* ci, const double* v, const double* x,
                        double* y, const double* b, cudaStream_t s);
cudaError_t launch_rowptr32(const long long* rp, int* out, long long n1, cudaStream_t s);
cudaError_t l1_couplings_count(long long n, int nb, const long long* ip, const int* ix, const int* owner,
                               const int* local, const char* el, const int* bstart, int* rows, int* bcnt, int* fcnt,
                               int* fflag, cudaStream_t s);
cudaError_t scan_ints(const int* in, int* out, long long count, void* temp, size_t* temp_bytes, cudaStream_t s);
cudaError_t l1_couplings_fill(long long n, const long long* ip, const int* ix, const double* vals, const int* owner,
                              const int* local, const char* el, const int* bstart, const int* brp, int* bci,
                              double* bv, const int* fscan, const int* fidx, int* frid, int* frp, int* fci,
                              double* fv, int nf, cudaStream_t s);
// PCG reductions: `part` holds PCG_PART doubles -- block partials and, at
// PCG_CNT_OFF, the arrival counter of the in-kernel final reduction, which
// must be zero before the first launch (it is reset by every launch)
cudaError_t launch_dot(const double* a, const double* b, long long n, double* part, double* out, int slot,
                       cudaStream_t s);
// x += alpha p, r -= alpha q, out[slot] = r'r with alpha = sc[rz] / sc[1]
cudaError_t launch_xr_update(double* x, double* r, const double* p, const double* q, long long n, const double* sc,
                             double* part, double* out, int slot, cudaStream_t s, int rz = 0);
// p = z + (sc[num] / sc[den]) p
cudaError_t launch_p_update(double* p, const double* z, long long n, const double* sc, cudaStream_t s, int num = 2,
                            int den = 0);
cudaError_t launch_spmv_dot(int n, const long long* rp, const int* rp32, const int* ci, const double* v,
                            const double* x, double* y, double* part, double* out, int slot, cudaStream_t s);
cudaError_t launch_residual(const double* b, double* out, long long n, cudaStream_t s);
// factor_ops.cu: small dense kernels of the per-factor methods and per-primitive entry points
cudaError_t launch_dmv(const double* M, long long ld, int rows, int inner, int trans, const double* v, double* y,
                       double alpha, double beta, cudaStream_t s);
cudaError_t launch_dense_check(const double* const* A, const int* m, const int* ld, int n, double* out, int* bad,
                               cudaStream_t s);
cudaError_t launch_form_q(const double* V, const double* tau, int m, int s, int qcols, double* Q, double* work,
                          cudaStream_t st);
cudaError_t launch_trsv(const double* L, long long ldl, int m, int nvec, const double* B, long long bvs,
                        long long bes, double* X, long long xvs, long long xes, int trans, cudaStream_t s);
cudaError_t launch_nonzero_flags(const double* const* ptrs, const long long* counts, int n, int* flags,
                                 cudaStream_t s);
cudaError_t launch_add_packed(double* const* dst, const long long* counts, const long long* offs, int n,
                              const double* packed, cudaStream_t s);
cudaError_t launch_gather_diff(const double* y, const double* x, const int* idx, double* out, long long n,
                               cudaStream_t s);
cudaError_t launch_scatter_base(double* y, const double* base, const int* idx, const double* d, long long n,
                                cudaStream_t s);
cudaError_t launch_mask(double* y, const unsigned char* owned, long long n, cudaStream_t s);


// ---------------------------------------------------------------------------
// Optional per-kernel-class timing with CUDA events on the launching stream
// (bench.py's roofline numbers).  Classes: see PROF_* below.
// ---------------------------------------------------------------------------
enum { PROF_GEMM = 0, PROF_GEMV = 1, PROF_SPMV = 2, PROF_QR = 3, PROF_CHOL = 4, PROF_MOVE = 5, PROF_VEC = 6,
       PROF_OZ = 7, PROF_OZSPLIT = 8, PROF_NCLS = 9 };
struct Profiler {
  bool on = false;
  struct Rec { int cls; cudaEvent_t a, b; double work; long long launches; };
  std::vector<Rec> recs;
  void reset();
  void read(double* out);  // out[3*cls + 0..2] = ms, work, launches
};
extern Profiler g_prof;
struct ProfScope {
  cudaStream_t s;
  int idx = -1;
  ProfScope(cudaStream_t st, int cls, double work);
  ~ProfScope();
};

// SGF_TRACE=4: host-side (no synchronisation) timing of a scope
struct HostTimer {
  const char* name;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit HostTimer(const char* n) : name(n) {}
  static bool on() {
    static bool v = getenv("SGF_TRACE") && atoi(getenv("SGF_TRACE")) == 4;
    return v;
  }
  static std::chrono::steady_clock::time_point& epoch() {  // reset by the factorization driver
    static std::chrono::steady_clock::time_point e = std::chrono::steady_clock::now();
    return e;
  }
  ~HostTimer() {
    if (on())
      fprintf(stderr, "[host] %-24s %8.2f ms  (from %.2f)\n", name,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
              std::chrono::duration<double, std::milli>(t0 - epoch()).count());
  }
};

// process-wide device chunk cache (runtime.cpp), per device
void* chunk_get(size_t bytes, size_t* cap);
void chunk_put(void* p, size_t cap);
void chunk_trim();
// Chunks of the apply plans' arenas.  The plan worker fills them through the
// context's upload stream while the main stream is still factorizing, so they
// cannot share the stream-ordered cache above: a released chunk carries an
// event recorded on the releasing stream (after its last users), and the
// stream of whoever takes it next waits for that event.
void* plan_chunk_get(size_t bytes, size_t* cap, cudaStream_t user);
void plan_chunk_put(void* p, size_t cap, cudaStream_t last_user);

// Asynchronous small host->device upload through a pinned staging ring (a
// cudaMemcpyAsync from pageable memory would synchronise the stream first
// and serialise host planning with device execution).  The ring is recycled
// with a stream synchronisation only when it is full.
void stage_upload(cudaStream_t st, void* dst, const void* src, size_t bytes);

// ---------------------------------------------------------------------------
// Device bump arena (chunks from the process-wide cache).
// ---------------------------------------------------------------------------
class Arena {
 public:
  explicit Arena(cudaStream_t s = nullptr, size_t chunk = (size_t)256 << 20) : s_(s), chunk_(chunk) {}
  ~Arena() { release(); }
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;
  void set_stream(cudaStream_t s) { s_ = s; }
  // chunks from the plan pool (plan_chunk_get/put): uploads run on s_, the
  // chunk's other users on `release_stream`
  void use_plan_pool(cudaStream_t release_stream) {
    plan_pool_ = true;
    rel_ = release_stream;
  }
  void* alloc_bytes(size_t bytes);
  double* alloc(size_t n) { return (double*)alloc_bytes(n * sizeof(double)); }
  template <class T>
  T* alloc_t(size_t n) { return (T*)alloc_bytes(n * sizeof(T)); }
  template <class T>
  T* upload(const std::vector<T>& v) {
    if (v.empty()) return nullptr;
    T* d = alloc_t<T>(v.size());
    stage_upload(s_, d, v.data(), v.size() * sizeof(T));
    return d;
  }
  void release();
  size_t used() const { return used_; }

 private:
  struct Chunk { char* base; size_t cap; size_t off; };
  cudaStream_t s_;
  size_t chunk_;
  std::vector<Chunk> chunks_;
  size_t used_ = 0;
  bool plan_pool_ = false;
  cudaStream_t rel_ = nullptr;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t order_ev = nullptr;  // sgf_stream_wait: orders the stream after a foreign one
  // uploads of the apply-plan worker: its own stream, so that its copies never
  // queue behind (or wait for a launch slot of) the factorization's backlog on
  // `stream`; `stream` waits for upload_ev before the plan is used (plan_sync_uploads)
  cudaStream_t upload_stream = nullptr;
  cudaEvent_t upload_ev = nullptr;
  std::string last_error;
  // grow-only pinned staging buffer for large host->device uploads; callers
  // synchronise the stream before reusing it
  void* pin = nullptr;
  size_t pin_cap = 0;
  void* pinned(size_t bytes) {
    if (bytes > pin_cap) {
      if (pin) {
        cudaStreamSynchronize(stream);  // copies may still read the old buffer
        cudaFreeHost(pin);
      }
      pin = nullptr;
      pin_cap = 0;
      SGF_CUDA(cudaMallocHost(&pin, bytes));
      pin_cap = bytes;
    }
    return pin;
  }
  ~Ctx() {
    if (pin) cudaFreeHost(pin);
  }
};
// copy n bytes host -> device through the context's pinned buffer (chunked,
// parallel host memcpy); synchronises the stream
void upload_pinned(Ctx& ctx, void* dst, const void* src, size_t bytes);

// ---------------------------------------------------------------------------
// Block table: symmetric block-sparse trailing matrix, blocks (a,b) a <= b,
// row-major rows = size[a], cols = size[b] (reference blockmatrix.py:14-83,
// including its live/peak byte accounting :25-43).
// ---------------------------------------------------------------------------
struct Blk {
  double* p;
  int rows, cols;
};

inline uint64_t bkey(int a, int b) {
  if (a > b) std::swap(a, b);
  return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
}

// Process-wide pool of host buffers for the hash maps below: a map of a
// level holds 10-20 MB, and fresh pages cost a fault each on first touch
// (~10 ms per level-1 table); buffers of a finished factorization are reused.
struct HostPool {
  std::mutex mu;
  std::multimap<size_t, void*> free;
  size_t bytes = 0;
  static constexpr size_t MAX = (size_t)2 << 30;
  static HostPool& get() {
    static HostPool* p = new HostPool;  // never destroyed: maps may outlive static destruction
    return *p;
  }
};
inline void* host_pool_get(size_t bytes) {
  HostPool& hp = HostPool::get();
  {
    std::lock_guard<std::mutex> lk(hp.mu);
    auto it = hp.free.find(bytes);
    if (it != hp.free.end()) {
      void* p = it->second;
      hp.free.erase(it);
      hp.bytes -= bytes;
      return p;
    }
  }
  void* p = std::malloc(bytes < 16 ? 16 : bytes);
  if (!p) throw std::bad_alloc();
  return p;
}
inline void host_pool_put(void* p, size_t bytes) {
  if (!p) return;
  HostPool& hp = HostPool::get();
  std::lock_guard<std::mutex> lk(hp.mu);
  if (hp.bytes + bytes > HostPool::MAX) {
    std::free(p);
    return;
  }
  hp.free.emplace(bytes, p);
  hp.bytes += bytes;
}

// Open-addressing hash map for 64-bit block keys (linear probing, backward-
// shift deletion): the symbolic phases do millions of lookups per level, where
// a node-based map's allocation and pointer chasing dominate.  Key ~0 is the
// empty marker (never a valid block key).  V must be trivially copyable.
template <class V>
class FlatMap {
 public:
  static constexpr uint64_t EMPTY = ~0ull;
  explicit FlatMap(size_t expect = 16) { reserve(expect); }
  FlatMap(const FlatMap&) = delete;
  FlatMap& operator=(const FlatMap&) = delete;
  FlatMap(FlatMap&& o) noexcept { steal(o); }
  FlatMap& operator=(FlatMap&& o) noexcept {
    if (this != &o) {
      release();
      steal(o);
    }
    return *this;
  }
  ~FlatMap() { release(); }
  size_t size() const { return n_; }
  void clear() {
    std::fill(keys_, keys_ + cap_, EMPTY);
    n_ = 0;
  }
  void reserve(size_t expect) {
    size_t cap = 16;
    while (cap < expect * 2) cap <<= 1;
    if (cap > cap_) rehash(cap);
  }
  V* find(uint64_t k) {
    size_t i = slot(k);
    for (;;) {
      if (keys_[i] == k) return &vals_[i];
      if (keys_[i] == EMPTY) return nullptr;
      i = (i + 1) & mask_;
    }
  }
  const V* find(uint64_t k) const { return const_cast<FlatMap*>(this)->find(k); }
  bool contains(uint64_t k) const { return find(k) != nullptr; }
  // the slot a key probes first (bulk inserts prefetch it ahead of use)
  void prefetch(uint64_t k) const {
    const size_t i = slot(k);
    __builtin_prefetch(keys_ + i, 1);
    __builtin_prefetch(vals_ + i, 1);
  }
  // returns the value slot and whether the key was new (value default-built)
  std::pair<V*, bool> emplace(uint64_t k) {
    if ((n_ + 1) * 2 > cap_) rehash(cap_ * 2);
    size_t i = slot(k);
    for (;;) {
      if (keys_[i] == k) return {&vals_[i], false};
      if (keys_[i] == EMPTY) {
        keys_[i] = k;
        vals_[i] = V();
        ++n_;
        return {&vals_[i], true};
      }
      i = (i + 1) & mask_;
    }
  }
  V& operator[](uint64_t k) { return *emplace(k).first; }
  bool erase(uint64_t k) {
    size_t i = slot(k);
    for (;;) {
      if (keys_[i] == EMPTY) return false;
      if (keys_[i] == k) break;
      i = (i + 1) & mask_;
    }
    // backward shift: pull later members of the probe run into the hole
    size_t j = i;
    for (;;) {
      j = (j + 1) & mask_;
      if (keys_[j] == EMPTY) break;
      const size_t h = slot(keys_[j]);
      const bool movable = (i <= j) ? (h <= i || h > j) : (h <= i && h > j);
      if (movable) {
        keys_[i] = keys_[j];
        vals_[i] = vals_[j];
        i = j;
      }
    }
    keys_[i] = EMPTY;
    --n_;
    return true;
  }
  template <class F>
  void for_each(F&& f) {
    for (size_t i = 0; i < cap_; ++i)
      if (keys_[i] != EMPTY) f(keys_[i], vals_[i]);
  }

 private:
  size_t slot(uint64_t k) const { return (size_t)((k * 0x9E3779B97F4A7C15ull) >> shift_); }
  void release() {
    if (keys_) host_pool_put(keys_, cap_ * sizeof(uint64_t));
    if (vals_) host_pool_put(vals_, cap_ * sizeof(V));
    keys_ = nullptr;
    vals_ = nullptr;
    cap_ = mask_ = n_ = 0;
  }
  void steal(FlatMap& o) {
    keys_ = o.keys_;
    vals_ = o.vals_;
    cap_ = o.cap_;
    mask_ = o.mask_;
    n_ = o.n_;
    shift_ = o.shift_;
    o.keys_ = nullptr;
    o.vals_ = nullptr;
    o.cap_ = o.mask_ = o.n_ = 0;
  }
  void rehash(size_t cap) {
    uint64_t* ok = keys_;
    V* ov = vals_;
    const size_t ocap = cap_;
    keys_ = (uint64_t*)host_pool_get(cap * sizeof(uint64_t));
    vals_ = (V*)host_pool_get(cap * sizeof(V));
    std::fill(keys_, keys_ + cap, EMPTY);
    cap_ = cap;
    mask_ = cap - 1;
    shift_ = 64;
    for (size_t c = cap; c > 1; c >>= 1) --shift_;
    n_ = 0;
    for (size_t i = 0; i < ocap; ++i)
      if (ok[i] != EMPTY) {
        size_t s = slot(ok[i]);
        while (keys_[s] != EMPTY) s = (s + 1) & mask_;
        keys_[s] = ok[i];
        vals_[s] = ov[i];
        ++n_;
      }
    if (ok) host_pool_put(ok, ocap * sizeof(uint64_t));
    if (ov) host_pool_put(ov, ocap * sizeof(V));
  }
  uint64_t* keys_ = nullptr;
  V* vals_ = nullptr;
  size_t cap_ = 0, mask_ = 0, n_ = 0;
  int shift_ = 64;
};

struct BlockTable {
  FlatMap<Blk> map;
  std::vector<std::vector<int>> adj;
  std::vector<int> size;
  long long live = 0, peak = 0;

  void init(const std::vector<int>& sizes) {
    size = sizes;
    adj.assign(sizes.size(), {});
    map.clear();
    map.reserve(sizes.size() * 8);
    live = peak = 0;
  }
  static long long nbytes(const Blk& b) { return 8LL * b.rows * b.cols; }
  Blk* find(int a, int b) { return map.find(bkey(a, b)); }
  void insert(int a, int b, Blk blk) {
    auto r = map.emplace(bkey(a, b));
    if (!r.second) live -= nbytes(*r.first);
    *r.first = blk;
    live += nbytes(blk);
    peak = std::max(peak, live);
    if (a != b) {
      add_adj(a, b);
      add_adj(b, a);
    }
  }
  // insert a block known to be new (setup: each pair appears once)
  void insert_new(int a, int b, Blk blk) {
    *map.emplace(bkey(a, b)).first = blk;
    live += nbytes(blk);
    peak = std::max(peak, live);
    if (a != b) {
      adj[a].push_back(b);
      adj[b].push_back(a);
    }
  }
  void add_adj(int a, int b) {
    auto& v = adj[a];
    if (std::find(v.begin(), v.end(), b) == v.end()) v.push_back(b);
  }
  void drop_key(uint64_t k) {
    if (Blk* p = map.find(k)) {
      live -= nbytes(*p);
      map.erase(k);
    }
  }
  void drop(int a) {
    for (int b : adj[a]) {
      drop_key(bkey(a, b));
      auto& v = adj[b];
      v.erase(std::remove(v.begin(), v.end(), a), v.end());
    }
    adj[a].clear();
    drop_key(bkey(a, a));
  }
  std::vector<int> nbrs(int a) const {
    std::vector<int> v = adj[a];
    std::sort(v.begin(), v.end());
    return v;
  }
};

// operand view of block (a,b) as the matrix with rows in a, cols in b
struct View {
  const double* p;
  long long rs, cs;
  int rows, cols;
};
inline View view_of(BlockTable& M, int a, int b) {
  Blk* blk = M.find(a, b);
  if (!blk) fail(SGF_INVALID_ARG, "internal: missing block");
  if (a <= b) return View{blk->p, (long long)blk->cols, 1, blk->rows, blk->cols};
  return View{blk->p, 1, (long long)blk->cols, blk->cols, blk->rows};
}

// ---------------------------------------------------------------------------
// Batched launch builders
// ---------------------------------------------------------------------------
struct GemmBatch {
  // per tile shape (128x128, 64x64, 64x16): the products and one 8-byte
  // record per output tile
  struct Set {
    std::vector<GemmTask> desc;
    std::vector<GemmTile> tiles;
    bool empty() const { return tiles.empty(); }
    void clear() {
      desc.clear();
      tiles.clear();
    }
  };
  Set big, small, narrow;
  std::vector<GemmSeg> segs;
  long long flops = 0;  // executed flops (information)

  // add all tiles of C(MxN) = beta*C + alpha * sum(segs)
  // lower_only: C is a symmetric diagonal block kept valid in its lower
  // triangle only; tiles strictly above the diagonal are skipped
  void add(double* C, long long c_rs, long long c_cs, int M, int N, double alpha, double beta,
           const std::vector<GemmSeg>& sg, int force = -1, bool lower_only = false) {
    add(C, c_rs, c_cs, M, N, alpha, beta, sg.data(), (int)sg.size(), force, lower_only);
  }
  // one segment (no temporary vector: a level adds ~1e5 of these)
  void add(double* C, long long c_rs, long long c_cs, int M, int N, double alpha, double beta, const GemmSeg& s1,
           int force = -1, bool lower_only = false) {
    add(C, c_rs, c_cs, M, N, alpha, beta, &s1, 1, force, lower_only);
  }
  void add(double* C, long long c_rs, long long c_cs, int M, int N, double alpha, double beta, const GemmSeg* sg,
           int nsg, int force, bool lower_only) {
    if (M <= 0 || N <= 0) return;
    int seg0 = (int)segs.size();
    segs.insert(segs.end(), sg, sg + nsg);
    // the 64x64 configuration is the fastest on B200 for every shape measured
    // (tools/gemm_bench.cu); the 128x128 path stays available via force = 1
    bool use_big = force == 1;
    static const bool narrow_off = getenv("SGF_NO_NARROW") != nullptr;
    const bool use_narrow = !use_big && N <= 16 && !narrow_off;  // basis-column products
    int bm = use_big ? 128 : 64, bn = use_narrow ? 16 : bm;
    Set& dst = use_big ? big : (use_narrow ? narrow : small);
    GemmTask t;
    t.C = C;
    t.c_rs = c_rs;
    t.c_cs = c_cs;
    t.M = M;
    t.N = N;
    t.m0 = 0;
    t.n0 = 0;
    t.seg0 = seg0;
    t.nseg = nsg;
    t.alpha = alpha;
    t.beta = beta;
    const uint32_t di = (uint32_t)dst.desc.size();
    dst.desc.push_back(t);
    const int ntm = (M + bm - 1) / bm, ntn = (N + bn - 1) / bn;
    for (int mt = 0; mt < ntm; ++mt)
      for (int nt = 0; nt < ntn; ++nt) {
        if (lower_only && nt * bn >= (mt + 1) * bm) continue;  // (64x16 tiles: n0 = 0 < m0 + 64)
        dst.tiles.push_back(GemmTile{di, (uint16_t)mt, (uint16_t)nt});
      }
    for (int i = 0; i < nsg; ++i) flops += 2LL * M * N * sg[i].K;
  }
  bool empty() const { return big.empty() && small.empty() && narrow.empty(); }
  // append another batch's products (segment and product indices shifted past ours)
  void append(const GemmBatch& o) {
    const int off = (int)segs.size();
    segs.insert(segs.end(), o.segs.begin(), o.segs.end());
    auto cat = [off](Set& d, const Set& src) {
      const uint32_t doff = (uint32_t)d.desc.size();
      const size_t b = d.desc.size(), bt = d.tiles.size();
      d.desc.insert(d.desc.end(), src.desc.begin(), src.desc.end());
      for (size_t i = b; i < d.desc.size(); ++i) d.desc[i].seg0 += off;
      d.tiles.insert(d.tiles.end(), src.tiles.begin(), src.tiles.end());
      for (size_t i = bt; i < d.tiles.size(); ++i) d.tiles[i].desc += doff;
    };
    cat(big, o.big);
    cat(small, o.small);
    cat(narrow, o.narrow);
    flops += o.flops;
  }
  void launch(Arena& scratch, cudaStream_t st);
  void clear() {
    big.clear();
    small.clear();
    narrow.clear();
    segs.clear();
  }
};

// Batched FP64 products on the INT8 tensor cores (ozaki.cu): operands are
// split once (split()), products are added per output block like GemmBatch.
struct OzOperand {
  int8_t* data = nullptr;
  int* e = nullptr;
  uint8_t* nz = nullptr;  // nonzero flags of the 128 x 32 tiles (when requested)
  int R = 0, K = 0, Rp = 0, Kp = 0;
};
struct OzBatch {
  std::vector<OzSplitJob> jobs;
  std::vector<OzTask> tasks;
  std::vector<OzSeg> segs;
  std::vector<std::pair<uint8_t*, size_t>> nz_clear;  // flag arrays zeroed before the splits
  double useful = 0.0;  // flops of the products (roofline accounting: dense, skipped zero tiles included)
  // nz_flags: record which 128 x 32 tiles of the operand hold a nonzero, so
  // products with it as the A operand skip the all-zero K tiles (block-sparse
  // couplings A_NB: 54-69% of their tiles are zero at levels 2-3 of 128^3)
  OzOperand split(Arena& mem, const double* x, long long rs, long long cs, int R, int K, bool nz_flags = false,
                  int* kfirst = nullptr, uint32_t* rmask = nullptr, int mwords = 0) {
    OzOperand o;
    o.R = R;
    o.K = K;
    o.Rp = (R + 127) / 128 * 128;
    o.Kp = (K + 31) / 32 * 32;
    o.data = mem.alloc_t<int8_t>((size_t)8 * o.Rp * o.Kp);
    o.e = mem.alloc_t<int>(o.Rp);
    static const bool nz_off = getenv("SGF_OZ_NO_SKIP") != nullptr;  // A/B switch: dense products
    if (nz_flags && !nz_off) {
      const size_t nb = (size_t)(o.Rp / 128) * (o.Kp / 32);
      o.nz = mem.alloc_t<uint8_t>(nb);
      nz_clear.push_back({o.nz, nb});
    }
    if (rmask) nz_clear.push_back({(uint8_t*)rmask, (size_t)R * mwords * sizeof(uint32_t)});
    jobs.push_back(OzSplitJob{x, rs, cs, R, K, o.Rp, o.Kp, o.data, o.e, o.nz, kfirst, rmask, mwords});
    return o;
  }
  void launch_splits(Arena& scratch, cudaStream_t st);
  // C (M x N) = beta*C + sum_i alpha_i A_i B_i^T, A_i with M rows, B_i with N
  // rows; lower_only skips tiles strictly above the diagonal; tri_b: B is
  // lower triangular (B[j][k] = 0 for k > j), so a tile stops at k < n0+128;
  // tri_a: A lower triangular (stop at k < m0+128); upper_b: B upper
  // triangular (B[j][k] = 0 for k < j), so a tile starts at k = n0
  void add(double* C, long long c_rs, long long c_cs, int M, int N, double beta,
           const std::vector<std::pair<std::pair<OzOperand, OzOperand>, double>>& terms, bool lower_only,
           bool tri_b, bool tri_a = false, bool upper_b = false) {
    if (M <= 0 || N <= 0) return;
    const int seg0 = (int)segs.size();
    for (auto& tm : terms) {
      const OzOperand& A = tm.first.first;
      const OzOperand& B = tm.first.second;
      segs.push_back(OzSeg{A.data, B.data, A.e, B.e, A.Rp, B.Rp, A.Kp / 32, tm.second, A.nz,
                           B.Kp == A.Kp ? B.nz : nullptr});
    }
    for (int m0 = 0; m0 < M; m0 += 128)
      for (int n0 = 0; n0 < N; n0 += 128) {
        if (lower_only && n0 >= m0 + 128) continue;
        int klim = 1 << 30;
        if (tri_b) klim = std::min(klim, (n0 + 128) / 32);
        if (tri_a) klim = std::min(klim, (m0 + 128) / 32);
        const int kstart = upper_b ? n0 / 32 : 0;
        tasks.push_back(OzTask{C, c_rs, c_cs, M, N, m0, n0, seg0, (int)terms.size(), beta, klim, kstart});
        for (auto& tm : terms) {
          const int kt = std::min(tm.first.first.Kp / 32, klim);
          const int ke = std::min(kt * 32, tm.first.first.K), kb = kstart * 32;
          if (ke > kb) useful += 2.0 * std::min(128, M - m0) * std::min(128, N - n0) * (ke - kb);
        }
      }
  }
  void launch(Arena& scratch, cudaStream_t st);
};

inline GemmSeg seg(const double* A, long long a_rs, long long a_ks, const double* B, long long b_rs, long long b_ks,
                   int K, int flags = 0) {
  GemmSeg s;
  s.A = A;
  s.B = B;
  s.a_rs = a_rs;
  s.a_ks = a_ks;
  s.b_rs = b_rs;
  s.b_ks = b_ks;
  s.K = K;
  s.flags = flags;
  return s;
}

struct CopyBatch {
  std::vector<CopyTask> tasks;
  void add(const double* src, long long s_rs, long long s_cs, double* dst, long long d_rs, long long d_cs, int rows,
           int cols) {
    if (rows <= 0 || cols <= 0) return;
    CopyTask t{src, dst, s_rs, s_cs, d_rs, d_cs, rows, cols};
    tasks.push_back(t);
  }
  // lower triangle of a square block, zeros above it (no separate zeroing pass)
  void add_lower(const double* src, long long s_rs, long long s_cs, double* dst, long long d_rs, long long d_cs,
                 int m) {
    if (m <= 0) return;
    CopyTask t{src, dst, s_rs, s_cs, d_rs, d_cs, m, m, 1};
    tasks.push_back(t);
  }
  void launch(Arena& scratch, cudaStream_t st);
};

void zero_upper(Arena& scratch, cudaStream_t st, const std::vector<TriTask>& tasks);

// Cholesky + explicit inverse of a batch of SPD matrices (W holds A on entry
// and L on exit; X must be zero on entry and holds L^{-1} on exit).
struct CholJob {
  double* W;
  double* X;
  int m;
  int node;  // for error messages
  int ld;    // leading dimension of W and X (>= m; even so rows are 16-byte aligned)
  const double* floor = nullptr;  // pivot floor (device) of the enclosing matrix; null: from this W
  int bw = 0;  // lower bandwidth of W (W[i][j] == 0 for i - j > bw; L inherits it); 0: dense
  bool upper_zero = false;  // W's strict upper triangle is zero on entry (no zeroing pass at the end)
};

// leading dimension of stored factor matrices: even, so every row starts
// 16-byte aligned and the apply GEMVs can use 128-bit loads
inline int pad_ld(int m) { return (m + 1) & ~1; }
// Breakdown statuses of Cholesky batches whose check is deferred (no host
// synchronisation per batch); verify() syncs and raises NotSPD for the
// earliest failing batch, lowest node id first (densela.py:106-110).
struct CholCheck {
  Arena* arena = nullptr;  // owns the status buffers until verify()
  struct Pending {
    int* status;
    double* piv;
    std::vector<int> nodes;
  };
  std::vector<Pending> pend;
  // deferred matrix symmetry check (setup): [max |A - A^T|, max |A|] as double bits
  unsigned long long* sym = nullptr;
  double sym_rtol = 1e-12;
  void verify(cudaStream_t st);
};
void chol_inv_batch(Ctx& ctx, Arena& scratch, std::vector<CholJob>& jobs, CholCheck* check = nullptr);
// same, with nodes of at least min_m unknowns factored recursively: the
// off-diagonal solve, the Schur update and the inverse's off-diagonal block
// are FP64 products on the INT8 tensor cores (ozaki.cu), the halves recurse
void chol_inv_rec(Ctx& ctx, Arena& scratch, std::vector<CholJob>& jobs, CholCheck* check, int min_m);

}  // namespace sgf
