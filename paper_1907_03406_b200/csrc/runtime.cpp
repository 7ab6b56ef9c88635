// Runtime utilities: arena allocator, batched launch builders, and the
// batched blocked Cholesky + explicit inverse used by elimination,
// compression and the final dense factor.
#include <omp.h>

#include "runtime.h"

#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <map>
#include <mutex>

namespace sgf {

unsigned long long g_kernel_launches = 0;
Profiler g_prof;

void Profiler::reset() {
  for (auto& r : recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  recs.clear();
}

void Profiler::read(double* out) {
  for (int i = 0; i < 3 * PROF_NCLS; ++i) out[i] = 0.0;
  for (auto& r : recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    out[3 * r.cls] += ms;
    out[3 * r.cls + 1] += r.work;
    out[3 * r.cls + 2] += (double)r.launches;
  }
}

ProfScope::ProfScope(cudaStream_t st, int cls, double work) : s(st) {
  if (!g_prof.on) return;
  Profiler::Rec r;
  r.cls = cls;
  r.work = work;
  r.launches = (long long)g_kernel_launches;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, st);
  idx = (int)g_prof.recs.size();
  g_prof.recs.push_back(r);
}

ProfScope::~ProfScope() {
  if (idx < 0) return;
  auto& r = g_prof.recs[idx];
  cudaEventRecord(r.b, s);
  r.launches = (long long)g_kernel_launches - r.launches;
}

void fail(int status, const std::string& msg) { throw Error{status, msg}; }

void upload_pinned(Ctx& ctx, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  const size_t chunk = (size_t)256 << 20;
  char* stage = (char*)ctx.pinned(std::min(bytes, chunk));
  for (size_t off = 0; off < bytes; off += chunk) {
    const size_t len = std::min(chunk, bytes - off);
    SGF_CUDA(cudaStreamSynchronize(ctx.stream));
    const char* s = (const char*)src + off;
    const long long nblk = (long long)((len + (1 << 20) - 1) >> 20);
#pragma omp parallel for
    for (long long b = 0; b < nblk; ++b) {
      const size_t o = (size_t)b << 20;
      std::memcpy(stage + o, s + o, std::min((size_t)1 << 20, len - o));
    }
    SGF_CUDA(cudaMemcpyAsync((char*)dst + off, stage, len, cudaMemcpyHostToDevice, ctx.stream));
  }
  SGF_CUDA(cudaStreamSynchronize(ctx.stream));
}

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  int st = (e == cudaErrorMemoryAllocation) ? SGF_OOM : SGF_CUDA;
  fail(st, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what);
}

void* Arena::alloc_bytes(size_t bytes) {
  bytes = (bytes + 255) & ~(size_t)255;
  if (bytes == 0) bytes = 256;
  for (auto& c : chunks_) {
    if (c.cap - c.off >= bytes) {
      void* p = c.base + c.off;
      c.off += bytes;
      used_ += bytes;
      return p;
    }
  }
  size_t cap = std::max(bytes, chunk_);
  auto t0 = std::chrono::steady_clock::now();
  void* p = plan_pool_ ? plan_chunk_get(cap, &cap, s_) : chunk_get(cap, &cap);
  if (HostTimer::on()) {
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 1.0) fprintf(stderr, "[arena] new %s chunk of %.1f MB took %.2f ms\n", plan_pool_ ? "plan" : "cache", cap / 1048576.0, ms);
  }
  chunks_.push_back(Chunk{(char*)p, cap, bytes});
  used_ += bytes;
  return p;
}

void Arena::release() {
  for (auto& c : chunks_) {
    if (plan_pool_) plan_chunk_put(c.base, c.cap, rel_);
    else chunk_put(c.base, c.cap);
  }
  chunks_.clear();
  used_ = 0;
}

// ---------------------------------------------------------------------------
// Process-wide cache of device chunks.  All library work of a context runs on
// one stream, so a chunk handed back by a finished phase can be reused by
// work enqueued later without synchronisation.  Repeated factorizations of
// the same problem then allocate nothing (cudaMalloc only when growing; the
// cache is emptied and the allocation retried on out-of-memory).
// ---------------------------------------------------------------------------
namespace {
std::mutex g_cache_mu;
std::map<int, std::multimap<size_t, void*>> g_cache;  // device -> (cap -> chunk)
struct PlanChunk {
  void* p;
  cudaEvent_t released;  // recorded after the chunk's last users
};
std::map<int, std::multimap<size_t, PlanChunk>> g_plan_cache;  // guarded by g_cache_mu
std::map<int, std::vector<cudaEvent_t>> g_plan_events;            // spare events per device (guarded by g_cache_mu)

// The ring is split into NSEG segments used in order; leaving a segment
// records an event, and re-entering it waits only for that event (work
// enqueued a whole ring ago), never for the whole stream.
constexpr int STAGE_NSEG = 8;
struct Stager {
  char* buf = nullptr;
  size_t cap = 0, seg = 0;  // total, per segment
  int cur = 0;
  size_t off = 0;           // offset inside the current segment
  cudaEvent_t ev[STAGE_NSEG] = {};
  bool used[STAGE_NSEG] = {};
  std::mutex mu;  // one ring per stream: the plan worker's uploads do not hold up the driver's
};
std::mutex g_stage_mu;  // guards the map only
std::map<cudaStream_t, Stager> g_stage;
}  // namespace

void stage_upload(cudaStream_t st, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  Stager* sp;
  {
    std::lock_guard<std::mutex> lk(g_stage_mu);
    sp = &g_stage[st];
  }
  Stager& s = *sp;
  auto tA = std::chrono::steady_clock::now();
  std::lock_guard<std::mutex> lk(s.mu);
  auto tB = std::chrono::steady_clock::now();
  const size_t need = (bytes + 255) & ~(size_t)255;
  if (need > s.seg) {  // (re)allocate a ring whose segments hold this upload
    if (s.buf) {
      SGF_CUDA(cudaStreamSynchronize(st));
      cudaFreeHost(s.buf);
    }
    s.seg = std::max(need, ((size_t)512 << 20) / STAGE_NSEG);
    s.cap = s.seg * STAGE_NSEG;
    SGF_CUDA(cudaMallocHost((void**)&s.buf, s.cap));
    for (int k = 0; k < STAGE_NSEG; ++k) {
      if (!s.ev[k]) SGF_CUDA(cudaEventCreateWithFlags(&s.ev[k], cudaEventDisableTiming));
      s.used[k] = false;
    }
    s.cur = 0;
    s.off = 0;
  }
  if (s.off + need > s.seg) {
    SGF_CUDA(cudaEventRecord(s.ev[s.cur], st));  // end of this segment's uses
    s.used[s.cur] = true;
    s.cur = (s.cur + 1) % STAGE_NSEG;
    if (s.used[s.cur]) {
      static const bool trace = getenv("SGF_TRACE") != nullptr;
      if (trace && cudaEventQuery(s.ev[s.cur]) == cudaErrorNotReady)
        fprintf(stderr, "[stage] waiting for staging segment %d\n", s.cur);
      SGF_CUDA(cudaEventSynchronize(s.ev[s.cur]));
    }
    s.off = 0;
  }
  char* p = s.buf + (size_t)s.cur * s.seg + s.off;
  s.off += need;
  if (bytes >= ((size_t)4 << 20)) {  // large task lists: one thread alone copies at only ~5 GB/s
    constexpr size_t BLK = (size_t)1 << 20;
    const long long nb = (long long)((bytes + BLK - 1) / BLK);
#pragma omp parallel for schedule(static)
    for (long long b = 0; b < nb; ++b)
      std::memcpy(p + b * BLK, (const char*)src + b * BLK, std::min(BLK, bytes - (size_t)b * BLK));
  } else {
    std::memcpy(p, src, bytes);
  }
  auto tC = std::chrono::steady_clock::now();
  SGF_CUDA(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, st));
  if (HostTimer::on()) {
    auto tD = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    if (ms(tA, tD) > 2.0)
      fprintf(stderr, "[stage] %.1f MB: lock %.2f ms, ring+memcpy %.2f ms, cudaMemcpyAsync %.2f ms\n", bytes / 1048576.0,
              ms(tA, tB), ms(tB, tC), ms(tC, tD));
  }
}

static int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

void* chunk_get(size_t bytes, size_t* cap) {
  const int dev = cur_device();
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto& cache = g_cache[dev];
    auto it = cache.lower_bound(bytes);
    if (it != cache.end() && it->first <= 2 * bytes + ((size_t)64 << 20)) {
      void* p = it->second;
      *cap = it->first;
      cache.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  static const bool trace = getenv("SGF_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    chunk_trim();
    e = cudaMalloc(&p, bytes);
  }
  SGF_CUDA(e);
  if (trace) {
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 1.0) fprintf(stderr, "[alloc] %.1f MB took %.2f ms\n", bytes / 1048576.0, ms);
  }
  *cap = bytes;
  return p;
}

void chunk_put(void* p, size_t cap) {
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache[dev].emplace(cap, p);
}

void chunk_trim() {
  cudaDeviceSynchronize();
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (auto& kv : g_cache[dev]) cudaFree(kv.second);
  g_cache[dev].clear();
  for (auto& kv : g_plan_cache[dev]) {
    cudaFree(kv.second.p);
    cudaEventDestroy(kv.second.released);
  }
  g_plan_cache[dev].clear();
}

void* plan_chunk_get(size_t bytes, size_t* cap, cudaStream_t user) {
  const int dev = cur_device();
  {
    std::unique_lock<std::mutex> lk(g_cache_mu);
    auto& cache = g_plan_cache[dev];
    auto it = cache.lower_bound(bytes);
    if (it != cache.end() && it->first <= 2 * bytes + ((size_t)64 << 20)) {
      const PlanChunk c = it->second;
      *cap = it->first;
      cache.erase(it);
      lk.unlock();
      // (cudaEventDestroy can block for as long as another thread waits in a
      // stream synchronisation -- 80 ms in the middle of a factorization --
      // so events go back to a free list instead)
      if (cudaEventQuery(c.released) != cudaSuccess) {
        cudaGetLastError();
        SGF_CUDA(cudaStreamWaitEvent(user, c.released, 0));
      }
      {
        std::lock_guard<std::mutex> lk2(g_cache_mu);
        g_plan_events[dev].push_back(c.released);
      }
      return c.p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    chunk_trim();
    e = cudaMalloc(&p, bytes);
  }
  SGF_CUDA(e);
  *cap = bytes;
  return p;
}

void plan_chunk_put(void* p, size_t cap, cudaStream_t last_user) {
  const int dev = cur_device();
  PlanChunk c{p, nullptr};
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto& spare = g_plan_events[dev];
    if (!spare.empty()) {
      c.released = spare.back();
      spare.pop_back();
    }
  }
  if ((!c.released && cudaEventCreateWithFlags(&c.released, cudaEventDisableTiming) != cudaSuccess) ||
      cudaEventRecord(c.released, last_user) != cudaSuccess) {
    // no event to order a later user by: wait for the device and free the chunk
    cudaGetLastError();
    cudaDeviceSynchronize();
    if (c.released) cudaEventDestroy(c.released);
    cudaFree(p);
    return;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_plan_cache[dev].emplace(cap, c);
}

// flops the tiles actually multiply (k range per segment after the
// triangular limits), for the roofline accounting
static double useful_flops(const GemmBatch::Set& st, const std::vector<GemmSeg>& segs, int bm, int bn,
                           bool padded = false) {
  double f = 0.0;
  for (const auto& tr : st.tiles) {
    const GemmTask& t = st.desc[tr.desc];
    const int m0 = tr.mt * bm, n0 = tr.nt * bn;
    const int rows = padded ? bm : std::min(bm, t.M - m0), cols = padded ? bn : std::min(bn, t.N - n0);
    for (int s = 0; s < t.nseg; ++s) {
      const GemmSeg& g = segs[t.seg0 + s];
      int kb = 0, ke = g.K;
      if (g.flags & SEG_KLIM_M) ke = std::min(ke, m0 + bm);
      if (g.flags & SEG_KLIM_N) ke = std::min(ke, n0 + bn);
      if (g.flags & SEG_KSTART_M) kb = std::max(kb, m0);
      if (g.flags & SEG_KSTART_N) kb = std::max(kb, n0);
      if (ke > kb) f += 2.0 * rows * cols * (ke - kb);
    }
  }
  return f;
}

static int trace_level() {
  static int v = getenv("SGF_TRACE") ? atoi(getenv("SGF_TRACE")) : 0;
  return v;
}

// SGF_TRACE=2: time every GEMM launch (synchronising) and print its rate
static void traced_gemm(Arena& scratch, const GemmBatch::Set& h, const GemmSeg* d_segs,
                        const std::vector<GemmSeg>& segs, int big, cudaStream_t st) {
  const int bm = big == 1 ? 128 : 64, bn = big == 1 ? 128 : (big == 2 ? 16 : 64);
  ProfScope ps(st, PROF_GEMM, g_prof.on ? useful_flops(h, segs, bm, bn) : 0.0);
  const GemmTask* d_desc = scratch.upload(h.desc);
  const GemmTile* d_tiles = scratch.upload(h.tiles);
  const int nt = (int)h.tiles.size();
  if (trace_level() != 2) {
    SGF_CUDA(launch_gemm(d_desc, d_tiles, nt, d_segs, big, st));
    return;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  SGF_CUDA(launch_gemm(d_desc, d_tiles, nt, d_segs, big, st));
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double f = useful_flops(h, segs, bm, bn);
  const double fx = useful_flops(h, segs, bm, bn, true);  // executed: full tiles over the same K ranges
  long long ksum = 0;
  for (auto& tr : h.tiles) {
    const GemmTask& t = h.desc[tr.desc];
    for (int s = 0; s < t.nseg; ++s) ksum += segs[t.seg0 + s].K;
  }
  fprintf(stderr, "[gemm] %s tiles=%7d avgK=%7.0f gflop=%9.3f ms=%8.3f tflops=%6.2f executed/useful=%5.2f\n",
          big == 1 ? "128" : (big == 2 ? " 16" : " 64"), nt, nt ? (double)ksum / nt : 0.0, f / 1e9, ms,
          f / (ms * 1e-3) / 1e12, fx / std::max(f, 1.0));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
}

void GemmBatch::launch(Arena& scratch, cudaStream_t st) {
  if (empty()) return;
  GemmSeg* d_segs = scratch.upload(segs);
  if (!big.empty()) traced_gemm(scratch, big, d_segs, segs, 1, st);
  if (!small.empty()) traced_gemm(scratch, small, d_segs, segs, 0, st);
  if (!narrow.empty()) traced_gemm(scratch, narrow, d_segs, segs, 2, st);
}

void OzBatch::launch_splits(Arena& scratch, cudaStream_t st) {
  if (jobs.empty()) return;
  if (nz_clear.size() <= 2) {
    for (auto& z : nz_clear) SGF_CUDA(cudaMemsetAsync(z.first, 0, z.second, st));
  } else {
    std::vector<ZeroRange> zr(nz_clear.size());
    for (size_t i = 0; i < nz_clear.size(); ++i) zr[i] = ZeroRange{nz_clear[i].first, nz_clear[i].second};
    SGF_CUDA(launch_zero_ranges(scratch.upload(zr), (int)zr.size(), st));
  }
  nz_clear.clear();
  // row-contiguous operands with aligned rows (rows staged once), other
  // row-contiguous or row-interleaved operands (coalesced CTA kernel) and the
  // rest, one launch each
  static const bool rows_off = getenv("SGF_OZ_SPLIT_ROWS") && atoi(getenv("SGF_OZ_SPLIT_ROWS")) == 0;
  std::vector<OzSplitJob> rowsj;
  std::vector<OzSplitJob> part[2];
  for (auto& j : jobs) {
    if (!rows_off && oz_split_rows_ok(j)) rowsj.push_back(j);
    else part[(j.cs == 1 || j.rs == 1) ? 0 : 1].push_back(j);  // the CTA kernel reads both
  }
  if (!rowsj.empty()) {
    int max_kp = 0;
    for (auto& j : rowsj) max_kp = std::max(max_kp, j.Kp);
    const int rpc = oz_split_rows_per_cta(max_kp);
    std::vector<long long> prefix(rowsj.size() + 1, 0);  // groups of rpc rows
    for (size_t i = 0; i < rowsj.size(); ++i) prefix[i + 1] = prefix[i] + rowsj[i].Rp / rpc;
    OzSplitJob* d_j = scratch.upload(rowsj);
    long long* d_p = scratch.upload(prefix);
    double bytes = 0.0;
    if (g_prof.on)
      for (auto& j : rowsj) bytes += 16.0 * j.Rp * j.Kp;
    ProfScope ps(st, PROF_OZSPLIT, bytes);
    SGF_CUDA(launch_oz_split_rows(d_j, d_p, (int)rowsj.size(), prefix.back(), max_kp, st));
  }
  if (HostTimer::on()) {
    auto desc = [](const char* what, const std::vector<OzSplitJob>& v) {
      if (v.empty()) return;
      long long rows = 0, el = 0;
      int kmax = 0, ntr = 0;
      for (auto& j : v) {
        rows += j.R;
        el += (long long)j.R * j.K;
        kmax = std::max(kmax, j.Kp);
        ntr += j.cs != 1;
      }
      fprintf(stderr, "[host] oz split %-5s %5zu jobs (%d col-major) rows %lld max Kp %d  %.2f GB fp64\n", what,
              v.size(), ntr, rows, kmax, el * 8e-9);
    };
    desc("rows", rowsj);
    desc("cta", part[0]);
    desc("warp", part[1]);
  }
  for (int w = 0; w < 2; ++w) {
    auto& js = part[w];
    if (js.empty()) continue;
    std::vector<long long> prefix(js.size() + 1, 0);  // 8-row groups
    for (size_t i = 0; i < js.size(); ++i) prefix[i + 1] = prefix[i] + js[i].Rp / 8;
    OzSplitJob* d_j = scratch.upload(js);
    long long* d_p = scratch.upload(prefix);
    double bytes = 0.0;  // FP64 read + 8 slices written per element
    if (g_prof.on)
      for (auto& j : js) bytes += 16.0 * j.Rp * j.Kp;
    ProfScope ps(st, PROF_OZSPLIT, bytes);
    SGF_CUDA(launch_oz_split(d_j, d_p, (int)js.size(), prefix.back(), st, w == 0));
  }
  jobs.clear();
}

void OzBatch::launch(Arena& scratch, cudaStream_t st) {
  if (tasks.empty()) return;
  OzSeg* d_s = scratch.upload(segs);
  OzTask* d_t = scratch.upload(tasks);
  ProfScope ps(st, PROF_OZ, useful);
  if (trace_level() == 2) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    SGF_CUDA(launch_oz_gemm(d_t, (int)tasks.size(), d_s, st));
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    fprintf(stderr, "[gemm] ozaki  tiles=%7zu segs=%7zu gflop=%9.3f ms=%8.3f tflops=%6.2f\n", tasks.size(),
            segs.size(), useful / 1e9, ms, useful / (ms * 1e-3) / 1e12);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  } else {
    SGF_CUDA(launch_oz_gemm(d_t, (int)tasks.size(), d_s, st));
  }
  tasks.clear();
  segs.clear();
  useful = 0.0;
}

void CopyBatch::launch(Arena& scratch, cudaStream_t st) {
  if (tasks.empty()) return;
  const size_t nt = tasks.size();
  std::vector<long long> prefix(nt);
  long long tot = 0;
  auto tiles = [&](size_t i) { return (long long)((tasks[i].rows + 31) / 32) * ((tasks[i].cols + 31) / 32); };
  if (nt < 65536) {
    for (size_t i = 0; i < nt; ++i) {
      prefix[i] = tot;
      tot += tiles(i);
    }
  } else {  // large merges: blocked two-pass exclusive scan
    constexpr size_t B = 4096;
    const size_t nb = (nt + B - 1) / B;
    std::vector<long long> bsum(nb + 1, 0);
#pragma omp parallel for schedule(static)
    for (size_t b = 0; b < nb; ++b) {
      long long s = 0;
      for (size_t i = b * B; i < std::min(nt, (b + 1) * B); ++i) s += tiles(i);
      bsum[b + 1] = s;
    }
    for (size_t b = 0; b < nb; ++b) bsum[b + 1] += bsum[b];
#pragma omp parallel for schedule(static)
    for (size_t b = 0; b < nb; ++b) {
      long long s = bsum[b];
      for (size_t i = b * B; i < std::min(nt, (b + 1) * B); ++i) {
        prefix[i] = s;
        s += tiles(i);
      }
    }
    tot = bsum[nb];
  }
  CopyTask* d_t = scratch.upload(tasks);
  long long* d_p = scratch.upload(prefix);
  double bytes = 0.0;
  if (g_prof.on)
    for (auto& t : tasks) bytes += 16.0 * t.rows * t.cols;
  ProfScope ps(st, PROF_MOVE, bytes);
  SGF_CUDA(launch_copy_tiled(d_t, d_p, (int)tasks.size(), tot, st));
}

void zero_upper(Arena& scratch, cudaStream_t st, const std::vector<TriTask>& tasks) {
  if (tasks.empty()) return;
  std::vector<long long> prefix(tasks.size());
  long long tot = 0;
  for (size_t i = 0; i < tasks.size(); ++i) {
    prefix[i] = tot;
    long long t = (tasks[i].m + 31) / 32;
    tot += t * t;
  }
  TriTask* d_t = scratch.upload(tasks);
  long long* d_p = scratch.upload(prefix);
  SGF_CUDA(launch_zero_upper(d_t, d_p, (int)tasks.size(), tot, st));
}

// ---------------------------------------------------------------------------
// Blocked left-looking Cholesky with the inverse built alongside.
// Per 64-column panel k (all jobs with m > k0 batched in each launch):
//   A: W[k0:, k]   -= L[k0:, :k0] L[k, :k0]^T            (panel update)
//      T_k          = L[k, :k0] X[:k0, :k0]               (inverse, part 1)
//   B: L_kk = chol(W_kk), D_k = L_kk^{-1}, X_kk = D_k    (diag tile, pivot check)
//   C: L[k1:, k]    = W[k1:, k] D_k^T                     (panel solve)
//      X[k, :k0]    = -D_k T_k                            (inverse, part 2)
// The breakdown rule is the reference's (densela.py:105-110).
// ---------------------------------------------------------------------------
// Recursive split of the large nodes: with W = [A11 .; A21 A22] (lower part),
//   (L11, X11) = chol_inv(A11);  L21 = A21 X11^T;  A22 -= L21 L21^T;
//   (L22, X22) = chol_inv(A22);  X21 = -X22 (L21 X11)
// The products of each split run on the INT8 tensor cores (ozaki.cu), every
// operand with its nonzero tile flags (A_BB is block-sparse, and so are its
// factor blocks: the products skip all-zero operand tiles);
// halves below min_m, and small nodes, take the blocked kernel above.  The
// pivot floor of every half is the enclosing node's (densela.py:105-110).
void chol_inv_rec(Ctx& ctx, Arena& scratch, std::vector<CholJob>& jobs, CholCheck* check, int min_m) {
  std::vector<CholJob> small, big;
  // (the int32 accumulators of a product hold K < 16.6k exactly: halves <= 16000)
  for (auto& j : jobs) (j.m >= min_m && min_m > 0 && j.m <= 32000 ? big : small).push_back(j);
  if (!small.empty()) chol_inv_batch(ctx, scratch, small, check);
  if (big.empty()) return;
  cudaStream_t st = ctx.stream;
  const int nb = (int)big.size();
  // pivot floors of the whole nodes, shared by their halves (one launch)
  {
    std::vector<const double*> wv;
    std::vector<int> mv, lv, who;
    for (int i = 0; i < nb; ++i)
      if (!big[i].floor) {
        wv.push_back(big[i].W);
        mv.push_back(big[i].m);
        lv.push_back(big[i].ld);
        who.push_back(i);
      }
    if (!wv.empty()) {
      double* f = scratch.alloc(wv.size());
      SGF_CUDA(launch_max_diag(scratch.upload(wv), scratch.upload(mv), scratch.upload(lv), (int)wv.size(), f, st));
      for (size_t k = 0; k < who.size(); ++k) big[who[k]].floor = f + k;
    }
  }
  std::vector<int> m1(nb), m2(nb);
  std::vector<CholJob> j11, j22;
  for (int i = 0; i < nb; ++i) {
    const CholJob& j = big[i];
    m1[i] = ((j.m / 2) + 63) / 64 * 64;
    m2[i] = j.m - m1[i];
    CholJob h = j;
    h.m = m1[i];
    j11.push_back(h);
  }
  chol_inv_rec(ctx, scratch, j11, check, min_m);
  // L21 = A21 X11^T  (X11 lower: tile k < n0 + 128)
  OzBatch oz;
  std::vector<OzOperand> a21(nb), x11(nb), x11t(nb), l21(nb);
  for (int i = 0; i < nb; ++i) {
    const CholJob& j = big[i];
    const long long ld = j.ld;
    a21[i] = oz.split(scratch, j.W + (long long)m1[i] * ld, ld, 1, m2[i], m1[i], true);  // block-sparse A21
    x11[i] = oz.split(scratch, j.X, ld, 1, m1[i], m1[i], true);
  }
  oz.launch_splits(scratch, st);
  for (int i = 0; i < nb; ++i) {
    const CholJob& j = big[i];
    const long long ld = j.ld;
    oz.add(j.W + (long long)m1[i] * ld, ld, 1, m2[i], m1[i], 0.0, {{{a21[i], x11[i]}, 1.0}}, false, true);
  }
  oz.launch(scratch, st);
  // A22 -= L21 L21^T (lower part)
  for (int i = 0; i < nb; ++i) {
    const CholJob& j = big[i];
    const long long ld = j.ld;
    l21[i] = oz.split(scratch, j.W + (long long)m1[i] * ld, ld, 1, m2[i], m1[i], true);
  }
  oz.launch_splits(scratch, st);
  for (int i = 0; i < nb; ++i) {
    const CholJob& j = big[i];
    const long long ld = j.ld;
    oz.add(j.W + (long long)m1[i] * ld + m1[i], ld, 1, m2[i], m2[i], 1.0, {{{l21[i], l21[i]}, -1.0}}, true, false);
  }
  oz.launch(scratch, st);
  for (int i = 0; i < nb; ++i) {
    const CholJob& j = big[i];
    CholJob h = j;
    h.W = j.W + (long long)m1[i] * j.ld + m1[i];
    h.X = j.X + (long long)m1[i] * j.ld + m1[i];
    h.m = m2[i];
    // the A22 update writes whole diagonal tiles: its upper part is no longer zero
    h.upper_zero = false;
    j22.push_back(h);
  }
  chol_inv_rec(ctx, scratch, j22, check, min_m);
  // T = L21 X11 (as L21 . (X11^T)^T; X11^T upper: tile k >= n0), then
  // X21 = -X22 T (X22 lower: tile k < m0 + 128)
  std::vector<double*> T(nb);
  std::vector<int> ldt(nb);
  for (int i = 0; i < nb; ++i) {
    const CholJob& j = big[i];
    ldt[i] = pad_ld(m1[i]);
    T[i] = scratch.alloc((size_t)m2[i] * ldt[i]);
    x11t[i] = oz.split(scratch, j.X, 1, j.ld, m1[i], m1[i], true);
  }
  oz.launch_splits(scratch, st);
  for (int i = 0; i < nb; ++i)
    oz.add(T[i], ldt[i], 1, m2[i], m1[i], 0.0, {{{l21[i], x11t[i]}, 1.0}}, false, false, false, true);
  oz.launch(scratch, st);
  std::vector<OzOperand> x22(nb), tt(nb);
  for (int i = 0; i < nb; ++i) {
    const CholJob& j = big[i];
    const long long ld = j.ld;
    x22[i] = oz.split(scratch, j.X + (long long)m1[i] * ld + m1[i], ld, 1, m2[i], m2[i], true);
    tt[i] = oz.split(scratch, T[i], 1, ldt[i], m1[i], m2[i], true);
  }
  oz.launch_splits(scratch, st);
  for (int i = 0; i < nb; ++i) {
    const CholJob& j = big[i];
    oz.add(j.X + (long long)m1[i] * j.ld, j.ld, 1, m2[i], m1[i], 0.0, {{{x22[i], tt[i]}, -1.0}}, false, false, true);
  }
  oz.launch(scratch, st);
  // L has exact zeros above the diagonal: the A12 block of W
  std::vector<TriTask> up;
  for (int i = 0; i < nb; ++i)
    if (!big[i].upper_zero) up.push_back(TriTask{big[i].W, big[i].m, big[i].ld});
  zero_upper(scratch, st, up);
}

void CholCheck::verify(cudaStream_t st) {
  if (sym) {  // an asymmetric matrix is reported before anything computed from it
    SGF_CUDA(cudaStreamSynchronize(st));
    unsigned long long h[3];
    SGF_CUDA(cudaMemcpy(h, sym, sizeof h, cudaMemcpyDeviceToHost));
    sym = nullptr;
    if (h[2]) {  // densela.py:43-49 _as_matrix
      pend.clear();
      fail(SGF_INVALID_ARG, "matrix contains NaN or Inf entries");
    }
    double asym, scale;
    std::memcpy(&asym, &h[0], sizeof(double));
    std::memcpy(&scale, &h[1], sizeof(double));
    if (asym > sym_rtol * std::max(scale, 1e-300)) {
      pend.clear();
      char buf[128];
      snprintf(buf, sizeof buf, "matrix is not symmetric (max asymmetry %.2e)", asym);
      fail(SGF_NON_SYMMETRIC, buf);
    }
  }
  if (pend.empty()) return;
  SGF_CUDA(cudaStreamSynchronize(st));
  for (auto& p : pend) {
    const int nj = (int)p.nodes.size();
    std::vector<int> status(nj);
    std::vector<double> piv(nj);
    SGF_CUDA(cudaMemcpy(status.data(), p.status, nj * sizeof(int), cudaMemcpyDeviceToHost));
    SGF_CUDA(cudaMemcpy(piv.data(), p.piv, nj * sizeof(double), cudaMemcpyDeviceToHost));
    int worst = -1;
    for (int i = 0; i < nj; ++i)
      if (status[i] != 0 && (worst < 0 || p.nodes[i] < p.nodes[worst])) worst = i;
    if (worst >= 0) {
      char buf[256];
      snprintf(buf, sizeof buf, "non-positive pivot %.3e at index %d (node %d)", piv[worst], status[worst] - 1,
               p.nodes[worst]);
      pend.clear();
      fail(SGF_NOT_SPD, buf);
    }
  }
  pend.clear();
}

void chol_inv_batch(Ctx& ctx, Arena& scratch, std::vector<CholJob>& jobs, CholCheck* check) {
  if (jobs.empty()) return;
  cudaStream_t st = ctx.stream;
  const int nj = (int)jobs.size();
  std::vector<const double*> wp(nj);
  std::vector<int> ms(nj), lds(nj);
  int mmax = 0;
  for (int i = 0; i < nj; ++i) {
    wp[i] = jobs[i].W;
    ms[i] = jobs[i].m;
    lds[i] = jobs[i].ld;
    mmax = std::max(mmax, jobs[i].m);
  }
  // breakdown status lives as long as the check that will read it
  Arena& keep = check ? *check->arena : scratch;
  double* d_floor = scratch.alloc(nj);
  {
    const double** d_wp = scratch.upload(wp);
    int* d_m = scratch.upload(ms);
    int* d_ld = scratch.upload(lds);
    SGF_CUDA(launch_max_diag(d_wp, d_m, d_ld, nj, d_floor, st));
  }
  int* d_status = keep.alloc_t<int>(nj);
  double* d_piv = keep.alloc(nj);
  SGF_CUDA(cudaMemsetAsync(d_status, 0, nj * sizeof(int), st));
  std::vector<double*> dinv(nj), tk(nj);
  for (int i = 0; i < nj; ++i) {
    dinv[i] = scratch.alloc(64 * 64);
    tk[i] = scratch.alloc((size_t)64 * std::max(jobs[i].m, 1));
  }

  // task lists of a panel built by host threads over contiguous job ranges,
  // concatenated in range order (3375 level-1 nodes at 128^3: the serial
  // loop kept the device waiting)
  const int nthr = nj >= 1024 ? std::max(1, std::min(omp_get_max_threads(), nj / 64)) : 1;
  double t_build = 0.0, t_launch = 0.0;
  for (int k0 = 0; k0 < mmax; k0 += 64) {
    auto tb0 = std::chrono::steady_clock::now();
    GemmBatch ga, gc;
    std::vector<DiagTask> dt;
    std::vector<double*> xd;
    std::vector<int> xl;
    std::vector<GemmBatch> tga(nthr), tgc(nthr);
    std::vector<std::vector<DiagTask>> tdt(nthr);
    std::vector<std::vector<double*>> txd(nthr);
    std::vector<std::vector<int>> txl(nthr);
#pragma omp parallel for num_threads(nthr) schedule(static, 1)
    for (int th = 0; th < nthr; ++th) {
      GemmBatch& ga = tga[th];
      GemmBatch& gc = tgc[th];
      std::vector<DiagTask>& dt = tdt[th];
      std::vector<double*>& xd = txd[th];
      std::vector<int>& xl = txl[th];
      const int i0 = (int)((long long)nj * th / nthr), i1 = (int)((long long)nj * (th + 1) / nthr);
    for (int i = i0; i < i1; ++i) {
      const int m = jobs[i].m;
      const long long ld = jobs[i].ld;
      if (m <= k0) continue;
      double* W = jobs[i].W;
      double* X = jobs[i].X;
      const int nb = std::min(64, m - k0), k1 = k0 + nb;
      // banded W (level-1 interiors in lexicographic order): L[i][j] = 0 for
      // i - j > bw, so the panel update and T_k only need K in [kb, k0) and
      // rows below k1 + bw (the skipped products are exact zeros)
      const bool band = jobs[i].bw > 0 && jobs[i].bw < m;
      const int kb = band ? std::max(0, (k0 - jobs[i].bw) / 64 * 64) : 0;
      const int rend = band ? std::min(m, k1 + jobs[i].bw) : m;
      if (k0 > 0) {
        // A: panel update and T_k (T_k is nb x k0 with leading dimension m)
        ga.add(W + k0 * ld + k0, ld, 1, rend - k0, nb, -1.0, 1.0,
               {seg(W + k0 * ld + kb, ld, 1, W + k0 * ld + kb, ld, 1, k0 - kb)});
        ga.add(tk[i], m, 1, nb, k0, 1.0, 0.0,
               {seg(W + k0 * ld + kb, ld, 1, X + (long long)kb * ld, 1, ld, k0 - kb, kb ? 0 : SEG_KSTART_N)}, 0);
      }
      DiagTask d;
      d.W = W;
      d.Dinv = dinv[i];
      d.ld = (int)ld;
      d.k0 = k0;
      d.nb = nb;
      d.floor = jobs[i].floor ? jobs[i].floor : d_floor + i;
      d.node = i;
      dt.push_back(d);
      xd.push_back(X);
      xl.push_back((int)ld);
      if (rend > k1)
        gc.add(W + k1 * ld + k0, ld, 1, rend - k1, nb, 1.0, 0.0,
               {seg(W + k1 * ld + k0, ld, 1, dinv[i], 64, 1, nb, SEG_KLIM_N)}, 0);
      if (k0 > 0)
        gc.add(X + k0 * ld, ld, 1, nb, k0, -1.0, 0.0, {seg(dinv[i], 64, 1, tk[i], 1, m, nb, SEG_KLIM_M)}, 0);
    }
    }
    for (int th = 0; th < nthr; ++th) {
      ga.append(tga[th]);
      gc.append(tgc[th]);
      dt.insert(dt.end(), tdt[th].begin(), tdt[th].end());
      xd.insert(xd.end(), txd[th].begin(), txd[th].end());
      xl.insert(xl.end(), txl[th].begin(), txl[th].end());
    }
    auto tb1 = std::chrono::steady_clock::now();
    t_build += std::chrono::duration<double, std::milli>(tb1 - tb0).count();
    ga.launch(scratch, st);
    {
      DiagTask* d_dt = scratch.upload(dt);
      double** d_xd = scratch.upload(xd);
      int* d_xl = scratch.upload(xl);
      ProfScope ps(st, PROF_CHOL, 0.0);
      SGF_CUDA(launch_diag_chol_ex(d_dt, (int)dt.size(), d_status, d_piv, d_xd, d_xl, st));
    }
    gc.launch(scratch, st);
    t_launch += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tb1).count();
  }
  if (HostTimer::on())
    fprintf(stderr, "[host] chol_inv_batch: %d jobs, %d threads, task build %.2f ms, uploads+launches %.2f ms\n", nj,
            nthr, t_build, t_launch);
  std::vector<TriTask> tri;
  for (auto& j : jobs)
    if (!j.upper_zero) tri.push_back(TriTask{j.W, j.m, j.ld});
  zero_upper(scratch, st, tri);

  CholCheck local;
  CholCheck& chk = check ? *check : local;
  CholCheck::Pending p;
  p.status = d_status;
  p.piv = d_piv;
  for (auto& j : jobs) p.nodes.push_back(j.node);
  chk.pend.push_back(std::move(p));
  if (!check) chk.verify(st);
}

}  // namespace sgf
