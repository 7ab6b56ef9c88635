// extern "C" boundary (include/sgf.h).  Every entry point converts internal
// errors to an sgf_status and records the message on the context.
#include <algorithm>
#include <cstdio>

#include "precond.h"
#include "primitives.h"

using namespace sgf;

struct sgf_ctx {
  Ctx c;
};
struct sgf_precond {
  Precond* p;
  sgf_ctx* ctx;
};
struct sgf_csr {
  Csr a;
  sgf_ctx* ctx;
};

namespace {
thread_local std::string g_orphan_error;

template <class F>
int guarded(sgf_ctx* ctx, F&& f) {
  try {
    // every entry point runs on its context's device (a process may hold
    // contexts on several GPUs)
    if (ctx && ctx->c.stream) SGF_CUDA(cudaSetDevice(ctx->c.device));
    f();
    return SGF_OK;
  } catch (const Error& e) {
    if (ctx) ctx->c.last_error = e.msg;
    else g_orphan_error = e.msg;
    return e.status;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->c.last_error = "host out of memory";
    return SGF_OOM;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.last_error = e.what();
    return SGF_INVALID_ARG;
  }
}

struct DevVec {
  double* p = nullptr;
  cudaStream_t s;
  DevVec(size_t n, cudaStream_t st) : s(st) { SGF_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * 8, st)); }
  ~DevVec() { cudaFreeAsync(p, s); }
};
}  // namespace

extern "C" {

int sgf_create(sgf_ctx** out, int device) {
  if (!out) return SGF_INVALID_ARG;
  *out = nullptr;
  sgf_ctx* ctx = new sgf_ctx();
  int st = guarded(ctx, [&] {
    SGF_CUDA(cudaSetDevice(device));
    ctx->c.device = device;
    SGF_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
    SGF_CUDA(cudaStreamCreateWithFlags(&ctx->c.upload_stream, cudaStreamNonBlocking));
    SGF_CUDA(cudaEventCreateWithFlags(&ctx->c.upload_ev, cudaEventDisableTiming));
    cudaMemPool_t pool;
    SGF_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    SGF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  });
  if (st != SGF_OK) {
    g_orphan_error = ctx->c.last_error;
    delete ctx;
    return st;
  }
  *out = ctx;
  return SGF_OK;
}

int sgf_destroy(sgf_ctx* ctx) {
  if (!ctx) return SGF_OK;
  if (ctx->c.stream) {
    cudaStreamSynchronize(ctx->c.stream);
    cudaStreamDestroy(ctx->c.stream);
  }
  if (ctx->c.order_ev) cudaEventDestroy(ctx->c.order_ev);
  if (ctx->c.upload_stream) {
    cudaStreamSynchronize(ctx->c.upload_stream);
    cudaStreamDestroy(ctx->c.upload_stream);
  }
  if (ctx->c.upload_ev) cudaEventDestroy(ctx->c.upload_ev);
  delete ctx;
  return SGF_OK;
}

const char* sgf_last_error(const sgf_ctx* ctx) { return ctx ? ctx->c.last_error.c_str() : g_orphan_error.c_str(); }

void* sgf_stream(sgf_ctx* ctx) { return ctx ? (void*)ctx->c.stream : nullptr; }

int sgf_sync(sgf_ctx* ctx) {
  return guarded(ctx, [&] { SGF_CUDA(cudaStreamSynchronize(ctx->c.stream)); });
}

int sgf_trim(sgf_ctx* ctx) {
  return guarded(ctx, [&] {
    SGF_CUDA(cudaSetDevice(ctx->c.device));
    SGF_CUDA(cudaStreamSynchronize(ctx->c.stream));
    chunk_trim();
  });
}

int sgf_factorize(sgf_ctx* ctx, const sgf_factor_args* args, sgf_precond** out) {
  if (!ctx || !args || !out) return SGF_INVALID_ARG;
  *out = nullptr;
  return guarded(ctx, [&] {
    SGF_CUDA(cudaSetDevice(ctx->c.device));
    Precond* p = factorize(ctx->c, *args);
    *out = new sgf_precond{p, ctx};
  });
}

int sgf_precond_free(sgf_precond* p) {
  if (!p) return SGF_OK;
  cudaStreamSynchronize(p->ctx->c.stream);
  delete p->p;
  delete p;
  return SGF_OK;
}

int64_t sgf_precond_n(const sgf_precond* p) { return p ? p->p->n : 0; }

const char* sgf_precond_stats_json(const sgf_precond* p) { return p ? p->p->stats.c_str() : ""; }

int sgf_precond_rank_trace(const sgf_precond* p, int32_t* out, int cap) {
  if (!p) return 0;
  const int n = (int)p->p->trace.size() / 3;
  if (out)
    for (int i = 0; i < std::min(n * 3, cap * 3); ++i) out[i] = p->p->trace[i];
  return n;
}

int sgf_precond_num_factors(const sgf_precond* p) { return p ? (int)p->p->factors.size() : 0; }

int sgf_precond_coupling_bytes(const sgf_precond* p, double* out) { return sgf_precond_coupling_bytes_level(p, 0, out); }

int sgf_precond_coupling_bytes_level(const sgf_precond* p, int level, double* out) {
  if (!p || !out) return SGF_INVALID_ARG;
  sgf_ctx* ctx = p->ctx;
  return guarded(ctx, [&] {
    SGF_CUDA(cudaStreamSynchronize(ctx->c.stream));
    double dense = 0.0, nz = 0.0;
    std::vector<uint32_t> mk;
    std::vector<int> kf;
    for (const Factor& f : p->p->factors) {
      if (f.type != SGF_FACTOR_ELIMINATION || !f.E || f.c <= 0 || (level > 0 && f.level != level)) continue;
      dense += 8.0 * f.c * f.m;
      if (f.emask) {
        mk.resize((size_t)f.c * f.emw);
        SGF_CUDA(cudaMemcpy(mk.data(), f.emask, mk.size() * 4, cudaMemcpyDeviceToHost));
        for (int r = 0; r < f.c; ++r)
          for (int w = 0; w < f.emw; ++w) {
            const uint32_t b = mk[(size_t)r * f.emw + w];
            for (int t = 0; t < 32; ++t)
              if ((b >> t) & 1u) nz += 8.0 * std::max(0, std::min(32, f.m - 32 * (32 * w + t)));
          }
      } else if (f.ekfirst) {
        kf.resize(f.c);
        SGF_CUDA(cudaMemcpy(kf.data(), f.ekfirst, kf.size() * 4, cudaMemcpyDeviceToHost));
        for (int r = 0; r < f.c; ++r) nz += 8.0 * std::max(0, f.m - kf[r]);
      } else {
        nz += 8.0 * f.c * f.m;
      }
    }
    // L^{-1} rows with tile masks: the lower triangle (dense) against its
    // nonzero tiles, each tile counted up to the diagonal
    for (const Factor& f : p->p->factors) {
      if (!f.xmask || (level > 0 && f.level != level)) continue;
      dense += 4.0 * f.m * (f.m + 1.0);
      mk.resize((size_t)f.m * f.xmw);
      SGF_CUDA(cudaMemcpy(mk.data(), f.xmask, mk.size() * 4, cudaMemcpyDeviceToHost));
      for (int r = 0; r < f.m; ++r)
        for (int w = 0; w < f.xmw; ++w) {
          const uint32_t b = mk[(size_t)r * f.xmw + w];
          for (int t = 0; t < 32; ++t)
            if ((b >> t) & 1u) nz += 8.0 * std::max(0, std::min(32, r + 1 - 32 * (32 * w + t)));
        }
    }
    out[0] = dense;
    out[1] = nz;
  });
}

// Diagnostic: bytes of the couplings E of one level (0 = all) as the forward
// sweeps read them under different skipping granularities:
//   out[0] dense, out[1] nonzero 32-column tiles, out[2] from the first
//   nonzero tile to the row's end, out[3] 256-column chunks from the first
//   nonzero tile (all-zero chunks skipped, last chunk kept), out[4] chunks
//   trimmed to their first..last nonzero tile, out[5] number of maximal runs
//   of nonzero tiles (one copy each at tile granularity)
int sgf_precond_coupling_bytes_detail(const sgf_precond* p, int level, double* out) {
  if (!p || !out) return SGF_INVALID_ARG;
  sgf_ctx* ctx = p->ctx;
  return guarded(ctx, [&] {
    SGF_CUDA(cudaStreamSynchronize(ctx->c.stream));
    for (int i = 0; i < 6; ++i) out[i] = 0.0;
    std::vector<uint32_t> mk;
    for (const Factor& f : p->p->factors) {
      if (f.type != SGF_FACTOR_ELIMINATION || !f.E || f.c <= 0 || (level > 0 && f.level != level)) continue;
      out[0] += 8.0 * f.c * f.m;
      if (!f.emask) {
        for (int i = 1; i < 5; ++i) out[i] += 8.0 * f.c * f.m;
        out[5] += f.c;
        continue;
      }
      mk.resize((size_t)f.c * f.emw);
      SGF_CUDA(cudaMemcpy(mk.data(), f.emask, mk.size() * 4, cudaMemcpyDeviceToHost));
      const int nt = (f.m + 31) / 32;
      for (int r = 0; r < f.c; ++r) {
        auto bit = [&](int t) { return (mk[(size_t)r * f.emw + (t >> 5)] >> (t & 31)) & 1u; };
        auto tw = [&](int t) { return std::max(0, std::min(32, f.m - 32 * t)); };
        int first = -1;
        bool prev = false;
        for (int t = 0; t < nt; ++t) {
          const bool b = bit(t);
          if (b) {
            out[1] += 8.0 * tw(t);
            if (first < 0) first = t;
            if (!prev) out[5] += 1;
          }
          prev = b;
        }
        if (first < 0) continue;
        for (int t = first; t < nt; ++t) out[2] += 8.0 * tw(t);
        for (int t0 = first; t0 < nt; t0 += 8) {
          int lo = -1, hi = -1;
          for (int t = t0; t < std::min(nt, t0 + 8); ++t)
            if (bit(t)) {
              if (lo < 0) lo = t;
              hi = t;
            }
          const bool last = t0 + 8 >= nt;
          if (lo < 0 && !last) continue;
          for (int t = t0; t < std::min(nt, t0 + 8); ++t) out[3] += 8.0 * tw(t);
          for (int t = lo; lo >= 0 && t <= hi; ++t) out[4] += 8.0 * tw(t);
        }
      }
    }
  });
}

int sgf_precond_factor_info(const sgf_precond* p, int k, int64_t* info) {
  if (!p || k < 0 || k >= (int)p->p->factors.size() || !info) return SGF_INVALID_ARG;
  const Factor& f = p->p->factors[k];
  info[0] = f.type;
  info[1] = f.node;
  info[2] = f.m;
  info[3] = f.c;
  info[4] = f.r;
  info[5] = f.level;
  info[6] = f.steps;
  info[7] = f.ncols;
  return SGF_OK;
}

int sgf_precond_factor_copy(const sgf_precond* p, int k, int what, void* host_out, int64_t cap_bytes) {
  if (!p || k < 0 || k >= (int)p->p->factors.size() || !host_out) return SGF_INVALID_ARG;
  sgf_ctx* ctx = p->ctx;
  return guarded(ctx, [&] {
    const Factor& f = p->p->factors[k];
    cudaStream_t st = ctx->c.stream;
    auto need = [&](int64_t bytes) {
      if (bytes > cap_bytes) fail(SGF_SHAPE, "output buffer too small");
    };
    const long long mm = (long long)f.m * f.m;
    switch (what) {
      case 0:
        need(8LL * f.m);
        std::memcpy(host_out, f.idx.data(), 8LL * f.m);
        break;
      case 1:
        need(8 * mm);
        SGF_CUDA(cudaMemcpy2DAsync(host_out, 8 * f.m, f.L, 8 * f.ld, 8 * f.m, f.m, cudaMemcpyDeviceToHost, st));
        break;
      case 2:
        need(8LL * f.c * f.m);
        materialize_l1_e(p->p);
        if (f.c)
          SGF_CUDA(cudaMemcpy2DAsync(host_out, 8 * f.m, f.E, 8 * f.ld, 8 * f.m, f.c, cudaMemcpyDeviceToHost, st));
        break;
      case 3:
        need(8LL * f.c);
        if (f.c) std::memcpy(host_out, f.nidx.data(), 8LL * f.c);
        break;
      case 4: {
        // Q = I - V T V^T (m x m), formed on the host from the reflectors
        need(8 * mm);
        const int m = f.m, s = f.steps;
        std::vector<double> V((size_t)m * s), T((size_t)s * s);
        if (s) {
          SGF_CUDA(cudaMemcpyAsync(V.data(), f.V, V.size() * 8, cudaMemcpyDeviceToHost, st));
          SGF_CUDA(cudaMemcpyAsync(T.data(), f.Tw, T.size() * 8, cudaMemcpyDeviceToHost, st));
        }
        SGF_CUDA(cudaStreamSynchronize(st));
        double* Q = (double*)host_out;
        std::vector<double> VT((size_t)s * m, 0.0);  // (T V^T)[a][j]
        for (int a = 0; a < s; ++a)
          for (int b = a; b < s; ++b) {
            const double tab = T[(size_t)a * s + b];
            if (tab == 0.0) continue;
            for (int j = 0; j < m; ++j) VT[(size_t)a * m + j] += tab * V[(size_t)b * m + j];
          }
        for (int i = 0; i < m; ++i)
          for (int j = 0; j < m; ++j) {
            double acc = (i == j) ? 1.0 : 0.0;
            for (int a = 0; a < s; ++a) acc -= V[(size_t)a * m + i] * VT[(size_t)a * m + j];
            Q[(size_t)i * m + j] = acc;
          }
        break;
      }
      case 5:
        need(8 * mm);
        SGF_CUDA(cudaMemcpy2DAsync(host_out, 8 * f.m, f.inv, 8 * f.ld, 8 * f.m, f.m, cudaMemcpyDeviceToHost, st));
        break;
      case 6:
        need(8LL * f.perm.size());
        for (size_t i = 0; i < f.perm.size(); ++i) ((int64_t*)host_out)[i] = f.perm[i];
        break;
      default:
        fail(SGF_INVALID_ARG, "unknown factor field");
    }
    SGF_CUDA(cudaStreamSynchronize(st));
  });
}

int sgf_apply(sgf_precond* p, int op, const double* x, double* y, int on_device) {
  if (!p || !x || !y) return SGF_INVALID_ARG;
  sgf_ctx* ctx = p->ctx;
  return guarded(ctx, [&] {
    cudaStream_t st = ctx->c.stream;
    const long long n = p->p->n;
    if (on_device) {
      apply_op(p->p, op, x, y);
      SGF_CUDA(cudaStreamSynchronize(st));
    } else {
      DevVec d(n, st);
      SGF_CUDA(cudaMemcpyAsync(d.p, x, n * 8, cudaMemcpyHostToDevice, st));
      apply_op(p->p, op, d.p, d.p);
      SGF_CUDA(cudaMemcpyAsync(y, d.p, n * 8, cudaMemcpyDeviceToHost, st));
      SGF_CUDA(cudaStreamSynchronize(st));
    }
  });
}

int sgf_cell_unknowns(int nx, int ny, int nz, int tx, int ty, int tz, const int64_t* lox, const int64_t* hix,
                      const int64_t* loy, const int64_t* hiy, const int64_t* loz, const int64_t* hiz, int components,
                      int64_t* out_ptr, int64_t* out_unknowns) {
  if (nx <= 0 || ny <= 0 || nz <= 0 || tx <= 0 || ty <= 0 || tz <= 0 || components <= 0 || !out_ptr || !out_unknowns)
    return SGF_INVALID_ARG;
  const long long nc = (long long)tx * ty * tz;
  const long long nv = (long long)nx * ny * nz;
  out_ptr[0] = 0;
  for (long long c = 0; c < nc; ++c) {
    const long long cx = c / ((long long)ty * tz), cy = (c / tz) % ty, cz = c % tz;
    const long long size = (hix[cx] - lox[cx] + 1) * (hiy[cy] - loy[cy] + 1) * (hiz[cz] - loz[cz] + 1);
    out_ptr[c + 1] = out_ptr[c] + size * components;
  }
  if (out_ptr[nc] != nv * components) return SGF_INVALID_ARG;
#pragma omp parallel for schedule(dynamic, 64)
  for (long long c = 0; c < nc; ++c) {
    const long long cx = c / ((long long)ty * tz), cy = (c / tz) % ty, cz = c % tz;
    const long long size = (out_ptr[c + 1] - out_ptr[c]) / components;
    int64_t* o = out_unknowns + out_ptr[c];
    long long s = 0;
    for (long long k = loz[cz]; k <= hiz[cz]; ++k)
      for (long long j = loy[cy]; j <= hiy[cy]; ++j)
        for (long long i = lox[cx]; i <= hix[cx]; ++i, ++s) {
          const long long v = i + nx * (j + (long long)ny * k);
          for (int q = 0; q < components; ++q) o[q * size + s] = v + q * nv;
        }
  }
  return SGF_OK;
}

uint64_t sgf_kernel_launches(void) { return g_kernel_launches; }

int sgf_profile_enable(int on) {
  g_prof.reset();
  g_prof.on = on != 0;
  return SGF_OK;
}

int sgf_profile_read(double* out, int cap) {
  if (!out || cap < 3 * PROF_NCLS) return SGF_INVALID_ARG;
  g_prof.read(out);
  return SGF_OK;
}

int sgf_csr_create(sgf_ctx* ctx, int64_t n, int64_t nnz, const int64_t* indptr, const int32_t* indices,
                   const double* values, int on_device, sgf_csr** out) {
  if (!ctx || !out) return SGF_INVALID_ARG;
  *out = nullptr;
  return guarded(ctx, [&] {
    if (n > INT32_MAX) fail(SGF_INVALID_ARG, "n exceeds int32");
    sgf_csr* A = new sgf_csr();
    A->ctx = ctx;
    A->a.ctx = &ctx->c;
    A->a.mem.set_stream(ctx->c.stream);
    A->a.n = n;
    A->a.nnz = nnz;
    cudaStream_t st = ctx->c.stream;
    A->a.rp = A->a.mem.alloc_t<long long>(n + 1);
    A->a.ci = A->a.mem.alloc_t<int>(std::max<int64_t>(nnz, 1));
    A->a.v = A->a.mem.alloc(std::max<int64_t>(nnz, 1));
    if (on_device) {
      SGF_CUDA(cudaMemcpyAsync(A->a.rp, indptr, (n + 1) * 8, cudaMemcpyDeviceToDevice, st));
      SGF_CUDA(cudaMemcpyAsync(A->a.ci, indices, nnz * 4, cudaMemcpyDeviceToDevice, st));
      SGF_CUDA(cudaMemcpyAsync(A->a.v, values, nnz * 8, cudaMemcpyDeviceToDevice, st));
    } else {  // host arrays: through the pinned staging ring (parallel copies, DMA overlapped)
      auto up = [&](void* dst, const void* src, size_t bytes) {
        constexpr size_t PIECE = (size_t)32 << 20;
        for (size_t o = 0; o < bytes; o += PIECE)
          stage_upload(st, (char*)dst + o, (const char*)src + o, std::min(PIECE, bytes - o));
      };
      up(A->a.rp, indptr, (size_t)(n + 1) * 8);
      up(A->a.ci, indices, (size_t)nnz * 4);
      up(A->a.v, values, (size_t)nnz * 8);
    }
    if (nnz <= (int64_t)INT32_MAX) {
      A->a.rp32 = A->a.mem.alloc_t<int>(n + 1);
      SGF_CUDA(launch_rowptr32(A->a.rp, A->a.rp32, n + 1, st));
    }
    SGF_CUDA(cudaStreamSynchronize(st));
    *out = A;
  });
}

int sgf_csr_free(sgf_csr* a) {
  if (!a) return SGF_OK;
  cudaStreamSynchronize(a->ctx->c.stream);
  delete a;
  return SGF_OK;
}

int sgf_spmv(sgf_csr* a, const double* x, double* y, int on_device) {
  if (!a) return SGF_INVALID_ARG;
  sgf_ctx* ctx = a->ctx;
  return guarded(ctx, [&] {
    cudaStream_t st = ctx->c.stream;
    const long long n = a->a.n;
    if (on_device) {
      spmv(&a->a, x, y, nullptr);
    } else {
      DevVec dx(n, st), dy(n, st);
      SGF_CUDA(cudaMemcpyAsync(dx.p, x, n * 8, cudaMemcpyHostToDevice, st));
      spmv(&a->a, dx.p, dy.p, nullptr);
      SGF_CUDA(cudaMemcpyAsync(y, dy.p, n * 8, cudaMemcpyDeviceToHost, st));
    }
    SGF_CUDA(cudaStreamSynchronize(st));
  });
}

static void run_pcg(sgf_ctx* ctx, sgf_csr* a, const MatFn& Aop, const PrecFn& M, const double* b, double* x, double tol,
                    int maxit, int true_every, int on_device, sgf_pcg_report* rep, double* history) {
  cudaStream_t st = ctx->c.stream;
  const long long n = a->a.n;
  if (on_device) {
    pcg(ctx->c, &a->a, Aop, M, b, x, tol, maxit, true_every, rep, history);
  } else {
    DevVec db(n, st), dx(n, st);
    SGF_CUDA(cudaMemcpyAsync(db.p, b, n * 8, cudaMemcpyHostToDevice, st));
    pcg(ctx->c, &a->a, Aop, M, db.p, dx.p, tol, maxit, true_every, rep, history);
    SGF_CUDA(cudaMemcpyAsync(x, dx.p, n * 8, cudaMemcpyDeviceToHost, st));
  }
  SGF_CUDA(cudaStreamSynchronize(st));
}

int sgf_pcg(sgf_ctx* ctx, sgf_csr* a, sgf_precond* p, const double* b, double* x, double tol, int maxit,
            int true_residual_every, int on_device, sgf_pcg_report* rep, double* history) {
  if (!ctx || !a || !b || !x || !rep || !history) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    if (p && p->p->n != a->a.n) fail(SGF_SHAPE, "preconditioner and matrix sizes differ");
    if ((p && p->ctx != ctx) || a->ctx != ctx) fail(SGF_INVALID_ARG, "matrix, preconditioner and solve must share a context");
    PrecFn M;
    if (p) {
      Precond* P = p->p;
      M = [P](const double* in, double* out) { apply_op(P, SGF_APPLY_INVERSE, in, out); };
    }
    run_pcg(ctx, a, MatFn(), M, b, x, tol, maxit, true_residual_every, on_device, rep, history);
  });
}

int sgf_pcg_cb(sgf_ctx* ctx, sgf_csr* a, sgf_precond_fn fn, void* user, const double* b, double* x, double tol,
               int maxit, int true_residual_every, int on_device, sgf_pcg_report* rep, double* history) {
  if (!ctx || !a || !fn || !b || !x || !rep || !history) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    if (a->ctx != ctx) fail(SGF_INVALID_ARG, "matrix and solve must share a context");
    PrecFn M = [fn, user](const double* in, double* out) {
      const int rc = fn(user, in, out);
      if (rc != 0) fail(rc > 0 && rc <= SGF_NON_SYMMETRIC ? rc : SGF_CUDA, "preconditioner callback failed");
    };
    run_pcg(ctx, a, MatFn(), M, b, x, tol, maxit, true_residual_every, on_device, rep, history);
  });
}

int sgf_pcg_ops(sgf_ctx* ctx, int64_t n, sgf_csr* a, sgf_matvec_fn mv, void* mv_user, sgf_precond* p,
                sgf_precond_fn pf, void* pf_user, const double* b, double* x, double tol, int maxit,
                int true_residual_every, int on_device, sgf_pcg_report* rep, double* history) {
  if (!ctx || (!a && !mv) || (a && mv) || (p && pf) || !b || !x || !rep || !history || n < 0) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    if (a && a->a.n != n) fail(SGF_SHAPE, "matrix and right-hand side sizes differ");
    if (p && p->p->n != n) fail(SGF_SHAPE, "preconditioner and right-hand side sizes differ");
    if ((a && a->ctx != ctx) || (p && p->ctx != ctx))
      fail(SGF_INVALID_ARG, "matrix, preconditioner and solve must share a context");
    MatFn Aop;
    if (mv)
      Aop = [mv, mv_user](const double* in, double* out) {
        const int rc = mv(mv_user, in, out);
        if (rc != 0) fail(rc > 0 && rc <= SGF_NON_SYMMETRIC ? rc : SGF_CUDA, "operator callback failed");
      };
    PrecFn M;
    if (p) {
      Precond* P = p->p;
      M = [P](const double* in, double* out) { apply_op(P, SGF_APPLY_INVERSE, in, out); };
    } else if (pf) {
      M = [pf, pf_user](const double* in, double* out) {
        const int rc = pf(pf_user, in, out);
        if (rc != 0) fail(rc > 0 && rc <= SGF_NON_SYMMETRIC ? rc : SGF_CUDA, "preconditioner callback failed");
      };
    }
    if (a) {
      run_pcg(ctx, a, Aop, M, b, x, tol, maxit, true_residual_every, on_device, rep, history);
    } else {
      // an operator callback: a matrix-less workspace owner of size n
      sgf_csr W;
      W.ctx = ctx;
      W.a.ctx = &ctx->c;
      W.a.mem.set_stream(ctx->c.stream);
      W.a.n = n;
      run_pcg(ctx, &W, Aop, M, b, x, tol, maxit, true_residual_every, on_device, rep, history);
    }
  });
}

int sgf_memcpy(sgf_ctx* ctx, void* dst, const void* src, int64_t bytes) {
  if (!ctx || bytes < 0 || (bytes && (!dst || !src))) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    if (bytes) SGF_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, ctx->c.stream));
    SGF_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int sgf_stream_wait(sgf_ctx* ctx, void* stream) {
  if (!ctx) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    if (!stream || (cudaStream_t)stream == ctx->c.stream) return;
    if (!ctx->c.order_ev) SGF_CUDA(cudaEventCreateWithFlags(&ctx->c.order_ev, cudaEventDisableTiming));
    SGF_CUDA(cudaEventRecord(ctx->c.order_ev, (cudaStream_t)stream));
    SGF_CUDA(cudaStreamWaitEvent(ctx->c.stream, ctx->c.order_ev, 0));
  });
}

int sgf_precond_shard_info(const sgf_precond* p, int64_t* n_local_factors, int64_t* n_local_unknowns,
                           int64_t* n_top) {
  if (!p) return SGF_INVALID_ARG;
  const Precond* P = p->p;
  const size_t nl = P->local_count();
  int64_t nu = 0;
  for (size_t i = 0; i < nl; ++i) nu += (int64_t)P->factors[i].idx.size();
  if (n_local_factors) *n_local_factors = (int64_t)nl;
  if (n_local_unknowns) *n_local_unknowns = nu;
  if (n_top) *n_top = (int64_t)P->top_idx.size();
  return SGF_OK;
}

int sgf_precond_shard_set(const sgf_precond* p, int which, int64_t* out, int64_t cap) {
  if (!p || !out || which < 0 || which > 1) return SGF_INVALID_ARG;
  const Precond* P = p->p;
  int64_t k = 0;
  if (which == 0) {
    for (size_t i = 0; i < P->local_count(); ++i)
      for (int64_t u : P->factors[i].idx) {
        if (k >= cap) return SGF_INVALID_ARG;
        out[k++] = u;
      }
  } else {
    if ((int64_t)P->top_idx.size() > cap) return SGF_INVALID_ARG;
    std::copy(P->top_idx.begin(), P->top_idx.end(), out);
  }
  return SGF_OK;
}

int sgf_apply_part(sgf_precond* p, int part, double* y) {
  if (!p || !y) return SGF_INVALID_ARG;
  return guarded(p->ctx, [&] { apply_part(p->p, part, y); });
}

int sgf_factor_apply(sgf_precond* p, int k, int op, double* x, int on_device) {
  if (!p || !x) return SGF_INVALID_ARG;
  sgf_ctx* ctx = p->ctx;
  return guarded(ctx, [&] {
    cudaStream_t st = ctx->c.stream;
    const long long n = p->p->n;
    if (on_device) {
      factor_apply(p->p, k, op, x);
    } else {
      DevVec d(n, st);
      SGF_CUDA(cudaMemcpyAsync(d.p, x, n * 8, cudaMemcpyHostToDevice, st));
      factor_apply(p->p, k, op, d.p);
      SGF_CUDA(cudaMemcpyAsync(x, d.p, n * 8, cudaMemcpyDeviceToHost, st));
    }
    SGF_CUDA(cudaStreamSynchronize(st));
  });
}

int sgf_potrf_batched(sgf_ctx* ctx, int batch, const int32_t* m, const double* const* A, const int32_t* lda,
                      double* const* L, const int32_t* ldl, int32_t* status, int32_t* pivot_index,
                      double* pivot_value) {
  if (!ctx || batch < 0 || (batch && (!m || !A || !lda || !L || !ldl || !status))) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    for (int b = 0; b < batch; ++b)
      if (m[b] < 0 || lda[b] < m[b] || ldl[b] < m[b]) fail(SGF_INVALID_ARG, "bad matrix size or leading dimension");
    potrf_batched(ctx->c, batch, m, A, lda, L, ldl, status, pivot_index, pivot_value);
  });
}

int sgf_trsm_batched(sgf_ctx* ctx, int batch, const int32_t* m, const int32_t* nrhs, const int32_t* mode,
                     const double* const* L, const int32_t* ldl, const double* const* B, const int32_t* ldb,
                     double* const* X, const int32_t* ldx) {
  if (!ctx || batch < 0 || (batch && (!m || !nrhs || !mode || !L || !ldl || !B || !ldb || !X || !ldx)))
    return SGF_INVALID_ARG;
  return guarded(ctx, [&] { trsm_batched(ctx->c, batch, m, nrhs, mode, L, ldl, B, ldb, X, ldx); });
}

int sgf_qrcp_batched(sgf_ctx* ctx, int batch, const int32_t* m, const int32_t* c, const double* const* A,
                     const int32_t* lda, double rank_tol, int full_q, double* const* Q, double* const* R,
                     int32_t* const* perm, int32_t* rank, int32_t* steps) {
  if (!ctx || batch < 0 || (batch && (!m || !c || !A || !lda || !Q || !R || !perm || !rank))) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    for (int b = 0; b < batch; ++b)
      if (m[b] < 0 || c[b] < 0 || lda[b] < c[b]) fail(SGF_INVALID_ARG, "bad matrix size or leading dimension");
    qrcp_batched(ctx->c, batch, m, c, A, lda, rank_tol, full_q, Q, R, perm, rank, steps);
  });
}

int sgf_gemm(sgf_ctx* ctx, int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
             double beta, double* C, int ldc) {
  if (!ctx || m < 0 || n < 0 || k < 0 || (m && n && !C)) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    if (m && n) gemm(ctx->c, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
  });
}

int sgf_exchange_accumulate(void* accum, const int32_t* idx, int64_t n, const double* packed) {
  if (!accum || n < 0 || (n && (!idx || !packed))) return SGF_INVALID_ARG;
  return guarded(nullptr, [&] { exchange_accumulate((ShardExchange*)accum, idx, n, packed); });
}

int sgf_apply_shard(sgf_precond* p, int stage, const double* x, double* y, double* top_buf, int mask) {
  if (!p || !x || !y || (!top_buf && !p->p->top_idx.empty())) return SGF_INVALID_ARG;
  return guarded(p->ctx, [&] {
    if (!p->p->sharded) fail(SGF_INVALID_ARG, "not a sharded preconditioner");
    apply_shard(p->p, stage, x, y, top_buf, mask);
    SGF_CUDA(cudaStreamSynchronize(p->ctx->c.stream));
  });
}

int sgf_vec_gather(sgf_ctx* ctx, const double* x, const int32_t* idx, double* out, int64_t n) {
  if (!ctx || n < 0 || (n && (!x || !idx || !out))) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    SGF_CUDA(launch_gather(x, idx, out, n, ctx->c.stream));
    SGF_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int sgf_vec_scatter(sgf_ctx* ctx, const double* v, const int32_t* idx, double* y, int64_t n) {
  if (!ctx || n < 0 || (n && (!v || !idx || !y))) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    SGF_CUDA(launch_scatter(v, idx, y, n, ctx->c.stream));
    SGF_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int sgf_pcg_dist(sgf_ctx* ctx, int64_t n, sgf_matvec_fn mv, void* mv_user, sgf_precond_fn pf, void* pf_user,
                 sgf_reduce_fn reduce, void* reduce_user, const double* b, double* x, double tol, int maxit,
                 int true_residual_every, sgf_pcg_report* rep, double* history) {
  if (!ctx || !mv || !reduce || !b || !x || !rep || !history || n < 0) return SGF_INVALID_ARG;
  return guarded(ctx, [&] {
    MatFn Aop = [mv, mv_user](const double* in, double* out) {
      const int rc = mv(mv_user, in, out);
      if (rc != 0) fail(rc > 0 && rc <= SGF_NON_SYMMETRIC ? rc : SGF_CUDA, "operator callback failed");
    };
    PrecFn M;
    if (pf)
      M = [pf, pf_user](const double* in, double* out) {
        const int rc = pf(pf_user, in, out);
        if (rc != 0) fail(rc > 0 && rc <= SGF_NON_SYMMETRIC ? rc : SGF_CUDA, "preconditioner callback failed");
      };
    else
      M = [ctx, n](const double* in, double* out) {
        SGF_CUDA(cudaMemcpyAsync(out, in, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->c.stream));
      };
    ReduceFn R = [reduce, reduce_user](double* v, int k) {
      if (reduce(reduce_user, v, k) != 0) fail(SGF_CUDA, "reduction callback failed");
    };
    pcg_dist(ctx->c, n, Aop, M, R, b, x, tol, maxit, true_residual_every, rep, history);
  });
}

}  // extern "C"
