// Level-synchronous driver of the hierarchical factorization (reference
// factorization.py:410-573, the paper's Alg. 4.1) on the device.
//
// Per level, host work is symbolic only (block table, neighbour lists, task
// lists); every floating-point operation runs in batched sm_100a kernels:
//   eliminations  all interiors of the level at once (they never touch each
//                 other): blocked POTRF + inverse, E = A_NB L^{-T} as one
//                 triangular DMMA GEMM, target-centric Schur GEMM with the
//                 contributors of a target block accumulated in ascending
//                 interior order (factorization.py:277-299, 485-489);
//   compressions  DAG wavefronts: a node waits for already-compressed adjacent
//                 nodes of lower id, non-adjacent compressions touch disjoint
//                 blocks, so the result equals the reference's ascending-id
//                 sequence (factorization.py:302-353, 490-519);
//   merge         one tiled copy launch per level (factorization.py:356-407);
//   final dense   one blocked POTRF (factorization.py:535-541).
// The analytic flop tally (densela.py:24-40) and the live/peak block-byte
// accounting (blockmatrix.py:25-43) are recomputed on the host in the
// reference's operation order, so the stats dict matches exactly.
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <exception>
#include <mutex>
#include <sstream>
#include <thread>

#include "precond.h"

namespace sgf {

namespace {

struct Node {
  std::vector<int64_t> active;
  double* phi = nullptr;  // device, active.size() x pi, row-major
  int kind = 0;
  bool interior = false;
};

struct LevelStats {
  int level, nodes, eliminated = 0, compressed = 0;
  std::vector<int> ranks;
};

struct State {
  Ctx* ctx;
  cudaStream_t st;
  const sgf_factor_args* a;
  int pi;
  BlockTable M;
  std::vector<Node> nodes;
  std::unique_ptr<Arena> lvl;  // blocks + phi of the current level
  Arena scratch;
  Arena persist;   // lives for the whole factorization (deferred status buffers)
  CholCheck chk;   // Cholesky breakdowns, verified at host sync points
  long long flops = 0;
  long long peak = 0;
  int comp_counter = 0;  // compressions so far (reference execution order)
  Precond* P;
  // sharding
  bool sharded = false;
  int my_rank = 0;
  std::vector<int> node_rank;  // per node of the current level: owning rank, -1 = top separator
  std::vector<std::pair<double*, long long>> regions;  // device regions holding the level's blocks
  bool l1_sym = true;          // level-1 apply through G = A_BB^{-1} and the sparse couplings
  std::vector<int> l1_bw;      // level-1 cells: lower bandwidth of the diagonal block (banded Cholesky)
  int64_t max_row_nnz = 0;     // longest CSR row (level-1 sparse elimination path when <= L1_KMAX + 1)
  int* l1_overflow = nullptr;   // device flag: a coupling row exceeded L1_KMAX (internal error)
  int oz_min_m = 1024;         // eliminations with a node this large use the INT8-emulated FP64 products (0: off)
  int oz_schur_min_m = 640;    // nodes this large (below oz_min_m) take only the Schur updates emulated
  int chol_oz_min_m = 1024;    // Cholesky/inverse of nodes this large split recursively onto those products (0: off)
  bool ekfirst = true;         // record the couplings' leading zeros for the apply (SGF_NO_EKFIRST=1: off)
  int qr_full_steps = 0;       // 1: QR past the rank as the reference does (its Q_2 is rounding-determined
                               //    there, so apply_half_inverse's dropped coordinates never match it exactly)
  std::vector<std::string> warnings;  // reference warnings.warn messages (stats "warnings", raised by Python)
  long long fa_extra = 0;      // apply flops of other ranks' factors
  int nf_extra = 0;            // number of other ranks' factors
  explicit State(cudaStream_t s) : scratch(s), persist(s, (size_t)4 << 20) { chk.arena = &persist; }
};

inline bool kind_in(int mask, int kind) { return (mask >> kind) & 1; }

// SGF_TRACE=1: per-phase wall times (stream synchronised) on stderr.
// SGF_TRACE=3: asynchronous timeline (no synchronisation): host and device
// start/end of every phase, printed at the end of the factorization.
struct Timeline {
  struct Rec {
    std::string name;
    double h0, h1;
    cudaEvent_t e0, e1;
  };
  std::vector<Rec> recs;
  std::chrono::steady_clock::time_point origin = std::chrono::steady_clock::now();
  cudaEvent_t eorigin = nullptr;
  double now() const {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - origin).count();
  }
};
Timeline* g_tl = nullptr;

struct Phase {
  const char* name;
  int level;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  int rec = -1;
  static int mode() {
    static int v = getenv("SGF_TRACE") ? atoi(getenv("SGF_TRACE")) : 0;
    return v;
  }
  static bool on() { return mode() == 1 || mode() == 2; }
  Phase(const char* n, int lv, cudaStream_t s) : name(n), level(lv), st(s) {
    if (on()) {
      cudaStreamSynchronize(st);
      t0 = std::chrono::steady_clock::now();
    } else if (mode() == 3 && g_tl) {
      Timeline::Rec r;
      r.name = std::string(n) + " L" + std::to_string(lv);
      r.h0 = g_tl->now();
      cudaEventCreate(&r.e0);
      cudaEventCreate(&r.e1);
      cudaEventRecord(r.e0, st);
      rec = (int)g_tl->recs.size();
      g_tl->recs.push_back(r);
    }
  }
  ~Phase() {
    if (rec >= 0 && g_tl) {
      cudaEventRecord(g_tl->recs[rec].e1, st);
      g_tl->recs[rec].h1 = g_tl->now();
      return;
    }
    if (!on()) return;
    cudaStreamSynchronize(st);
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[sgf] L%d %-10s %9.2f ms\n", level, name, ms);
  }
};

void timeline_begin(cudaStream_t st) {
  if (Phase::mode() != 3) return;
  g_tl = new Timeline();
  cudaEventCreate(&g_tl->eorigin);
  cudaEventRecord(g_tl->eorigin, st);
}

void timeline_end(cudaStream_t st) {
  if (!g_tl) return;
  cudaStreamSynchronize(st);
  fprintf(stderr, "[timeline] %-16s %9s %9s | %9s %9s\n", "phase", "host0", "host1", "dev0", "dev1");
  for (auto& r : g_tl->recs) {
    float d0 = 0, d1 = 0;
    cudaEventElapsedTime(&d0, g_tl->eorigin, r.e0);
    cudaEventElapsedTime(&d1, g_tl->eorigin, r.e1);
    fprintf(stderr, "[timeline] %-16s %9.2f %9.2f | %9.2f %9.2f\n", r.name.c_str(), r.h0, r.h1, d0, d1);
  }
  fprintf(stderr, "[timeline] total host %.2f ms\n", g_tl->now());
  delete g_tl;
  g_tl = nullptr;
}

// ---------------------------------------------------------------------------
// Level-1 couplings (precond.h L1Couplings): the CSR entries between the
// unknowns of the level-1 interiors this rank eliminates (rows in factor
// order) and their neighbours, in both orientations, values gathered on the
// device from the CSR values.
// ---------------------------------------------------------------------------
void build_l1_couplings(State& S, const long long* d_ip, const int* d_ix, const int* d_own, const int* d_loc,
                        const double* d_vals) {
  HostTimer ht("setup l1 couplings");
  const sgf_factor_args& a = *S.a;
  const int nc = a.level_ncells[0];
  const int64_t n = a.n;
  std::vector<char> el(nc, 0);
  std::vector<int> bstart(nc, 0);
  int maxm = 0;
  long long nb = 0;
  for (int c = 0; c < nc; ++c) {
    const int m = (int)(a.l1_ptr[c + 1] - a.l1_ptr[c]);
    bstart[c] = (int)nb;
    if (a.cell_interior[c] && m > 0 && (!S.sharded || S.node_rank[c] == S.my_rank)) {
      el[c] = 1;
      maxm = std::max(maxm, m);
      nb += m;
    }
  }
  if (maxm == 0 || maxm > 1024) {  // the symmetric kernel holds a row pair set per lane
    S.l1_sym = false;
    return;
  }
  cudaStream_t st = S.st;
  Arena& sc = S.scratch;
  const char* d_el = sc.upload(el);
  const int* d_bs = sc.upload(bstart);
  int* rows = sc.alloc_t<int>(nb + 1);
  int* bcnt = sc.alloc_t<int>(nb + 1);
  int* fcnt = sc.alloc_t<int>(n + 1);
  int* fflag = sc.alloc_t<int>(n + 1);
  SGF_CUDA(cudaMemsetAsync(bcnt + nb, 0, sizeof(int), st));
  SGF_CUDA(cudaMemsetAsync(fcnt + n, 0, sizeof(int), st));
  SGF_CUDA(cudaMemsetAsync(fflag + n, 0, sizeof(int), st));
  SGF_CUDA(l1_couplings_count(n, (int)nb, d_ip, d_ix, d_own, d_loc, d_el, d_bs, rows, bcnt, fcnt, fflag, st));
  L1Couplings& L = S.P->l1;
  Arena& store = S.P->store;
  L.nb = (int)nb;
  L.b_rp = store.alloc_t<int>(nb + 1);
  int* fscan = sc.alloc_t<int>(n + 1);
  int* fidx = sc.alloc_t<int>(n + 1);
  size_t tb = 0, t1 = 0;
  SGF_CUDA(scan_ints(bcnt, L.b_rp, nb, nullptr, &tb, st));
  SGF_CUDA(scan_ints(fcnt, fscan, n, nullptr, &t1, st));
  tb = std::max(tb, t1);
  void* temp = sc.alloc_bytes(std::max<size_t>(tb, 256));
  SGF_CUDA(scan_ints(bcnt, L.b_rp, nb, temp, &tb, st));
  SGF_CUDA(scan_ints(fcnt, fscan, n, temp, &tb, st));
  SGF_CUDA(scan_ints(fflag, fidx, n, temp, &tb, st));
  // sizes for the allocations (the device is otherwise idle here)
  int tot[3];
  SGF_CUDA(cudaMemcpyAsync(&tot[0], L.b_rp + nb, sizeof(int), cudaMemcpyDeviceToHost, st));
  SGF_CUDA(cudaMemcpyAsync(&tot[1], fscan + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  SGF_CUDA(cudaMemcpyAsync(&tot[2], fidx + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  SGF_CUDA(cudaStreamSynchronize(st));
  L.b_ci = store.alloc_t<int>(std::max(tot[0], 1));
  L.b_v = store.alloc(std::max(tot[0], 1));
  L.nf = tot[2];
  L.f_rid = store.alloc_t<int>(std::max(tot[2], 1));
  L.f_rp = store.alloc_t<int>(tot[2] + 1);
  L.f_ci = store.alloc_t<int>(std::max(tot[1], 1));
  L.f_v = store.alloc(std::max(tot[1], 1));
  SGF_CUDA(l1_couplings_fill(n, d_ip, d_ix, d_vals, d_own, d_loc, d_el, d_bs, L.b_rp, L.b_ci, L.b_v, fscan, fidx,
                             L.f_rid, L.f_rp, L.f_ci, L.f_v, L.nf, st));
  L.ready = true;
}

// ---------------------------------------------------------------------------
// level 1: nodes, basis rows, and the CSR -> block scatter (blockmatrix.py:97-144)
// ---------------------------------------------------------------------------
void setup_level1(State& S) {
  const sgf_factor_args& a = *S.a;
  const int nc = a.level_ncells[0];
  const int64_t n = a.n;
  const int pi = S.pi;
  // One pinned staging region for every level-1 upload:
  //   [indptr | indices | values | owner | local | Pi double buffer]
  // staged with parallel copies, DMA enqueued without synchronisation (a
  // helper thread staging during the block discovery was slower: it competes
  // with the OpenMP loops for cores and memory bandwidth).
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const int64_t chunk_rows = std::max<int64_t>(1, ((int64_t)64 << 20) / (pi * (int64_t)sizeof(double)));
  const size_t half = (size_t)std::min<int64_t>(chunk_rows, std::max<int64_t>(n, 1)) * pi;
  const size_t o_ip = 0, o_ix = o_ip + al((n + 1) * 8), o_v = o_ix + al(std::max<int64_t>(a.nnz, 1) * 4);
  const size_t o_own = o_v + (a.values_on_device ? 0 : al(std::max<int64_t>(a.nnz, 1) * 8));
  const size_t o_loc = o_own + al(n * 4), o_phi = o_loc + al(n * 4);
  char* pin = (char*)S.ctx->pinned(o_phi + 2 * half * sizeof(double));
  long long* d_ip = S.scratch.alloc_t<long long>(n + 1);
  int* d_ix = S.scratch.alloc_t<int>(std::max<int64_t>(a.nnz, 1));
  double* d_vhost = a.values_on_device ? nullptr : S.scratch.alloc(std::max<int64_t>(a.nnz, 1));
  int* d_own = S.scratch.alloc_t<int>(n);
  int* d_loc = S.scratch.alloc_t<int>(n);
  // owner / local live directly in their pinned upload slots (no host
  // vectors to fault in, no staging copy)
  int32_t* owner = (int32_t*)(pin + o_own);
  int32_t* local = (int32_t*)(pin + o_loc);
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < n; ++u) owner[u] = -1;
  std::vector<int> sizes(nc);
  S.nodes.assign(nc, Node());
  int bad_cover = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(| : bad_cover)
  for (int c = 0; c < nc; ++c) {
    const int64_t b = a.l1_ptr[c], e = a.l1_ptr[c + 1];
    sizes[c] = (int)(e - b);
    Node& nd = S.nodes[c];
    nd.active.assign(a.l1_unknowns + b, a.l1_unknowns + e);
    nd.kind = a.cell_kind[c];
    nd.interior = a.cell_interior[c] != 0;
    for (int64_t i = b; i < e; ++i) {
      const int64_t u = a.l1_unknowns[i];
      if (u < 0 || u >= n) { bad_cover = 1; continue; }
      owner[u] = c;  // a duplicate shows up as a hole below
      local[u] = (int32_t)(i - b);
    }
  }
  if (bad_cover || a.l1_ptr[nc] != n) fail(SGF_INVALID_ARG, "level-1 cells do not partition the unknowns");
  int hole = 0;
#pragma omp parallel for schedule(static) reduction(| : hole)
  for (int64_t u = 0; u < n; ++u) hole |= owner[u] < 0;
  if (hole) fail(SGF_INVALID_ARG, "node unknown lists do not cover all unknowns");

  // symmetry of pattern and values (blockmatrix.py:105-113) is checked on the
  // device once the CSR is uploaded (sym_check_kernel), verified at the first
  // synchronisation point before any other result; the host only needs the
  // longest row here.  Column indices are sorted per row.
  {
    Phase ph(" s-sym", -1, S.st);
    int64_t rowmax = 0;
#pragma omp parallel for reduction(max : rowmax)
    for (int64_t r = 0; r < n; ++r) rowmax = std::max<int64_t>(rowmax, a.indptr[r + 1] - a.indptr[r]);
    S.max_row_nnz = rowmax;
  }

  // block discovery, per cell (rows of a cell are its unknowns): coupled
  // cells b > a; the symmetric pattern makes the (b, a) side redundant
  HostTimer htd("setup discovery");
  std::vector<std::vector<int>> up(nc);
  std::vector<char> has_diag(nc, 0);
  S.l1_bw.assign(nc, 0);
#pragma omp parallel for schedule(dynamic, 64)
  for (int c = 0; c < nc; ++c) {
    auto& v = up[c];
    int bw = 0;  // lower bandwidth of the diagonal block in the cell's unknown order
    for (int64_t i = a.l1_ptr[c]; i < a.l1_ptr[c + 1]; ++i) {
      const int64_t r = a.l1_unknowns[i];
      for (int64_t e = a.indptr[r]; e < a.indptr[r + 1]; ++e) {
        const int cb = owner[a.indices[e]];
        if (cb == c) {
          has_diag[c] = 1;
          bw = std::max(bw, (int)(i - a.l1_ptr[c]) - local[a.indices[e]]);
        } else if (cb > c && std::find(v.begin(), v.end(), cb) == v.end()) {
          v.push_back(cb);
        }
      }
    }
    S.l1_bw[c] = bw;
    std::sort(v.begin(), v.end());
  }
  HostTimer htd2("setup blocks");
  S.M.init(sizes);
  long long total = 0;
  for (int c = 0; c < nc; ++c) {
    if (has_diag[c]) total += (long long)sizes[c] * sizes[c];
    for (int b : up[c]) total += (long long)sizes[c] * sizes[b];
  }
  S.lvl.reset(new Arena(S.st));
  double* base = S.lvl->alloc(std::max<long long>(total, 1));
  SGF_CUDA(cudaMemsetAsync(base, 0, std::max<long long>(total, 1) * sizeof(double), S.st));
  S.regions.assign(1, {base, total});
  // blocks in lexicographic (a, b) order: the reference's insertion order.
  // The table inserts are DRAM-latency bound (random slots): adjacency lists
  // are sized first and every insert prefetches the slot of one 16 ahead.
  std::vector<long long> diag_off(nc, -1);
  std::vector<std::vector<long long>> up_off(nc);
  {
    std::vector<int> deg(nc, 0);
    for (int c = 0; c < nc; ++c) {
      deg[c] += (int)up[c].size();
      for (int b : up[c]) ++deg[b];
    }
#pragma omp parallel for schedule(static)
    for (int c = 0; c < nc; ++c) S.M.adj[c].reserve(deg[c]);
  }
  struct NewBlk {
    int a, b;
    long long off;
  };
  std::vector<NewBlk> nbk;
  nbk.reserve(S.M.map.size() + nc * 8);
  long long off = 0;
  for (int c = 0; c < nc; ++c) {
    if (has_diag[c]) {
      diag_off[c] = off;
      nbk.push_back({c, c, off});
      off += (long long)sizes[c] * sizes[c];
    }
    for (int b : up[c]) {
      up_off[c].push_back(off);
      nbk.push_back({c, b, off});
      off += (long long)sizes[c] * sizes[b];
    }
  }
  S.M.map.reserve(nbk.size());
  constexpr size_t PF = 16;
  for (size_t i = 0; i < nbk.size(); ++i) {
    if (i + PF < nbk.size()) S.M.map.prefetch(bkey(nbk[i + PF].a, nbk[i + PF].b));
    const NewBlk& e = nbk[i];
    S.M.insert_new(e.a, e.b, Blk{base + e.off, sizes[e.a], sizes[e.b]});
  }
  HostTimer hts("setup scatter");
  // scatter the CSR entries into the blocks on the device (entries stored
  // once, in the (min,max) orientation)
  Phase ph_dst(" s-scatter", -1, S.st);
  {
    std::vector<int> up_ptr(nc + 1, 0), up_cell;
    std::vector<long long> up_o;
    for (int c = 0; c < nc; ++c) {
      up_ptr[c + 1] = up_ptr[c] + (int)up[c].size();
      up_cell.insert(up_cell.end(), up[c].begin(), up[c].end());
      up_o.insert(up_o.end(), up_off[c].begin(), up_off[c].end());
    }
    CsrScatter P;
    {
      struct Piece {
        size_t off;
        void* dst;
        const void* src;
        size_t bytes;
      };
      std::vector<Piece> pieces = {{o_ip, d_ip, a.indptr, (size_t)(n + 1) * 8},
                                   {o_ix, d_ix, a.indices, (size_t)a.nnz * 4},
                                   {o_own, d_own, nullptr, (size_t)n * 4},   // already in place
                                   {o_loc, d_loc, nullptr, (size_t)n * 4}};
      if (d_vhost) pieces.push_back({o_v, d_vhost, a.values, (size_t)a.nnz * 8});
      constexpr size_t BLK = (size_t)1 << 20;
      for (auto& pc : pieces) {
        const long long nb = (long long)((pc.bytes + BLK - 1) / BLK);
        if (pc.src) {
#pragma omp parallel for schedule(static)
          for (long long b = 0; b < nb; ++b) {
            const size_t o = (size_t)b * BLK;
            std::memcpy(pin + pc.off + o, (const char*)pc.src + o, std::min(BLK, pc.bytes - o));
          }
        }
        if (pc.bytes) SGF_CUDA(cudaMemcpyAsync(pc.dst, pin + pc.off, pc.bytes, cudaMemcpyHostToDevice, S.st));
      }
    }
    const double* d_vals = a.values_on_device ? a.values : d_vhost;
    {
      unsigned long long* sym = S.persist.alloc_t<unsigned long long>(3);
      SGF_CUDA(cudaMemsetAsync(sym, 0, 3 * sizeof(unsigned long long), S.st));
      SGF_CUDA(launch_sym_check(n, d_ip, d_ix, d_vals, sym, S.st));
      S.chk.sym = sym;
    }
    P.indptr = d_ip;
    P.indices = d_ix;
    P.values = d_vals;
    P.owner = d_own;
    P.local = d_loc;
    P.size = S.scratch.upload(sizes);
    P.diag_off = S.scratch.upload(diag_off);
    P.up_ptr = S.scratch.upload(up_ptr);
    P.up_cell = up_cell.empty() ? d_own : S.scratch.upload(up_cell);
    P.up_off = up_o.empty() ? d_ip : S.scratch.upload(up_o);
    P.base = base;
    P.n = n;
    P.cell_rank = nullptr;
    P.my_rank = S.my_rank;
    if (S.sharded) P.cell_rank = S.scratch.upload(S.node_rank);
    SGF_CUDA(launch_csr_scatter(&P, S.st));
    if (S.l1_sym) build_l1_couplings(S, d_ip, d_ix, d_own, d_loc, d_vals);
  }

  // basis rows of every node: Pi[active] in cell order
  Phase ph_phi(" s-phi", -1, S.st);
  // rows are generated straight into the context's pinned buffer, in chunks,
  // each chunk's DMA overlapping the generation of the next
  double* d_phi = S.lvl->alloc(std::max<size_t>((size_t)n * pi, 1));
  double* hp_buf[2] = {(double*)(pin + o_phi), (double*)(pin + o_phi) + half};
  cudaEvent_t done[2] = {nullptr, nullptr};
  SGF_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  SGF_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  const int ps = a.degree == 0 ? 1 : (a.degree == 1 ? 4 : 10);
  const int64_t nv = a.n_vertices;
  auto mono = [&](int64_t v, int q) -> double {
    const double x = a.coords[3 * v], y = a.coords[3 * v + 1], z = a.coords[3 * v + 2];
    switch (q) {
      case 0: return 1.0;
      case 1: return x;
      case 2: return y;
      case 3: return z;
      case 4: return x * x;
      case 5: return y * y;
      case 6: return z * z;
      case 7: return x * y;
      case 8: return y * z;
      default: return z * x;
    }
  };
  // Pi from the coordinates (basis.py:27-62): monomials [1 x y z (x^2 y^2
  // z^2 xy yz zx)], block diagonal per component, column / max |column|
  std::vector<double> scale(ps, 1.0);
  if (!a.phi) {
    for (int q = 0; q < ps; ++q) {
      double mx = 0.0;
#pragma omp parallel for reduction(max : mx)
      for (int64_t v = 0; v < nv; ++v) mx = std::max(mx, std::fabs(mono(v, q)));
      scale[q] = (mx == 0.0) ? 1.0 : mx;
    }
  }
  int k = 0;
  for (int64_t r0 = 0; r0 < n; r0 += chunk_rows, k ^= 1) {
    const int64_t r1 = std::min<int64_t>(n, r0 + chunk_rows);
    SGF_CUDA(cudaEventSynchronize(done[k]));  // the copy that last used this half has landed
    double* hp = hp_buf[k];
    if (a.phi) {
#pragma omp parallel for
      for (int64_t i = r0; i < r1; ++i)
        std::memcpy(hp + (size_t)(i - r0) * pi, a.phi + (size_t)a.l1_unknowns[i] * pi, pi * sizeof(double));
    } else {
#pragma omp parallel for
      for (int64_t i = r0; i < r1; ++i) {
        const int64_t u = a.l1_unknowns[i];
        const int64_t c = u / nv, v = u % nv;
        double* row = hp + (size_t)(i - r0) * pi;
        for (int q = 0; q < pi; ++q) row[q] = 0.0;
        for (int q = 0; q < ps; ++q) row[c * ps + q] = mono(v, q) / scale[q];
      }
    }
    SGF_CUDA(cudaMemcpyAsync(d_phi + (size_t)r0 * pi, hp, (size_t)(r1 - r0) * pi * sizeof(double),
                             cudaMemcpyHostToDevice, S.st));
    SGF_CUDA(cudaEventRecord(done[k], S.st));
  }
  // the pinned buffer is reused only after a stream synchronisation
  // (upload_pinned); the events can go once their copies are enqueued
  cudaEventDestroy(done[0]);
  cudaEventDestroy(done[1]);
  for (int c = 0; c < nc; ++c) S.nodes[c].phi = d_phi + (size_t)a.l1_ptr[c] * pi;
}

// ---------------------------------------------------------------------------
// eliminations of one level (factorization.py:277-299)
// ---------------------------------------------------------------------------
void eliminate_level(State& S, const std::vector<int>& elim, int level) {
  if (elim.empty()) return;
  cudaStream_t st = S.st;
  BlockTable& M = S.M;
  Precond* P = S.P;
  struct EI {
    int x, m, c, ld;
    std::vector<int> nb;
    std::vector<int> off;
    double *W, *X, *E;
  };
  std::vector<EI> info(elim.size());
  // sharded: this rank computes only its own interiors; the symbolic part
  // (fill, block table, flop and byte tallies) still covers every interior
  std::vector<char> own(elim.size(), 1);
  CopyBatch cp;
  std::vector<CholJob> jobs;
  HostTimer ht0("elim setup+chol");
  size_t tot_w = 0, tot_e = 0;
  for (size_t q = 0; q < elim.size(); ++q) {
    EI& e = info[q];
    e.x = elim[q];
    e.m = M.size[e.x];
    e.nb = M.nbrs(e.x);
    e.c = 0;
    for (int j : e.nb) {
      e.off.push_back(e.c);
      e.c += M.size[j];
    }
    e.ld = pad_ld(e.m);
    if (S.sharded) own[q] = S.node_rank[e.x] == S.my_rank;
    if (!own[q]) continue;
    tot_w += (size_t)e.m * e.ld;
    tot_e += (size_t)e.c * e.ld;
  }
  // one region per kind for the whole level: L, L^{-1} (zeroed once: the
  // inverse kernel writes the lower triangle only) and the couplings E
  double* Wall = P->store.alloc(std::max<size_t>(tot_w, 1));
  double* Xall = P->store.alloc(std::max<size_t>(tot_w, 1));
  double* Eall = tot_e ? P->store.alloc(tot_e) : nullptr;
  SGF_CUDA(cudaMemsetAsync(Xall, 0, tot_w * sizeof(double), st));
  size_t ow = 0, oe = 0;
  for (size_t q = 0; q < elim.size(); ++q) {
    EI& e = info[q];
    if (!own[q]) continue;
    const size_t mm = (size_t)e.m * e.ld;
    e.W = Wall + ow;
    e.X = Xall + ow;
    ow += mm;
    e.E = e.c ? Eall + oe : nullptr;
    oe += (size_t)e.c * e.ld;
    Blk* d = M.find(e.x, e.x);
    if (!d) fail(SGF_NOT_SPD, "interior node without a diagonal block");
    // diagonal blocks are valid in their lower triangle only: copy that, zero above
    cp.add_lower(d->p, d->cols, 1, e.W, e.ld, 1, e.m);
    jobs.push_back(CholJob{e.W, e.X, e.m, e.x, e.ld});
    jobs.back().upper_zero = true;
    if (level == 1 && !S.l1_bw.empty()) jobs.back().bw = std::max(1, S.l1_bw[e.x]);
  }
  cp.launch(S.scratch, st);
  {
    HostTimer htc("elim chol_inv_batch");
    // large nodes (level 3 at 128^3) factor recursively with their products
    // on the INT8 tensor cores; the rest blocked on DMMA
    chol_inv_rec(*S.ctx, S.scratch, jobs, &S.chk, S.chol_oz_min_m);
  }
  // level 1: G = A_BB^{-1} = X^T X (X = L^{-1}), lower triangle, for the
  // apply (precond.h L1Couplings); K range of tile (i0, j0) starts at max(i0, j0)
  double* Gall = nullptr;
  const bool want_g = level == 1 && S.l1_sym && P->l1.ready;
  if (want_g && tot_w) {
    Gall = P->store.alloc(tot_w);
    GemmBatch gg;
    size_t og = 0;
    for (size_t q = 0; q < info.size(); ++q) {
      if (!own[q]) continue;
      const EI& e = info[q];
      gg.add(Gall + og, e.ld, 1, e.m, e.m, 1.0, 0.0,
             {seg(e.X, 1, e.ld, e.X, 1, e.ld, e.m, SEG_KSTART_M | SEG_KSTART_N)}, -1, true);
      og += (size_t)e.m * e.ld;
    }
    gg.launch(S.scratch, st);
  }
  HostTimer hte("elim E gemm");
  const auto elap0 = std::chrono::steady_clock::now();
  auto elap = [&](const char* what) {
    if (HostTimer::on())
      fprintf(stderr, "[host]   el %-16s %8.2f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - elap0).count());
  };
  // Large nodes take the FP64 products on the INT8 tensor cores (ozaki.cu):
  // E = A_NB X^T (X lower triangular) and the Schur updates E_a E_b^T, with
  // every operand split once.  Small nodes keep the DMMA GEMM.
  int maxm = 0;
  for (size_t qi = 0; qi < info.size(); ++qi)
    if (own[qi]) maxm = std::max(maxm, info[qi].m);
  // (int32 accumulators hold 8 pairs x K x 127^2 exactly for K < 16.6k)
  const bool use_oz = S.oz_min_m > 0 && maxm >= S.oz_min_m && maxm <= 16000;
  // mid-size nodes (level 2 at 128^3): E on DMMA (its K = m is too short for
  // the emulated product's two-pass epilogue), the Schur updates emulated
  const bool oz_schur = use_oz || (S.oz_schur_min_m > 0 && S.oz_min_m > 0 && maxm >= S.oz_schur_min_m &&
                                   maxm <= 16000);
  OzBatch oz;
  std::vector<std::vector<OzOperand>> eop(oz_schur ? info.size() : 0);
  GemmBatch ge;
  // level 1 with short matrix rows: E and the Schur updates as gathers of
  // L^{-1} and G (l1_sparse.cu); every coupling row has <= L1_KMAX nonzeros
  static const bool no_l1_sparse = getenv("SGF_NO_L1SPARSE") != nullptr;
  int maxc = 0;
  for (size_t qi = 0; qi < info.size(); ++qi)
    if (own[qi]) maxc = std::max(maxc, info[qi].c);
  const bool sparse1 =
      Gall && !oz_schur && !no_l1_sparse && S.max_row_nnz <= L1_KMAX + 1 && l1_e_fits(maxm, maxc);
  std::vector<long long> rl_base(info.size(), 0);
  std::vector<L1RowTask> l1r;
  std::vector<L1ETask> l1e;
  long long rl_rows = 0;
  if (sparse1)
    for (size_t qi = 0; qi < info.size(); ++qi)
      if (own[qi]) {
        rl_base[qi] = rl_rows;
        rl_rows += info[qi].c;
      }
  long long fl_chol = 0, fl_e = 0, fl_s = 0;
  static const bool dmma_skip = !getenv("SGF_NO_DMMA_SKIP");
  std::vector<int*> xkf(info.size(), nullptr);
  std::vector<uint32_t*> xmk(info.size(), nullptr);
  std::vector<int> xmw(info.size(), 0);
  std::vector<NzFlagJob> nzjobs;
  for (size_t qi = 0; qi < info.size(); ++qi) {
    const EI& e = info[qi];
    long long f = (long long)e.m * e.m * e.m / 3;
    OzOperand xop;
    if (use_oz && own[qi]) {
      // L^{-1}'s rows: first nonzero column and 32-column tile masks for the
      // apply (the interior's diagonal block is block-sparse, and so is its
      // inverse factor below the diagonal)
      if (S.ekfirst && e.m <= 16384) {
        const int mw = (e.m + 1023) / 1024;
        xkf[qi] = P->store.alloc_t<int>(e.m);
        xmk[qi] = P->store.alloc_t<uint32_t>((size_t)e.m * mw);
        xmw[qi] = mw;
      }
      xop = oz.split(S.scratch, e.X, e.ld, 1, e.m, e.m, false, xkf[qi], xmk[qi], xmw[qi]);
    }
    for (size_t q = 0; q < e.nb.size(); ++q) {
      const int rows = M.size[e.nb[q]];
      if (own[qi]) {
        View v = view_of(M, e.nb[q], e.x);  // A_NB: |N| x m
        if (sparse1) {
          // stored (N, B): v.cs == 1, |N| x m;  stored (B, N): v.rs == 1, m x |N|
          const bool trans = v.rs == 1 && v.cs != 1;
          l1r.push_back(L1RowTask{v.p, trans ? e.m : v.rows, trans ? v.rows : e.m, trans ? 1 : 0,
                                  rl_base[qi] + e.off[q]});
          if (q == 0) l1e.push_back(L1ETask{e.X, (long long)e.ld, e.E, (long long)e.ld, e.m, e.c, rl_base[qi]});
        } else if (use_oz) {
          OzOperand aop = oz.split(S.scratch, v.p, v.rs, v.cs, v.rows, e.m, true);  // block-sparse A_NB
          oz.add(e.E + (long long)e.off[q] * e.ld, e.ld, 1, v.rows, e.m, 0.0, {{{aop, xop}, 1.0}}, false, true);
        } else {
          GemmSeg sg = seg(v.p, v.rs, v.cs, e.X, e.ld, 1, e.m, SEG_KLIM_N);
          if (dmma_skip && e.m <= 8192) {  // block-sparse A_NB: K steps over its all-zero tiles skipped
            sg.a_nzk = (e.m + 15) / 16;
            uint8_t* fl = S.scratch.alloc_t<uint8_t>((size_t)((v.rows + 63) / 64) * sg.a_nzk);
            nzjobs.push_back(NzFlagJob{v.p, v.rs, v.cs, v.rows, e.m, fl});
            sg.a_nz = fl;
          }
          ge.add(e.E + (long long)e.off[q] * e.ld, e.ld, 1, v.rows, e.m, 1.0, 0.0, sg);
        }
      }
      f += (long long)e.m * e.m * rows;
    }
    long long fs = 0;
    for (size_t p = 0; p < e.nb.size(); ++p)
      for (size_t q = p; q < e.nb.size(); ++q) fs += 2LL * M.size[e.nb[p]] * e.m * M.size[e.nb[q]];
    S.flops += f + fs;
    if (Phase::mode()) {
      fl_chol += (long long)e.m * e.m * e.m / 3;
      fl_e += f - (long long)e.m * e.m * e.m / 3;
      fl_s += fs;
    }
  }
  elap("E products");
  static const bool zero_stats = getenv("SGF_ZERO_STATS") != nullptr;
  if (zero_stats) {  // diagnostics: all-zero 128 x 32 tiles of the A_NB operands of E
    unsigned long long* cnt = S.scratch.alloc_t<unsigned long long>(2);
    SGF_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), st));
    for (size_t qi = 0; qi < info.size(); ++qi) {
      if (!own[qi]) continue;
      for (size_t q = 0; q < info[qi].nb.size(); ++q) {
        View v = view_of(M, info[qi].nb[q], info[qi].x);
        SGF_CUDA(launch_zero_tiles(v.p, v.rs, v.cs, v.rows, v.cols, 128, 32, cnt, st));
      }
    }
    unsigned long long h[2];
    SGF_CUDA(cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, st));
    SGF_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "[sgf] L%d A_NB 128x32 tiles: %llu of %llu all zero (%.1f%%)\n", level, h[0], h[1],
            100.0 * h[0] / std::max(1ull, h[1]));
  }
  if (Phase::mode())
    fprintf(stderr, "[sgf] L%d eliminate: %zu nodes, max m %d, flops chol %.3e E %.3e schur %.3e (%s)\n", level,
            info.size(), maxm, (double)fl_chol, (double)fl_e, (double)fl_s,
            use_oz ? "int8-emulated" : (oz_schur ? "E dmma, schur int8-emulated" : "dmma"));
  if (!nzjobs.empty()) {
    std::vector<long long> tp(nzjobs.size() + 1, 0);
    for (size_t i = 0; i < nzjobs.size(); ++i)
      tp[i + 1] = tp[i] + (long long)((nzjobs[i].rows + 63) / 64) * ((nzjobs[i].cols + 15) / 16);
    ProfScope ps(st, PROF_MOVE, 0.0);
    SGF_CUDA(launch_nz_flags64(S.scratch.upload(nzjobs), S.scratch.upload(tp), (int)nzjobs.size(), tp.back(), st));
  }
  elap("nz flags");
  ge.launch(S.scratch, st);
  elap("E launch");
  int *rl_n = nullptr, *rl_k = nullptr;
  double* rl_a = nullptr;
  if (sparse1 && rl_rows > 0) {
    // the row lists outlive the level: E is formed from them on first use
    rl_n = P->store.alloc_t<int>(rl_rows);
    rl_k = P->store.alloc_t<int>(rl_rows * L1_KMAX);
    rl_a = P->store.alloc(rl_rows * L1_KMAX);
    if (!S.l1_overflow) {
      S.l1_overflow = S.persist.alloc_t<int>(1);
      SGF_CUDA(cudaMemsetAsync(S.l1_overflow, 0, sizeof(int), st));
    }
    SGF_CUDA(cudaMemsetAsync(rl_n, 0, rl_rows * sizeof(int), st));
    ProfScope ps(st, PROF_MOVE, 0.0);
    SGF_CUDA(launch_l1_rows(S.scratch.upload(l1r), (int)l1r.size(), rl_n, rl_k, rl_a, S.l1_overflow, st));
    static const bool eager = getenv("SGF_L1E_EAGER") != nullptr;
    if (eager) {
      SGF_CUDA(launch_l1_e(S.scratch.upload(l1e), (int)l1e.size(), maxm, maxc, rl_n, rl_k, rl_a, st));
    } else {
      auto& pe = P->l1e;
      pe.pending = true;
      pe.tasks = l1e;
      pe.max_m = maxm;
      pe.max_c = maxc;
      pe.rl_n = rl_n;
      pe.rl_k = rl_k;
      pe.rl_a = rl_a;
    }
  }
  if (use_oz) {
    oz.launch_splits(S.scratch, st);
    oz.launch(S.scratch, st);
  }
  if (zero_stats && tot_e) {  // diagnostics: all-zero 128 x 32 tiles of the couplings E
    unsigned long long* cnt = S.scratch.alloc_t<unsigned long long>(2);
    SGF_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), st));
    for (size_t qi = 0; qi < info.size(); ++qi) {
      if (!own[qi]) continue;
      const EI& e = info[qi];
      for (size_t q = 0; q < e.nb.size(); ++q)
        SGF_CUDA(launch_zero_tiles(e.E + (long long)e.off[q] * e.ld, e.ld, 1, M.size[e.nb[q]], e.m, 128, 32, cnt, st));
    }
    unsigned long long h[2];
    SGF_CUDA(cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, st));
    SGF_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "[sgf] L%d E 128x32 tiles: %llu of %llu all zero (%.1f%%)%s\n", level, h[0], h[1],
            100.0 * h[0] / std::max(1ull, h[1]), sparse1 ? " (level-1 E formed later: not yet written)" : "");
  }
  // per row of E, its first nonzero column (apply: the leading zeros of the
  // couplings are skipped; written by the operand split below)
  std::vector<int*> ekf(info.size(), nullptr);
  std::vector<uint32_t*> emk(info.size(), nullptr);
  int emw = 0;
  if (oz_schur) {
    // the couplings as Schur operands, one split per neighbour block
    long long tot_c = 0;
    for (size_t qi = 0; qi < info.size(); ++qi)
      if (own[qi]) tot_c += info[qi].c;
    int* kf_all = (S.ekfirst && tot_c) ? P->store.alloc_t<int>(tot_c) : nullptr;
    // row masks of the couplings' 32-column tiles (apply: all-zero tiles skipped)
    const int mw = (maxm + 1023) / 1024;
    emw = mw;
    uint32_t* mk_all = (S.ekfirst && tot_c && maxm <= 16384) ? P->store.alloc_t<uint32_t>(tot_c * mw) : nullptr;
    long long okf = 0;
    for (size_t qi = 0; qi < info.size(); ++qi) {
      if (!own[qi]) continue;
      const EI& e = info[qi];
      if (kf_all) ekf[qi] = kf_all + okf;
      if (mk_all) emk[qi] = mk_all + okf * mw;
      okf += e.c;
      // nonzero tile flags: the Schur products E_a E_b^T skip the K tiles
      // where E_a or E_b is zero (the couplings are block-sparse: 30-50% of
      // their 128 x 32 tiles are zero at levels 2-3 of 128^3)
      for (size_t q = 0; q < e.nb.size(); ++q)
        eop[qi].push_back(oz.split(S.scratch, e.E + (long long)e.off[q] * e.ld, e.ld, 1, M.size[e.nb[q]], e.m, true,
                                   kf_all ? ekf[qi] + e.off[q] : nullptr,
                                   mk_all ? emk[qi] + (long long)e.off[q] * mw : nullptr, mw));
    }
    oz.launch_splits(S.scratch, st);
    if (zero_stats && kf_all) {  // diagnostics: leading zeros of the couplings' rows
      std::vector<int> h(tot_c);
      SGF_CUDA(cudaMemcpyAsync(h.data(), kf_all, tot_c * sizeof(int), cudaMemcpyDeviceToHost, st));
      SGF_CUDA(cudaStreamSynchronize(st));
      double lead = 0, tot = 0;
      long long o = 0;
      for (size_t qi = 0; qi < info.size(); ++qi) {
        if (!own[qi]) continue;
        for (int r = 0; r < info[qi].c; ++r) lead += std::min(h[o + r], info[qi].m);
        tot += (double)info[qi].c * info[qi].m;
        o += info[qi].c;
      }
      fprintf(stderr, "[sgf] L%d E rows: %.1f%% of the entries are leading zeros\n", level, 100.0 * lead / tot);
      const bool pat = atoi(getenv("SGF_ZERO_STATS")) == 2;
      for (size_t q = 0; pat && q < eop[0].size() && eop[0][q].nz; ++q) {  // SGF_ZERO_STATS=2: first node's tiles
        const OzOperand& o = eop[0][q];
        const int nr = o.Rp / 128, nk = o.Kp / 32;
        std::vector<uint8_t> f((size_t)nr * nk);
        SGF_CUDA(cudaMemcpy(f.data(), o.nz, f.size(), cudaMemcpyDeviceToHost));
        for (int r = 0; r < nr; ++r) {
          std::string line;
          for (int k = 0; k < nk; ++k) line += f[(size_t)r * nk + k] ? '#' : '.';
          fprintf(stderr, "[sgf] L%d nb %zu rt %d %s\n", level, q, r, line.c_str());
        }
      }
    }
  }

  // Schur targets in the reference's insertion order (ascending interior id,
  // neighbour pairs a <= b); a target first seen without a block is a fill,
  // created zero (blockmatrix.py:65-72) when its first contributor runs
  // contributions of a target: a list threaded through one flat array (in
  // ascending interior order; no per-target heap allocation)
  struct Contrib {
    int q, p, r, next;
  };
  struct Target {
    int a, b;
    int q0;                 // first contributing interior (creation point of a fill)
    long long fill = -1;    // offset in the fill region, -1: existing block
    int head = -1, tail = -1, count = 0;
  };
  elap("schur splits");
  HostTimer ht1("elim targets");
  std::vector<Target> targets;
  std::vector<Contrib> cbuf;
  std::vector<int> fills;  // target ids of fills, in creation order
  long long fill_elems = 0;
  {
    size_t pairs = 0;
    for (auto& e : info) pairs += e.nb.size() * (e.nb.size() + 1) / 2;
    FlatMap<int> tix(pairs / 2 + 16);
    targets.reserve(pairs / 2 + 16);
    cbuf.reserve(pairs);
    for (size_t q = 0; q < info.size(); ++q) {
      const EI& e = info[q];
      for (size_t p = 0; p < e.nb.size(); ++p)
        for (size_t r = p; r < e.nb.size(); ++r) {
          const int A = e.nb[p], B = e.nb[r];
          auto ins = tix.emplace(bkey(A, B));
          if (ins.second) {
            *ins.first = (int)targets.size();
            targets.push_back(Target{A, B, (int)q, -1});
            if (!M.find(A, B)) {
              targets.back().fill = fill_elems;
              fills.push_back(*ins.first);
              fill_elems += (long long)M.size[A] * M.size[B];
            }
          }
          if (own[q]) {
            Target& T = targets[*ins.first];
            const int ci = (int)cbuf.size();
            cbuf.push_back(Contrib{(int)q, (int)p, (int)r, -1});
            if (T.tail >= 0) cbuf[T.tail].next = ci;
            else T.head = ci;
            T.tail = ci;
            ++T.count;
          }
        }
    }
  }
  double* fill_base = nullptr;
  if (fill_elems > 0) {
    fill_base = S.lvl->alloc(fill_elems);
    SGF_CUDA(cudaMemsetAsync(fill_base, 0, fill_elems * sizeof(double), st));
    S.regions.push_back({fill_base, fill_elems});
  }
  // Schur GEMMs first (the level's largest device work), table bookkeeping after
  {
    HostTimer ht("schur tasks");
    GemmBatch gs;
    std::vector<GemmSeg> sg;
    std::vector<L1SchurTask> l1s;
    std::vector<L1Contrib> l1c;
    for (auto& T : targets) {
      double* bp;
      int br, bc;
      if (T.fill < 0) {
        Blk* blk = M.find(T.a, T.b);  // T.a <= T.b: rows in a
        bp = blk->p;
        br = blk->rows;
        bc = blk->cols;
      } else {
        bp = fill_base + T.fill;
        br = M.size[T.a];
        bc = M.size[T.b];
      }
      if (T.count == 0) continue;  // sharded: no contributor on this rank
      if (sparse1) {
        const int c0 = (int)l1c.size();
        for (int ci = T.head; ci >= 0; ci = cbuf[ci].next) {
          const Contrib& c = cbuf[ci];
          const EI& e = info[c.q];
          l1c.push_back(L1Contrib{rl_base[c.q] + e.off[c.p], rl_base[c.q] + e.off[c.r], Gall + (e.X - Xall),
                                  (long long)e.ld});
        }
        for (int r0 = 0; r0 < br; r0 += 64)
          l1s.push_back(L1SchurTask{bp, (long long)bc, r0, br, bc, T.a == T.b, c0, T.count});
        continue;
      }
      sg.clear();
      for (int ci = T.head; ci >= 0; ci = cbuf[ci].next) {
        const Contrib& c = cbuf[ci];
        const EI& e = info[c.q];
        sg.push_back(seg(e.E + (long long)e.off[c.p] * e.ld, e.ld, 1, e.E + (long long)e.off[c.r] * e.ld, e.ld, 1, e.m));
      }
      // diagonal blocks are kept valid in their lower triangle only: every
      // consumer (Cholesky of the node, densify + Cholesky) reads only that
      if (oz_schur) {
        std::vector<std::pair<std::pair<OzOperand, OzOperand>, double>> terms;
        for (int ci = T.head; ci >= 0; ci = cbuf[ci].next)
          terms.push_back({{eop[cbuf[ci].q][cbuf[ci].p], eop[cbuf[ci].q][cbuf[ci].r]}, -1.0});
        oz.add(bp, bc, 1, br, bc, 1.0, terms, T.a == T.b, false);
      } else {
        gs.add(bp, bc, 1, br, bc, -1.0, 1.0, sg, -1, T.a == T.b);
      }
    }
    HostTimer ht2("schur launch");
    if (!l1s.empty()) {
      ProfScope ps(st, PROF_MOVE, 0.0);
      SGF_CUDA(launch_l1_schur(S.scratch.upload(l1s), (int)l1s.size(), S.scratch.upload(l1c), rl_n, rl_k, rl_a, st));
    }
    gs.launch(S.scratch, st);
    oz.launch(S.scratch, st);
  }
  {
    HostTimer ht("elim bookkeeping");
    // factor records in parallel (they read the actives, cleared only below)
    std::vector<Factor> recs(info.size());
#pragma omp parallel for schedule(dynamic, 8)
    for (size_t q = 0; q < info.size(); ++q) {
      if (!own[q]) continue;
      const EI& e = info[q];
      Factor& f = recs[q];
      f.type = SGF_FACTOR_ELIMINATION;
      f.node = e.x;
      f.level = level;
      f.m = e.m;
      f.ld = e.ld;
      f.c = e.c;
      f.idx = S.nodes[e.x].active;
      f.nidx.reserve(e.c);
      for (int j : e.nb) f.nidx.insert(f.nidx.end(), S.nodes[j].active.begin(), S.nodes[j].active.end());
      f.L = e.W;
      f.inv = e.X;
      f.E = e.E;
      f.ekfirst = ekf[q];
      f.emask = emk[q];
      f.emw = emk[q] ? emw : 0;
      f.xkfirst = xkf[q];
      f.xmask = xmk[q];
      f.xmw = xmw[q];
      if (Gall) f.G = Gall + (e.X - Xall);
      if (level == 1 && !S.l1_bw.empty()) f.bw = std::max(1, S.l1_bw[e.x]);
    }
    // replay the reference sequence for the table and its byte accounting:
    // interior q creates the fills it touches first, then is dropped
    size_t fi = 0;
    for (size_t q = 0; q < info.size(); ++q) {
      const EI& e = info[q];
      for (; fi < fills.size() && targets[fills[fi]].q0 == (int)q; ++fi) {
        const Target& T = targets[fills[fi]];
        M.insert(T.a, T.b, Blk{fill_base + T.fill, M.size[T.a], M.size[T.b]});
      }
      // factor record (before the node's actives are cleared)
      if (own[q]) {
        P->factors.push_back(std::move(recs[q]));
      } else {  // another rank's factor: kept only in the tallies
        S.fa_extra += 4LL * e.m * e.m + 4LL * e.m * e.c;
        ++S.nf_extra;
      }
      M.drop(e.x);
      M.size[e.x] = 0;
      S.nodes[e.x].active.clear();
      S.nodes[e.x].phi = nullptr;
    }
  }
}

// ---------------------------------------------------------------------------
// compressions of one level in DAG wavefronts (factorization.py:302-353)
// ---------------------------------------------------------------------------
struct CompOut {
  int node;
  Factor f;
  int rank;
};

// per compressed node, prepared for the whole level before the wavefronts:
// the node's diagonal block and basis rows do not change until its own
// compression, so every Cholesky + inverse and L^T Phi runs in one batch
struct CompPre {
  double *L, *X, *LP;
  int ld;
};

void compress_wave(State& S, const std::vector<int>& wave, const std::vector<int>& seqno,
                   const std::vector<int>& forced, int level, std::vector<CompOut>& out,
                   std::unordered_map<int, CompPre>& pre) {
  HostTimer htpre("c-wave total host");
  const auto lap0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (HostTimer::on())
      fprintf(stderr, "[host]   cw %-16s %8.2f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - lap0).count());
  };
  cudaStream_t st = S.st;
  BlockTable& M = S.M;
  Precond* P = S.P;
  const sgf_factor_args& a = *S.a;
  const int pi = S.pi;
  const bool lowrank = a.mode == SGF_MODE_LOWRANK;
  struct CI {
    int c, m, cN, ld;
    std::vector<int> nb;
    std::vector<char> raw;
    std::vector<int> col;  // column offset in N of each neighbour's block
    double *L, *X, *LP, *N, *tau, *nrm2, *ref2;
    int* perm;
    std::vector<double*> Z;
  };
  const int nw = (int)wave.size();
  std::vector<CI> ci(nw);
  for (int w = 0; w < nw; ++w) {
    CI& c = ci[w];
    c.c = wave[w];
    c.m = M.size[c.c];
    c.nb = M.nbrs(c.c);
    c.cN = lowrank ? 0 : pi;
    for (int j : c.nb) {
      const bool raw = lowrank || kind_in(a.raw_kind_mask, S.nodes[j].kind);
      c.raw.push_back(raw);
      c.col.push_back(c.cN);
      c.cN += raw ? M.size[j] : pi;
    }
    const CompPre& pr = pre.at(c.c);
    c.L = pr.L;
    c.X = pr.X;
    c.LP = pr.LP;
    c.ld = pr.ld;
    c.N = S.scratch.alloc((size_t)c.m * std::max(c.cN, 1));
    const int kmax = std::max(std::min(c.m, c.cN), 1);
    c.tau = S.scratch.alloc(kmax);
    c.nrm2 = S.scratch.alloc(std::max(c.cN, 1));
    c.ref2 = S.scratch.alloc(std::max(c.cN, 1));
    c.perm = S.scratch.alloc_t<int>(std::max(c.cN, 1));
  }

  lap("setup");
  // the filtered products M_BN Phi_N
  GemmBatch g1;
  for (auto& c : ci) {
    c.Z.assign(c.nb.size(), nullptr);
    for (size_t q = 0; q < c.nb.size(); ++q) {
      if (c.raw[q]) continue;
      View v = view_of(M, c.c, c.nb[q]);  // m x |N|
      c.Z[q] = S.scratch.alloc((size_t)c.m * pi);
      g1.add(c.Z[q], pi, 1, c.m, pi, 1.0, 0.0, {seg(v.p, v.rs, v.cs, S.nodes[c.nb[q]].phi, 1, pi, v.cols)});
    }
  }
  g1.launch(S.scratch, st);
  lap("g1");
  // assemble N (column major): [L^T Phi_B | L^{-1} M_BN Phi_N or L^{-1} M_BN]
  GemmBatch g2;
  CopyBatch cn;
  for (auto& c : ci) {
    if (!lowrank) cn.add(c.LP, pi, 1, c.N, 1, c.m, c.m, pi);
    for (size_t q = 0; q < c.nb.size(); ++q) {
      double* dstc = c.N + (long long)c.col[q] * c.m;
      if (c.raw[q]) {
        View v = view_of(M, c.c, c.nb[q]);
        g2.add(dstc, 1, c.m, c.m, v.cols, 1.0, 0.0, {seg(c.X, c.ld, 1, v.p, v.cs, v.rs, c.m, SEG_KLIM_M)});
      } else {
        g2.add(dstc, 1, c.m, c.m, pi, 1.0, 0.0, {seg(c.X, c.ld, 1, c.Z[q], 1, pi, c.m, SEG_KLIM_M)});
      }
    }
  }
  cn.launch(S.scratch, st);
  g2.launch(S.scratch, st);
  lap("g2");

  // pivoted QR (truncated at the rank), ranks read back
  std::vector<QrTask> qt(nw);
  int* d_out = S.scratch.alloc_t<int>(2 * nw);
  int max_m = 1, max_c = 1;
  for (int w = 0; w < nw; ++w) {
    CI& c = ci[w];
    QrTask& t = qt[w];
    t.Nm = c.N;
    t.tau = c.tau;
    t.nrm2 = c.nrm2;
    t.ref2 = c.ref2;
    t.perm = c.perm;
    t.replay = nullptr;
    t.nreplay = 0;
    if (a.replay_ptr && seqno[w] < a.n_replay) {
      const int64_t b = a.replay_ptr[seqno[w]], e = a.replay_ptr[seqno[w] + 1];
      std::vector<int> rp(a.replay_perm + b, a.replay_perm + e);
      t.replay = S.scratch.upload(rp);
      t.nreplay = (int)rp.size();
    }
    t.m = c.m;
    t.c = c.cN;
    t.forced_rank = lowrank ? forced[w] : -1;
    t.full_steps = S.qr_full_steps;
    t.tol = a.rank_tol;
    t.out_rank = d_out + w;
    t.out_steps = d_out + nw + w;
    t.tmp = S.scratch.alloc((size_t)std::max(c.m, 1) * std::max(c.cN, 1));
    max_m = std::max(max_m, c.m);
    max_c = std::max(max_c, c.cN);
  }
  {
    QrTask* d_qt = S.scratch.upload(qt);
    ProfScope ps(st, PROF_QR, 0.0);
    SGF_CUDA(launch_qrcp(d_qt, nw, max_m, st, max_c));
  }
  lap("qr launched");
  std::vector<int> rs(2 * nw);
  {
    HostTimer htw("c-wave rank wait");  // (the copy to pageable memory waits for the stream)
    SGF_CUDA(cudaMemcpyAsync(rs.data(), d_out, 2 * nw * sizeof(int), cudaMemcpyDeviceToHost, st));
    SGF_CUDA(cudaStreamSynchronize(st));
  }
  HostTimer htp("c-wave post-rank host");
  S.chk.verify(st);  // a breakdown upstream must surface before ranks are used
  if (Phase::mode() == 1) {
    long long sm = 0, sc = 0, ss = 0;
    for (int w = 0; w < nw; ++w) sm += ci[w].m, sc += ci[w].cN, ss += rs[nw + w];
    fprintf(stderr, "[sgf] L%d wave: %d nodes, max m %d, max cols %d, mean m %.0f cols %.0f steps %.1f\n", level, nw,
            max_m, max_c, (double)sm / nw, (double)sc / nw, (double)ss / nw);
  }

  // reflectors V and the compact-WY T (Q = H_0...H_{s-1} = I - V T V^T)
  std::vector<QrFinishTask> ft(nw);
  std::vector<double*> V(nw), Tw(nw), G(nw);
  GemmBatch gg;
  for (int w = 0; w < nw; ++w) {
    CI& c = ci[w];
    const int s = rs[nw + w];
    V[w] = s ? P->store.alloc((size_t)c.m * s) : nullptr;
    Tw[w] = s ? P->store.alloc((size_t)s * s) : nullptr;
    G[w] = s ? S.scratch.alloc((size_t)s * s) : nullptr;
    QrFinishTask& f = ft[w];
    f.Nm = c.N;
    f.tau = c.tau;
    f.steps = d_out + nw + w;
    f.rank = d_out + w;
    f.V = V[w];
    f.Tm = Tw[w];
    f.Q1 = nullptr;
    f.G = G[w];
    f.m = c.m;
    if (s) gg.add(G[w], s, 1, s, s, 1.0, 0.0, {seg(V[w], c.m, 1, V[w], c.m, 1, c.m)});
  }
  {
    QrFinishTask* d_ft = S.scratch.upload(ft);
    ProfScope ps(st, PROF_QR, 0.0);
    SGF_CUDA(launch_qr_finish(d_ft, nw, 0, st));
    gg.launch(S.scratch, st);
    int max_s = 1;
    for (int w = 0; w < nw; ++w) max_s = std::max(max_s, rs[nw + w]);
    SGF_CUDA(launch_qr_finish(d_ft, nw, 1, st, max_s));
  }
  // inv = Q^T L^{-1} = L^{-1} - V T^T (V^T L^{-1}) and the basis update
  // Q1^T L^T Phi = first r rows of (L^T Phi - V T^T (V^T L^T Phi))
  std::vector<double*> inv(nw), Y(nw), Y2(nw), Zp(nw), Zp2(nw);
  std::vector<double*> newphi(nw, nullptr);
  CopyBatch ci0;
  GemmBatch gy, gy2, gin;
  for (int w = 0; w < nw; ++w) {
    CI& c = ci[w];
    const int r = rs[w], s = rs[nw + w];
    inv[w] = P->store.alloc((size_t)c.m * c.ld);
    ci0.add(c.X, c.ld, 1, inv[w], c.ld, 1, c.m, c.m);
    if (r > 0) {
      newphi[w] = S.lvl->alloc((size_t)r * pi);
      ci0.add(c.LP, pi, 1, newphi[w], pi, 1, r, pi);
    }
    if (!s) continue;
    Y[w] = S.scratch.alloc((size_t)s * c.m);
    Y2[w] = S.scratch.alloc((size_t)s * c.m);
    Zp[w] = S.scratch.alloc((size_t)s * pi);
    Zp2[w] = S.scratch.alloc((size_t)s * pi);
    gy.add(Y[w], c.m, 1, s, c.m, 1.0, 0.0, {seg(V[w], c.m, 1, c.X, 1, c.ld, c.m, SEG_KSTART_N)});
    gy.add(Zp[w], pi, 1, s, pi, 1.0, 0.0, {seg(V[w], c.m, 1, c.LP, 1, pi, c.m)});
    gy2.add(Y2[w], c.m, 1, s, c.m, 1.0, 0.0, {seg(Tw[w], 1, s, Y[w], 1, c.m, s, SEG_KLIM_M)});
    gy2.add(Zp2[w], pi, 1, s, pi, 1.0, 0.0, {seg(Tw[w], 1, s, Zp[w], 1, pi, s, SEG_KLIM_M)});
    gin.add(inv[w], c.ld, 1, c.m, c.m, -1.0, 1.0, {seg(V[w], 1, c.m, Y2[w], 1, c.m, s)});
    if (r > 0) gin.add(newphi[w], pi, 1, r, pi, -1.0, 1.0, {seg(V[w], 1, c.m, Zp2[w], 1, pi, s)});
  }
  ci0.launch(S.scratch, st);
  gy.launch(S.scratch, st);
  gy2.launch(S.scratch, st);
  gin.launch(S.scratch, st);

  // new couplings Q1^T L^{-1} M_BN (rows of inv), identity diagonal
  GemmBatch gn;
  std::vector<double*> id_ptr;
  std::vector<int> id_sz;
  std::vector<std::vector<Blk>> newblk(nw);
  for (int w = 0; w < nw; ++w) {
    CI& c = ci[w];
    const int r = rs[w];
    if (r <= 0) continue;
    for (size_t q = 0; q < c.nb.size(); ++q) {
      const int j = c.nb[q];
      View v = view_of(M, c.c, j);  // m x |N|
      const int nj = v.cols;
      double* p = S.lvl->alloc((size_t)r * nj);
      if (c.c < j) {
        newblk[w].push_back(Blk{p, r, nj});
        gn.add(p, nj, 1, r, nj, 1.0, 0.0, {seg(inv[w], c.ld, 1, v.p, v.cs, v.rs, c.m)});
      } else {
        newblk[w].push_back(Blk{p, nj, r});
        gn.add(p, 1, r, r, nj, 1.0, 0.0, {seg(inv[w], c.ld, 1, v.p, v.cs, v.rs, c.m)});
      }
    }
    double* I = S.lvl->alloc((size_t)r * r);
    id_ptr.push_back(I);
    id_sz.push_back(r);
    newblk[w].push_back(Blk{I, r, r});  // last: diagonal
  }
  gn.launch(S.scratch, st);
  if (!id_ptr.empty()) {
    double** d_p = S.scratch.upload(id_ptr);
    int* d_s = S.scratch.upload(id_sz);
    SGF_CUDA(launch_fill_identity(d_p, d_s, (int)id_ptr.size(), st));
  }
  // QR permutations (information / parity): kept on the device and read
  // back once at the end of the factorization (no per-wave synchronisation)
  std::vector<int*> perm_dev(nw, nullptr);
  for (int w = 0; w < nw; ++w)
    if (ci[w].cN > 0) {
      perm_dev[w] = S.persist.alloc_t<int>(ci[w].cN);
      SGF_CUDA(cudaMemcpyAsync(perm_dev[w], ci[w].perm, ci[w].cN * sizeof(int), cudaMemcpyDeviceToDevice, st));
    }

  // host structure updates and factor records
  for (int w = 0; w < nw; ++w) {
    CI& c = ci[w];
    const int r = rs[w], s = rs[nw + w];
    long long f = (long long)c.m * c.m * c.m / 3;
    for (int j : c.nb) f += (long long)c.m * c.m * M.size[j];
    f += 2LL * c.m * c.m * pi;
    for (size_t q = 0; q < c.nb.size(); ++q)
      if (!lowrank && !c.raw[q]) f += 2LL * c.m * M.size[c.nb[q]] * pi;
    f += 2LL * c.m * c.cN * c.cN;
    for (int j : c.nb) f += 2LL * r * c.m * M.size[j];
    f += 2LL * r * c.m * pi;
    S.flops += f;

    CompOut o;
    o.node = c.c;
    o.rank = r;
    o.f.type = SGF_FACTOR_COMPRESSION;
    o.f.node = c.c;
    o.f.level = level;
    o.f.m = c.m;
    o.f.ld = c.ld;
    o.f.r = r;
    o.f.steps = s;
    o.f.idx = S.nodes[c.c].active;
    o.f.L = c.L;
    o.f.inv = inv[w];
    o.f.V = V[w];
    o.f.Tw = Tw[w];
    o.f.perm_dev = perm_dev[w];
    o.f.ncols = c.cN;
    out.push_back(std::move(o));

    M.drop(c.c);
    M.size[c.c] = r;
    if (r > 0) {
      M.insert(c.c, c.c, newblk[w].back());
      for (size_t q = 0; q < c.nb.size(); ++q) M.insert(c.c, c.nb[q], newblk[w][q]);
    }
    S.nodes[c.c].active.resize(r);
    S.nodes[c.c].phi = newphi[w];
  }
}

void compress_level(State& S, const std::vector<int>& comp, int level, LevelStats& ls) {
  if (comp.empty()) return;
  const sgf_factor_args& a = *S.a;
  BlockTable& M = S.M;
  const int nc = (int)comp.size();
  // rank-trace replay checks in reference order (factorization.py:492-509)
  std::vector<int> forced(nc, -1);
  if (a.mode == SGF_MODE_LOWRANK) {
    for (int i = 0; i < nc; ++i) {
      const int k = S.comp_counter + i;
      char buf[256];
      if (k >= a.n_trace) {
        snprintf(buf, sizeof buf, "rank trace exhausted; structural divergence at level %d, node %d", level,
                 comp[i]);
        fail(SGF_TRACE, buf);
      }
      const int lv = a.trace[3 * k], nd = a.trace[3 * k + 1], r = a.trace[3 * k + 2];
      if (lv != level || nd != comp[i]) {
        snprintf(buf, sizeof buf, "rank trace divergence: expected [%d, %d], reached [%d, %d]", lv, nd, level,
                 comp[i]);
        fail(SGF_TRACE, buf);
      }
      forced[i] = r;
    }
  }
  std::unordered_map<int, int> pos;
  for (int i = 0; i < nc; ++i) pos[comp[i]] = i;
  std::vector<int> wv(nc, 0);
  int nwaves = 0;
  for (int i = 0; i < nc; ++i) {
    int w = 0;
    for (int b : M.adj[comp[i]]) {
      auto it = pos.find(b);
      if (it != pos.end() && it->second < i) w = std::max(w, wv[it->second] + 1);
    }
    wv[i] = w;
    nwaves = std::max(nwaves, w + 1);
  }
  // Cholesky + inverse of every compressed node's diagonal block and L^T Phi,
  // one batch for the level (factorization.py:317, 320)
  std::unordered_map<int, CompPre> pre;
  {
    cudaStream_t st = S.st;
    const int pi = S.pi;
    CopyBatch cp;
    GemmBatch glp;
    std::vector<CholJob> jobs;
    for (int c : comp) {
      const int m = M.size[c];
      CompPre p;
      p.ld = pad_ld(m);
      const size_t mm = (size_t)m * p.ld;
      p.L = S.P->store.alloc(mm);
      p.X = S.P->store.alloc(mm);
      SGF_CUDA(cudaMemsetAsync(p.X, 0, mm * sizeof(double), st));
      p.LP = S.lvl->alloc((size_t)m * pi);
      Blk* d = M.find(c, c);
      if (!d) fail(SGF_NOT_SPD, "compressed node without a diagonal block");
      cp.add_lower(d->p, d->cols, 1, p.L, p.ld, 1, m);
      jobs.push_back(CholJob{p.L, p.X, m, c, p.ld});
      jobs.back().upper_zero = true;
      pre[c] = p;
    }
    cp.launch(S.scratch, st);
    chol_inv_batch(*S.ctx, S.scratch, jobs, &S.chk);
    for (int c : comp) {
      const CompPre& p = pre[c];
      const int m = M.size[c];
      glp.add(p.LP, pi, 1, m, pi, 1.0, 0.0, {seg(p.L, 1, p.ld, S.nodes[c].phi, 1, pi, m, SEG_KSTART_M)});
    }
    glp.launch(S.scratch, st);
  }
  std::vector<CompOut> outs;
  for (int w = 0; w < nwaves; ++w) {
    std::vector<int> nodes, seqno, fr;
    for (int i = 0; i < nc; ++i)
      if (wv[i] == w) {
        nodes.push_back(comp[i]);
        seqno.push_back(S.comp_counter + i);
        int r = forced[i];
        if (r > M.size[comp[i]]) {
          S.warnings.push_back("forced rank " + std::to_string(r) + " exceeds node size " +
                               std::to_string(M.size[comp[i]]) + "; clipping");
          r = M.size[comp[i]];
        }
        fr.push_back(r);
      }
    {
      Phase ph(" c-wave", w, S.st);
      compress_wave(S, nodes, seqno, fr, level, outs, pre);
    }
    S.scratch.release();
  }
  std::sort(outs.begin(), outs.end(), [](const CompOut& x, const CompOut& y) { return x.node < y.node; });
  for (auto& o : outs) {
    S.P->trace.push_back(level);
    S.P->trace.push_back(o.node);
    S.P->trace.push_back(o.rank);
    ls.ranks.push_back(o.rank);
    ls.compressed++;
    S.P->factors.push_back(std::move(o.f));
  }
  S.comp_counter += nc;
}

// ---------------------------------------------------------------------------
// merge into the next level (factorization.py:356-407)
// ---------------------------------------------------------------------------
void merge_level(State& S, const int64_t* father, int next_nc, const int8_t* kinds, const int8_t* interior) {
  HostTimer ht("merge");
  cudaStream_t st = S.st;
  BlockTable& M = S.M;
  const int nc = (int)S.nodes.size();
  const int pi = S.pi;
  std::vector<std::vector<int>> kids(next_nc);
  for (int c = 0; c < nc; ++c) {
    const int64_t f = father[c];
    if (f < 0 || f >= next_nc) fail(SGF_INVALID_ARG, "bad father map");
    kids[f].push_back(c);
  }
  std::vector<int> fof(nc), oof(nc), nsize(next_nc, 0);
  std::vector<Node> nn(next_nc);
  long long phi_rows = 0;
  for (int f = 0; f < next_nc; ++f) {
    int pos = 0;
    for (int c : kids[f]) {  // ascending child id
      fof[c] = f;
      oof[c] = pos;
      pos += (int)S.nodes[c].active.size();
      nn[f].active.insert(nn[f].active.end(), S.nodes[c].active.begin(), S.nodes[c].active.end());
    }
    nsize[f] = pos;
    nn[f].kind = kinds[f];
    nn[f].interior = interior[f] != 0;
    phi_rows += pos;
  }
  std::unique_ptr<Arena> nl(new Arena(st));
  CopyBatch cp;
  double* phi = nl->alloc(std::max<long long>(phi_rows * pi, 1));
  {
    long long off = 0;
    for (int f = 0; f < next_nc; ++f) {
      nn[f].phi = phi + off * pi;
      for (int c : kids[f]) {
        const int rows = (int)S.nodes[c].active.size();
        if (rows) cp.add(S.nodes[c].phi, pi, 1, phi + (off + oof[c]) * pi, pi, 1, rows, pi);
      }
      off += nsize[f];
    }
  }
  HostTimer htk("merge keys+blocks");
  // every live child block lands in its father block at the children's
  // offsets.  Father blocks are laid out in first-appearance order of a walk
  // over the table (identical on every rank of a sharded run); their order
  // does not matter otherwise: the copies hit disjoint regions, neighbour
  // lists are sorted where used, and the live/peak tally only grows here.
  struct MB {
    Blk b;
    int a0, b0;
    long long off;  // father block offset in the new level region
  };
  std::vector<MB> mbs;
  mbs.reserve(M.map.size());
  BlockTable N;
  N.init(nsize);
  std::vector<std::pair<uint64_t, long long>> order;
  FlatMap<long long> newoff(M.map.size());
  long long tot = 0;
  // live blocks in table-walk order, then the father-key inserts with the
  // slot of the insert 16 ahead prefetched (DRAM-latency bound otherwise)
  struct LiveBlk {
    Blk b;
    int a0, b0;
    uint64_t fk;
  };
  std::vector<LiveBlk> live;
  live.reserve(M.map.size());
  M.map.for_each([&](uint64_t k, Blk& b) {
    if ((long long)b.rows * b.cols == 0) return;
    const int a0 = (int)(k >> 32), b0 = (int)(k & 0xffffffffu);
    live.push_back(LiveBlk{b, a0, b0, bkey(fof[a0], fof[b0])});
  });
  constexpr size_t PF = 16;
  for (size_t i = 0; i < live.size(); ++i) {
    if (i + PF < live.size()) newoff.prefetch(live[i + PF].fk);
    const LiveBlk& L = live[i];
    auto ins = newoff.emplace(L.fk);
    if (ins.second) {
      const int fa = (int)(L.fk >> 32), fb = (int)(L.fk & 0xffffffffu);
      *ins.first = tot;
      order.push_back({L.fk, tot});
      tot += (long long)nsize[fa] * nsize[fb];
    }
    mbs.push_back(MB{L.b, L.a0, L.b0, *ins.first});
  }
  double* base = nl->alloc(std::max<long long>(tot, 1));
  if (tot) SGF_CUDA(cudaMemsetAsync(base, 0, tot * sizeof(double), st));
  S.regions.assign(1, {base, tot});
  if (S.sharded) {
    std::vector<int> nr(next_nc, -1);
    for (int f = 0; f < next_nc; ++f)
      if (!kids[f].empty()) nr[f] = S.node_rank[kids[f].front()];
    S.node_rank.swap(nr);
  }
  for (auto& o : order) {
    const int fa = (int)(o.first >> 32), fb = (int)(o.first & 0xffffffffu);
    N.insert(fa, fb, Blk{base + o.second, nsize[fa], nsize[fb]});
  }
  HostTimer htc("merge copy tasks");
  {
    const size_t nm = mbs.size();
    std::vector<size_t> pos(nm + 1, 0);
    for (size_t i = 0; i < nm; ++i)
      pos[i + 1] = pos[i] + ((fof[mbs[i].a0] == fof[mbs[i].b0] && mbs[i].a0 != mbs[i].b0) ? 2 : 1);
    const size_t base_task = cp.tasks.size();
    cp.tasks.resize(base_task + pos[nm]);
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < nm; ++i) {
      const MB& e = mbs[i];
      const Blk& b = e.b;
      const int fa = fof[e.a0], fb = fof[e.b0], oa = oof[e.a0], ob = oof[e.b0];
      CopyTask* t = &cp.tasks[base_task + pos[i]];
      double* fp = base + e.off;
      if (fa == fb) {
        const long long cols = nsize[fa];
        t[0] = CopyTask{b.p, fp + (long long)oa * cols + ob, b.cols, 1, cols, 1, b.rows, b.cols};
        if (e.a0 != e.b0) t[1] = CopyTask{b.p, fp + (long long)ob * cols + oa, 1, b.cols, cols, 1, b.cols, b.rows};
      } else if (fa < fb) {
        const long long cols = nsize[fb];
        t[0] = CopyTask{b.p, fp + (long long)oa * cols + ob, b.cols, 1, cols, 1, b.rows, b.cols};
      } else {
        const long long cols = nsize[fa];
        t[0] = CopyTask{b.p, fp + (long long)ob * cols + oa, 1, b.cols, cols, 1, b.cols, b.rows};
      }
    }
  }
  {
    Phase ph(" m-copy", -1, st);
    cp.launch(S.scratch, st);
  }
  {
    Phase ph(" m-free", -1, st);
    S.scratch.release();
    S.lvl = std::move(nl);  // frees the old level (stream ordered)
  }
  Phase ph(" m-move", -1, st);
  S.M = std::move(N);
  S.nodes = std::move(nn);
}

// ---------------------------------------------------------------------------
// final dense factor (factorization.py:535-541, blockmatrix.py:148-170)
// ---------------------------------------------------------------------------
void final_dense(State& S) {
  cudaStream_t st = S.st;
  BlockTable& M = S.M;
  std::vector<int> rem;
  for (int c = 0; c < (int)S.nodes.size(); ++c)
    if (!S.nodes[c].active.empty()) rem.push_back(c);
  if (rem.empty()) return;
  std::unordered_map<int, int> off;
  int tot = 0;
  for (int c : rem) {
    off[c] = tot;
    tot += M.size[c];
  }
  Precond* P = S.P;
  const int ldt = pad_ld(tot);
  const size_t tt = (size_t)tot * ldt;
  double* D = P->store.alloc(tt);
  double* X = P->store.alloc(tt);
  SGF_CUDA(cudaMemsetAsync(D, 0, tt * sizeof(double), st));
  SGF_CUDA(cudaMemsetAsync(X, 0, tt * sizeof(double), st));
  CopyBatch cp;
  M.map.for_each([&](uint64_t k, Blk& b) {
    const int a0 = (int)(k >> 32), b0 = (int)(k & 0xffffffffu);
    auto ia = off.find(a0), ib = off.find(b0);
    if (ia == off.end() || ib == off.end()) return;
    cp.add(b.p, b.cols, 1, D + (long long)ia->second * ldt + ib->second, ldt, 1, b.rows, b.cols);
    if (a0 != b0) cp.add(b.p, 1, b.cols, D + (long long)ib->second * ldt + ia->second, ldt, 1, b.cols, b.rows);
  });
  cp.launch(S.scratch, st);
  std::vector<CholJob> jobs{CholJob{D, X, tot, -1, ldt}};
  chol_inv_batch(*S.ctx, S.scratch, jobs, &S.chk);
  S.flops += (long long)tot * tot * tot / 3;
  Factor f;
  f.type = SGF_FACTOR_DENSE;
  f.node = -1;
  f.m = tot;
  f.ld = ldt;
  for (int c : rem) f.idx.insert(f.idx.end(), S.nodes[c].active.begin(), S.nodes[c].active.end());
  f.L = D;
  f.inv = X;
  P->factors.push_back(std::move(f));
}

// End of the sharded local phase: the live trailing-matrix blocks in key
// order (the same list on every rank: the symbolic loop is identical), the
// ones holding nonzero data on this rank (own cells' blocks, partial Schur
// sums of shared blocks; an all-zero block contributes nothing to the sum),
// packed into one device buffer for the caller's collective.
void build_exchange(State& S, ShardExchange& X) {
  cudaStream_t st = S.st;
  std::vector<std::pair<uint64_t, Blk>> blks;
  S.M.map.for_each([&](uint64_t k, Blk& b) {
    if ((long long)b.rows * b.cols > 0 && b.p) blks.push_back({k, b});
  });
  std::sort(blks.begin(), blks.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
  const int nb = (int)blks.size();
  X.st = st;
  X.ptrs.resize(nb);
  X.counts.resize(nb);
  X.total = 0;
  for (int i = 0; i < nb; ++i) {
    X.ptrs[i] = blks[i].second.p;
    X.counts[i] = (long long)blks[i].second.rows * blks[i].second.cols;
    X.total += 8 * X.counts[i];
  }
  std::vector<int> flags(std::max(nb, 1), 0);
  if (nb) {
    int* d_flags = S.scratch.alloc_t<int>(nb);
    SGF_CUDA(launch_nonzero_flags(S.scratch.upload(X.ptrs), S.scratch.upload(X.counts), nb, d_flags, st));
    SGF_CUDA(cudaMemcpyAsync(flags.data(), d_flags, nb * sizeof(int), cudaMemcpyDeviceToHost, st));
    SGF_CUDA(cudaStreamSynchronize(st));
  }
  long long off = 0;
  CopyBatch cp;
  std::vector<long long> offs;
  for (int i = 0; i < nb; ++i) {
    if (!flags[i]) continue;
    X.send_idx.push_back(i);
    const int a0 = (int)(blks[i].first >> 32), b0 = (int)(blks[i].first & 0xffffffffu);
    X.send_meta.insert(X.send_meta.end(), {a0, b0, S.node_rank[a0], S.node_rank[b0]});
    offs.push_back(off);
    off += X.counts[i];
  }
  X.send_len = off;
  X.send_buf = S.scratch.alloc(std::max<long long>(off, 1));
  // pack: every block is a contiguous row-major rows x cols matrix
  for (size_t j = 0; j < X.send_idx.size(); ++j) {
    const Blk& b = blks[X.send_idx[j]].second;
    cp.add(b.p, b.cols, 1, X.send_buf + offs[j], b.cols, 1, b.rows, b.cols);
  }
  cp.launch(S.scratch, st);
  SGF_CUDA(cudaStreamSynchronize(st));
  X.scratch = &S.scratch;
}

std::string stats_json(const sgf_factor_args& a, int64_t n, const std::vector<LevelStats>& lv, int max_after,
                       int max_seen, int final_dense, long long flops, long long flops_apply, long long peak,
                       int nfactors, const std::vector<std::string>& warnings) {
  std::ostringstream o;
  o << "{\"n\": " << n << ", \"levels\": " << lv.size() << ", \"per_level\": [";
  for (size_t i = 0; i < lv.size(); ++i) {
    if (i) o << ", ";
    o << "{\"level\": " << lv[i].level << ", \"nodes\": " << lv[i].nodes << ", \"eliminated\": " << lv[i].eliminated
      << ", \"compressed\": " << lv[i].compressed << ", \"ranks\": [";
    for (size_t k = 0; k < lv[i].ranks.size(); ++k) o << (k ? ", " : "") << lv[i].ranks[k];
    o << "]}";
  }
  o << "], \"max_node_size\": " << max_after << ", \"max_node_seen\": " << max_seen
    << ", \"final_dense_size\": " << final_dense << ", \"flops_factorize\": " << flops
    << ", \"flops_apply\": " << flops_apply << ", \"peak_blocks_bytes\": " << peak << ", \"factors\": " << nfactors
    << ", \"warnings\": [";
  for (size_t i = 0; i < warnings.size(); ++i) o << (i ? ", " : "") << "\"" << warnings[i] << "\"";
  o << "]}";
  (void)a;
  return o.str();
}

// Builds the apply plan on a worker thread, one level's factors at a time, in
// submission order.  Factors live in a deque, so the pointers handed over stay
// valid while the driver keeps appending; the worker reads only fields that are
// final when a level's function returns.  Allocation and staging go through the
// mutex-guarded chunk cache and pinned ring.
class PlanWorker {
 public:
  explicit PlanWorker(Precond* P) : P_(P) {
    SGF_CUDA(cudaGetDevice(&dev_));
    plan_init(P);
    th_ = std::thread([this] { run(); });
  }
  ~PlanWorker() { stop(); }
  void push(size_t begin, size_t end) {
    std::vector<const Factor*> fs;
    for (size_t i = begin; i < end; ++i) fs.push_back(&P_->factors[i]);
    if (fs.empty()) return;
    std::lock_guard<std::mutex> lk(mu_);
    q_.push_back({begin, std::move(fs)});
    cv_.notify_one();
  }
  // wait for every queued level; rethrows a failure of the worker
  void finish() {
    stop();
    if (err_) std::rethrow_exception(err_);
  }

 private:
  void stop() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      done_ = true;
    }
    cv_.notify_one();
    if (th_.joinable()) th_.join();
  }
  void run() {
    cudaSetDevice(dev_);
    for (;;) {
      std::pair<size_t, std::vector<const Factor*>> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return done_ || !q_.empty(); });
        if (q_.empty()) return;
        job = std::move(q_.front());
        q_.pop_front();
      }
      if (err_) continue;  // drain after a failure
      try {
        plan_extend_ptrs(P_, job.first, job.second);
      } catch (...) {
        err_ = std::current_exception();
      }
    }
  }
  Precond* P_;
  int dev_ = 0;
  std::thread th_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::pair<size_t, std::vector<const Factor*>>> q_;
  bool done_ = false;
  std::exception_ptr err_;
};

}  // namespace

void exchange_accumulate(ShardExchange* X, const int32_t* idx, int64_t n, const double* packed) {
  std::vector<double*> dst(n);
  std::vector<long long> cnt(n), offs(n);
  long long off = 0;
  for (int64_t j = 0; j < n; ++j) {
    if (idx[j] < 0 || idx[j] >= (int64_t)X->ptrs.size()) fail(SGF_INVALID_ARG, "exchange block index out of range");
    dst[j] = X->ptrs[idx[j]];
    cnt[j] = X->counts[idx[j]];
    offs[j] = off;
    off += cnt[j];
  }
  if (n) {
    Arena& sc = *X->scratch;
    SGF_CUDA(launch_add_packed(sc.upload(dst), sc.upload(cnt), sc.upload(offs), (int)n, packed, X->st));
  }
  SGF_CUDA(cudaStreamSynchronize(X->st));
}


Precond* factorize(Ctx& ctx, const sgf_factor_args& a) {
  if (a.n <= 0 || a.nlevels <= 0 || !a.indptr || !a.indices || !a.values || !a.l1_ptr || !a.l1_unknowns)
    fail(SGF_INVALID_ARG, "incomplete factorization arguments");
  if (a.pi_cols <= 0 || (!a.phi && !a.coords)) fail(SGF_INVALID_ARG, "missing polynomial basis");
  if (!a.phi) {
    const int ps = a.degree == 0 ? 1 : (a.degree == 1 ? 4 : 10);
    if (a.degree < 0 || a.degree > 2 || (a.components != 1 && a.components != 3) ||
        a.pi_cols != ps * a.components || a.n_vertices * a.components != a.n)
      fail(SGF_INVALID_ARG, "inconsistent basis description");
  }
  if (a.n > (int64_t)INT32_MAX) fail(SGF_INVALID_ARG, "n exceeds int32 index range");
  std::unique_ptr<Precond> P(new Precond());
  P->ctx = &ctx;
  P->n = a.n;
  P->store.set_stream(ctx.stream);
  State S(ctx.stream);
  S.ctx = &ctx;
  S.st = ctx.stream;
  S.a = &a;
  S.pi = a.pi_cols;
  S.P = P.get();
  const bool compression = a.compression && a.mode != SGF_MODE_EXACT;
  S.l1_sym = !getenv("SGF_NO_L1SYM") && a.nnz <= (int64_t)INT32_MAX;
  if (getenv("SGF_OZAKI_MIN_M")) S.oz_min_m = atoi(getenv("SGF_OZAKI_MIN_M"));
  if (getenv("SGF_NO_EKFIRST")) S.ekfirst = false;
  if (getenv("SGF_QR_FULL_STEPS")) S.qr_full_steps = atoi(getenv("SGF_QR_FULL_STEPS")) ? 1 : 0;
  if (getenv("SGF_OZAKI_CHOL_MIN_M")) S.chol_oz_min_m = atoi(getenv("SGF_OZAKI_CHOL_MIN_M"));
  if (getenv("SGF_OZAKI_SCHUR_MIN_M")) S.oz_schur_min_m = atoi(getenv("SGF_OZAKI_SCHUR_MIN_M"));
  if (S.oz_min_m <= 0) S.chol_oz_min_m = 0;
  PlanWorker planner(P.get());  // destroyed (joined) before P and S
  if (a.shard_count > 1) {
    if (!a.cell_rank || !a.exchange || a.shard_rank < 0 || a.shard_rank >= a.shard_count || a.shard_stop_level < 1)
      fail(SGF_INVALID_ARG, "incomplete sharding arguments");
    S.sharded = true;
    S.my_rank = a.shard_rank;
    S.node_rank.assign(a.cell_rank, a.cell_rank + a.level_ncells[0]);
    for (int r : S.node_rank)
      if (r < -1 || r >= a.shard_count) fail(SGF_INVALID_ARG, "cell rank out of range");
  }
  bool exchanged = false, stopped = false;
  // end of the local phase: record the split, sum the trailing matrix onto
  // rank 0 through the caller's collective; the other ranks stop here
  auto end_local_phase = [&]() {
    exchanged = true;
    P->sharded = true;
    P->shard_rank = S.my_rank;
    P->n_local = P->factors.size();
    for (auto& nd : S.nodes) P->top_idx.insert(P->top_idx.end(), nd.active.begin(), nd.active.end());
    ShardExchange X;
    build_exchange(S, X);
    sgf_exchange e;
    e.nblocks = (int64_t)X.ptrs.size();
    e.nsend = (int64_t)X.send_idx.size();
    e.send_idx = X.send_idx.data();
    e.send_meta = X.send_meta.data();
    e.send_buf = X.send_buf;
    e.send_len = X.send_len;
    e.accum = S.my_rank == 0 ? &X : nullptr;
    const int rc = a.exchange(a.exchange_user, &e);
    if (rc != 0) fail(SGF_CUDA, "shard exchange callback failed");
    SGF_CUDA(cudaStreamSynchronize(S.st));
    P->exchange_log.push_back({(int64_t)X.send_idx.size(), 8 * X.send_len, (int64_t)X.ptrs.size(), X.total});
    if (S.my_rank != 0) stopped = true;
    else S.sharded = false;  // rank 0 now holds the whole trailing matrix and eliminates everything
  };

  std::vector<std::pair<size_t, size_t>> plan_pend;
  auto flush_plan = [&]() {
    for (auto& r : plan_pend) planner.push(r.first, r.second);
    plan_pend.clear();
  };
  timeline_begin(S.st);
  HostTimer::epoch() = std::chrono::steady_clock::now();
  { Phase ph("setup", 0, S.st); setup_level1(S); }
  S.peak = 0;
  std::vector<LevelStats> per_level;
  int max_seen = 0, max_after = 0;
  long long cell_off = 0, father_off = 0;
  for (int t = 0; t < a.nlevels; ++t) {
    const int ncell = a.level_ncells[t];
    long long remaining = 0;
    int maxsz = 0;
    for (auto& nd : S.nodes) {
      remaining += (long long)nd.active.size();
      maxsz = std::max(maxsz, (int)nd.active.size());
    }
    if (remaining == 0) break;
    if (t > 0 && remaining < max_seen) break;
    if (ncell == 1) break;
    max_seen = std::max(max_seen, maxsz);
    LevelStats ls;
    ls.level = t + 1;
    ls.nodes = ncell;
    std::vector<int> elim;
    for (int c = 0; c < (int)S.nodes.size(); ++c)
      if (S.nodes[c].interior && !S.nodes[c].active.empty()) elim.push_back(c);
    {
      Phase ph("eliminate", t + 1, S.st);
      const size_t f0 = P->factors.size();
      eliminate_level(S, elim, t + 1);
      // the level's apply plan is built on the worker thread; handed over
      // after the merge is enqueued, so the worker's task-list staging does not
      // compete with the merge's host work (the device still has the
      // level's kernels and the merge copies queued)
      plan_pend.push_back({f0, P->factors.size()});
    }
    ls.eliminated = (int)elim.size();
    S.scratch.release();  // chunks are reused in stream order: no sync needed
    if (S.sharded && t + 1 == a.shard_stop_level) {
      end_local_phase();
      if (stopped) break;
    }
    if (compression && (t + 1) > a.skip_levels) {
      std::vector<int> comp;
      for (int c = 0; c < (int)S.nodes.size(); ++c)
        if (kind_in(a.compress_kind_mask, S.nodes[c].kind) && !S.nodes[c].active.empty()) comp.push_back(c);
      {
        Phase ph("compress", t + 1, S.st);
        const size_t f0 = P->factors.size();
        compress_level(S, comp, t + 1, ls);
        plan_pend.push_back({f0, P->factors.size()});
      }
    }
    for (auto& nd : S.nodes) max_after = std::max(max_after, (int)nd.active.size());
    per_level.push_back(ls);
    S.peak = std::max(S.peak, S.M.peak);
    if (t + 1 < a.nlevels) {
      const long long old_live = S.M.live;
      cell_off += ncell;
      Phase ph("merge", t + 1, S.st);
      merge_level(S, a.father + father_off, a.level_ncells[t + 1], a.cell_kind + cell_off,
                  a.cell_interior + cell_off);
      flush_plan();
      father_off += ncell;
      S.peak = std::max(S.peak, old_live + S.M.live);
    } else {
      break;
    }
  }
  flush_plan();
  if (S.sharded && !exchanged) end_local_phase();  // the hierarchy ended before the stop level
  size_t before = P->factors.size();
  if (!stopped) {
    Phase ph("dense", 0, S.st);
    const size_t f0 = P->factors.size();
    final_dense(S);
    planner.push(f0, P->factors.size());
  }
  int final_size = 0;
  if (P->factors.size() > before) {
    final_size = P->factors.back().m;
    S.peak = std::max(S.peak, S.M.peak);
  }
  if (!stopped && a.mode == SGF_MODE_LOWRANK && S.comp_counter < a.n_trace) {
    char buf[160];
    snprintf(buf, sizeof buf, "rank trace has %d unreplayed entries; first: [%d, %d, %d]", a.n_trace - S.comp_counter,
             a.trace[3 * S.comp_counter], a.trace[3 * S.comp_counter + 1], a.trace[3 * S.comp_counter + 2]);
    fail(SGF_TRACE, buf);
  }
  std::unique_ptr<HostTimer> ht_tail(new HostTimer("tail: verify + device drain"));
  S.chk.verify(S.st);
  SGF_CUDA(cudaStreamSynchronize(S.st));
  ht_tail.reset(new HostTimer("tail: perms, stats"));
  if (S.l1_overflow) {
    int ov = 0;
    SGF_CUDA(cudaMemcpy(&ov, S.l1_overflow, sizeof(int), cudaMemcpyDeviceToHost));
    if (ov) fail(SGF_INVALID_ARG, "internal: level-1 coupling row with more nonzeros than its CSR row");
  }
  {  // QR column permutations: asynchronous copies into one pinned buffer, one synchronisation
    size_t tot = 0;
    for (auto& f : P->factors)
      if (f.perm_dev) tot += f.ncols;
    if (tot) {
      int* hp = (int*)S.ctx->pinned(tot * sizeof(int));  // (the setup's staging buffer: idle by now)
      size_t off = 0;
      for (auto& f : P->factors)
        if (f.perm_dev) {
          SGF_CUDA(cudaMemcpyAsync(hp + off, f.perm_dev, f.ncols * sizeof(int), cudaMemcpyDeviceToHost, S.st));
          off += f.ncols;
        }
      SGF_CUDA(cudaStreamSynchronize(S.st));
      off = 0;
      for (auto& f : P->factors)
        if (f.perm_dev) {
          f.perm.assign(hp + off, hp + off + f.ncols);
          off += f.ncols;
          f.perm_dev = nullptr;
        }
    }
  }
  S.scratch.release();
  S.lvl.reset();
  long long fa = S.fa_extra;
  for (auto& f : P->factors) {
    const long long m = f.m;
    fa += (f.type == SGF_FACTOR_ELIMINATION) ? 4 * m * m + 4 * m * f.c : 4 * m * m;
  }
  // on a sharded rank 0 the tallies include the other ranks' factors, so the
  // stats equal the single-GPU ones; the other ranks' stats cover their local phase
  P->stats = stats_json(a, a.n, per_level, max_after, max_seen, final_size, S.flops, fa, S.peak,
                        (int)P->factors.size() + S.nf_extra, S.warnings);
  ht_tail.reset(new HostTimer("tail: apply plan finish"));
  planner.finish();
  plan_finish(P.get());
  ht_tail.reset();
  timeline_end(S.st);
  SGF_CUDA(cudaStreamSynchronize(S.st));
  return P.release();
}

void materialize_l1_e(Precond* P) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto& pe = P->l1e;
  if (!pe.pending) return;
  cudaStream_t st = P->ctx->stream;
  L1ETask* d = P->store.alloc_t<L1ETask>(pe.tasks.size());
  SGF_CUDA(cudaMemcpyAsync(d, pe.tasks.data(), pe.tasks.size() * sizeof(L1ETask), cudaMemcpyHostToDevice, st));
  SGF_CUDA(launch_l1_e(d, (int)pe.tasks.size(), pe.max_m, pe.max_c, pe.rl_n, pe.rl_k, pe.rl_a, st));
  SGF_CUDA(cudaStreamSynchronize(st));  // the host task list goes away below
  pe.pending = false;
  std::vector<L1ETask>().swap(pe.tasks);
}

}  // namespace sgf
