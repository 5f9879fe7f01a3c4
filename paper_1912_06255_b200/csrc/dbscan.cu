// dbscan.cu — host orchestration of the B200 DBSCAN path and the C ABI
// declared in include/dbscan.h. Alg 1 of PAPER.md:
//   Cells (a1-a4) -> NeighborCells (a5) -> MarkCore (a6, a7)
//   -> ClusterCore (a8) -> labels (a9) -> ClusterBorder (a10).
// Every step runs in this library's kernels on the caller's stream.
#include <algorithm>
#include <mutex>
#include <thread>
#include <cstdlib>
#include <cstdio>
#include <cmath>
#include <cstring>

#include "../../include/dbscan.h"
#include "internal.h"

namespace db {

static thread_local std::string g_last_error;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    throw Error(e == cudaErrorMemoryAllocation ? DBSCAN_ENOMEM : DBSCAN_ECUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
  }
}

typedef unsigned __int128 u128;

static uint64_t isqrt_u128(u128 v) {  // floor(sqrt(v)), v < 2^126
  uint64_t r = 0;
  for (int b = 63; b >= 0; --b) {
    uint64_t c = r | (1ull << b);
    if ((u128)c * c <= v) r = c;
  }
  return r;
}

static int bit_width(uint64_t v) {
  int w = 0;
  while (v) { ++w; v >>= 1; }
  return w;
}

// work counters of the measurement build (common.cuh DB_WORK), one reader per
// translation unit (registered by static initialisers: function-local list)
static std::vector<WorkIo>& work_fns() {
  static std::vector<WorkIo> v;
  return v;
}
void work_register(WorkIo fn) { work_fns().push_back(fn); }
static constexpr bool counting_build() {
#ifdef DB_COUNT_WORK
  return true;
#else
  return false;
#endif
}

struct Priv {
  bool dev = false;
  cudaStream_t st = nullptr;  // stream of the call; device outputs are freed on it
  // pointers this library allocated (freed by dbscan_result_free)
  void* core = nullptr;
  void* cluster = nullptr;
  void* border_off = nullptr;
  void* border_ids = nullptr;
};

static void init_device_once(int dev, int* sms) {
  static std::mutex mu;
  static bool done[64] = {};
  static int nsm[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) { *sms = 148; return; }
  if (!done[dev]) {
    // Keep freed stream-ordered memory in the pool across calls so repeated
    // calls do not re-map device memory.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    nsm[dev] = v > 0 ? v : 148;
    done[dev] = true;
    (void)cudaGetLastError();
  }
  *sms = nsm[dev];
}

struct Timer {
  bool on;
  cudaStream_t st;
  cudaEvent_t* ev = nullptr;  // DBSCAN_NSTAGES + 1 events of the thread's cache
  int mark[DBSCAN_NSTAGES + 1];
  int n = 0;
  Timer(bool on_, cudaStream_t s, cudaEvent_t* evs) : on(on_), st(s), ev(evs) {}
  void stage(int s) {  // begin stage s (ends the previous one)
    if (!on) return;
    DB_CUDA(cudaEventRecord(ev[n], st));
    mark[n++] = s;
  }
  void close() {  // end the last stage
    if (on && n > 0) DB_CUDA(cudaEventRecord(ev[n], st));
  }
  void finish(float* out) {  // after close() and a synchronisation of the stream
    if (!on || n == 0) return;
    for (int i = 0; i < n; ++i) {
      float ms = 0;
      DB_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      out[mark[i]] += ms;
    }
    float tot = 0;
    DB_CUDA(cudaEventElapsedTime(&tot, ev[0], ev[n]));
    out[DBSCAN_STAGE_TOTAL] = tot;
  }
};

// Workspaces: what a call needs beyond its inputs and outputs, kept across
// calls in a process-wide pool (per device) so that a call makes no allocator
// call per temporary and creates no events or streams — whichever thread
// makes it (threads may come and go). A call takes an idle workspace (or a new
// one) and returns it when it has finished with it (its stream is idle).
//  * dev: device memory for the temporaries (Ctx::alloc), regrown after a
//    call that needed more;
//  * pin: 1 MB of pinned host memory for small transfers (Ctx::upload, fetch);
//  * events: the call's 4 events and the stage timer's;
//  * side: a second stream (host-path copies of finished outputs overlap the
//    remaining stages on the call's stream).
struct Workspace {
  int dev = -1;
  Arena mem, pin;
  cudaEvent_t plain[4] = {};
  cudaEvent_t timed[DBSCAN_NSTAGES + 1] = {};
  bool timed_made = false;
  cudaStream_t side = nullptr;
};

static std::mutex g_ws_mu;
static std::vector<Workspace*>* g_ws_idle = new std::vector<Workspace*>();  // (never destroyed: exit order)

static size_t g_ws_hwm[64] = {};  // largest workspace memory so far, per device (under g_ws_mu)

static Workspace* ws_acquire(int dev, bool timed, cudaStream_t st) {
  Workspace* w = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (size_t i = 0; i < g_ws_idle->size(); ++i)
      if ((*g_ws_idle)[i]->dev == dev) {
        w = (*g_ws_idle)[i];
        (*g_ws_idle)[i] = g_ws_idle->back();
        g_ws_idle->pop_back();
        break;
      }
  }
  if (!w) {
    static const bool trace = getenv("DB_TRACE_WS") != nullptr;
    if (trace) fprintf(stderr, "workspace: new\n");
    w = new Workspace();
    w->dev = dev;
    // a new workspace (a call concurrent with others) starts at the size the
    // others have grown to (stream-ordered: usable by this call's kernels)
    size_t hwm = 0;
    {
      std::lock_guard<std::mutex> lk(g_ws_mu);
      hwm = dev >= 0 && dev < 64 ? g_ws_hwm[dev] : 0;
    }
    void* m = nullptr;
    if (hwm && cudaMallocAsync(&m, hwm, st) == cudaSuccess) {
      w->mem.base = static_cast<char*>(m);
      w->mem.cap = hwm;
    } else {
      (void)cudaGetLastError();
    }
    for (auto& x : w->plain) DB_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    DB_CUDA(cudaStreamCreateWithFlags(&w->side, cudaStreamNonBlocking));
    void* p = nullptr;
    if (cudaMallocHost(&p, (size_t)1 << 20) == cudaSuccess) {
      w->pin.base = static_cast<char*>(p);
      w->pin.cap = (size_t)1 << 20;
    } else {
      (void)cudaGetLastError();
    }
  }
  else {  // an idle workspace smaller than another one has grown to: catch up (stream-ordered)
    size_t hwm = 0;
    {
      std::lock_guard<std::mutex> lk(g_ws_mu);
      hwm = dev >= 0 && dev < 64 ? g_ws_hwm[dev] : 0;
    }
    void* m = nullptr;
    if (w->mem.cap < hwm && cudaMallocAsync(&m, hwm, st) == cudaSuccess) {
      if (w->mem.base) (void)cudaFreeAsync(w->mem.base, st);
      w->mem.base = static_cast<char*>(m);
      w->mem.cap = hwm;
    }
    (void)cudaGetLastError();
  }
  if (timed && !w->timed_made) {
    for (auto& x : w->timed) DB_CUDA(cudaEventCreate(&x));
    w->timed_made = true;
  }
  return w;
}

static void ws_release(Workspace* w) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  g_ws_idle->push_back(w);
}

// returns w to the pool when the call ends (Ctx has already waited for its stream)
struct WsGuard {
  Workspace* w;
  ~WsGuard() {
    if (w) ws_release(w);
  }
};

void arena_grow(Arena& a, size_t need, cudaStream_t st) {
  static const bool trace = getenv("DB_TRACE_WS") != nullptr;
  if (trace) fprintf(stderr, "workspace %p: grow %zu -> need %zu\n", (void*)&a, a.cap, need);
  if (a.base) DB_CUDA(cudaFreeAsync(a.base, st));
  a.base = nullptr;
  a.cap = 0;
  size_t cap = (need + need / 8 + ((size_t)1 << 20)) & ~(size_t)255;
  int dv = 0;
  if (cudaGetDevice(&dv) == cudaSuccess && dv >= 0 && dv < 64) {  // at least what the others have
    std::lock_guard<std::mutex> lk(g_ws_mu);
    cap = std::max(cap, g_ws_hwm[dv]);
  }
  void* p = nullptr;
  if (cudaMallocAsync(&p, cap, st) != cudaSuccess) {  // keep going without a workspace
    (void)cudaGetLastError();
    return;
  }
  DB_CUDA(cudaStreamSynchronize(st));
  a.base = static_cast<char*>(p);
  a.cap = cap;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    g_ws_hwm[dev] = std::max(g_ws_hwm[dev], cap);
  }
}

// frees the idle workspaces (dbscan_release_workspace)
static void ws_release_idle() {
  std::vector<Workspace*> v;
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    v.swap(*g_ws_idle);
  }
  for (Workspace* w : v) {
    if (w->mem.base) (void)cudaFree(w->mem.base);
    if (w->pin.base) (void)cudaFreeHost(w->pin.base);
    for (auto& x : w->plain) if (x) (void)cudaEventDestroy(x);
    for (auto& x : w->timed) if (x) (void)cudaEventDestroy(x);
    if (w->side) (void)cudaStreamDestroy(w->side);
    delete w;
  }
}

// Host-path outputs that are constant (no border point: border_off = 0; no
// core point: every output) are written on the host instead of crossing the
// host link, by several threads (one thread writes pinned memory at ~10 GB/s,
// slower than the link; the link is what concurrent calls share).
static void host_fill(void* dst, int byte, size_t bytes) {
  const size_t chunk = (size_t)8 << 20;
  const int nt = (int)std::min<size_t>(8, (bytes + chunk - 1) / chunk);
  if (nt <= 1) {
    std::memset(dst, byte, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (bytes + nt - 1) / nt;
  for (int t = 1; t < nt; ++t) {
    const size_t o = per * t;
    if (o < bytes) th.emplace_back([=] { std::memset((char*)dst + o, byte, std::min(per, bytes - o)); });
  }
  std::memset(dst, byte, std::min(per, bytes));
  for (auto& x : th) x.join();
}

static int run(const int32_t* pts, int64_t n, int32_t d, int64_t eps, int64_t min_pts,
               uint32_t flags, cudaStream_t st, dbscan_result* out, int32_t* uids, int64_t ucap,
               double rho) {
  const bool dev_io = flags & DBSCAN_F_DEVICE_IO;
  const bool caller_out = flags & DBSCAN_F_CALLER_OUT;
  Priv* priv = new Priv();
  priv->dev = dev_io;
  priv->st = st;
  out->priv = priv;
  int dev = 0;
  DB_CUDA(cudaGetDevice(&dev));
  WsGuard wsg{ws_acquire(dev, flags & DBSCAN_F_TIMING, st)};  // (declared first: released last)
  Workspace& ws = *wsg.w;
  Ctx c;
  c.st = st;
  init_device_once(dev, &c.sms);
  c.ar = &ws.mem;
  c.flags = flags;
  c.pin = ws.pin.base ? &ws.pin : nullptr;
  static const bool tracing = getenv("DB_TRACE") != nullptr;
  c.tracing = tracing;
  if (tracing) c.mark("start");
  Timer tm(flags & DBSCAN_F_TIMING, st, ws.timed);
  struct {
    cudaEvent_t* e;
  } evs{ws.plain};
  c.side = ws.side;
  c.fork_ev = evs.e[0];
  c.join_ev = evs.e[1];
  c.stage_fn = [](void* t, int s) { static_cast<Timer*>(t)->stage(s); };
  c.stage_obj = &tm;
  unsigned long long hw[4] = {0, 0, 0, 0};
  if (counting_build()) {  // measurement build: start the call's counters at zero
    for (WorkIo fn : work_fns()) fn(hw, st);
    hw[0] = hw[1] = hw[2] = hw[3] = 0;
  }

  // ---- outputs
  auto out_alloc = [&](size_t bytes, void** slot) -> void* {
    void* p = nullptr;
    if (dev_io) {
      cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, st);
      if (e != cudaSuccess) { (void)cudaGetLastError(); throw Error(DBSCAN_ENOMEM, "output allocation"); }
    } else {
      p = std::malloc(bytes ? bytes : 16);
      if (!p) throw Error(DBSCAN_ENOMEM, "host output allocation");
    }
    *slot = p;
    return p;
  };
  // (for n > 0 allocated right after the bounding-box launch, so the GPU
  // starts while the host allocates)
  auto alloc_outputs = [&]() {
    if (caller_out) return;
    out->core = (uint8_t*)out_alloc((size_t)n, &priv->core);
    out->cluster = (int32_t*)out_alloc(sizeof(int32_t) * (size_t)n, &priv->cluster);
    out->border_off = (int64_t*)out_alloc(sizeof(int64_t) * (size_t)(n + 1), &priv->border_off);
  };
  // border_ids: the caller's buffer (F_CALLER_OUT with capacity) when it fits
  auto ids_alloc = [&](int64_t nnz) -> int32_t* {
    if (caller_out && uids && nnz <= ucap) return uids;
    return (int32_t*)out_alloc(sizeof(int32_t) * (size_t)nnz, &priv->border_ids);
  };
  if (n == 0) {
    alloc_outputs();
    out->border_ids = ids_alloc(0);
    if (dev_io) DB_CUDA(cudaMemsetAsync(out->border_off, 0, sizeof(int64_t), st));
    else out->border_off[0] = 0;
    if (dev_io) DB_CUDA(cudaStreamSynchronize(st));
    return DBSCAN_OK;
  }

  // ---- host-side geometry and the exact-arithmetic path (readings 4, 5, 17)
  const u128 eps2 = (u128)eps * (u128)eps;
  const u128 dc2 = (u128)d * (u128)(eps + 1) * (u128)(eps + 1);
  if (dc2 >= ((u128)1 << 62)) throw Error(DBSCAN_ERANGE, "d*(eps+1)^2 >= 2^62");
  const uint64_t s = isqrt_u128(eps2 / (u128)d) + 1;  // < 2^31 since eps^2/d < 2^62
  // 32-bit distance path (reading 4): every distance test compares
  // points of cells at most R apart per axis, so |a_k - b_k| <= (R+1)s - 1;
  // if d ((R+1)s - 1)^2 < 2^32 the plain squared sum is exact in uint32.
  const uint64_t Rr = (uint64_t)(eps - 1) / s + 1;
  const u128 span = (u128)(Rr + 1) * s - 1;
  const bool wide = (flags & DBSCAN_F_FORCE_WIDE) || dc2 >= ((u128)1 << 32) ||
                    (u128)d * span * span >= ((u128)1 << 32);
  Geo g{};
  g.d = d;
  g.D = d <= 2 ? 2 : (d <= 4 ? 4 : 8);
  g.s = (uint32_t)s;
  g.eps2 = (uint64_t)eps2;
  g.eps = (uint64_t)eps;
  g.clampc = (uint32_t)(eps + 1);
  g.R = (uint32_t)((uint64_t)(eps - 1) / s + 1);
  // rho-approximate connectivity (row f4): largest integer m = t - 1 with
  // 2 m sqrt(d) <= eps rho, i.e. 4 d m^2 <= (eps rho)^2; t = 1 is exact
  g.at = 0;
  if (rho > 0) {
    const long double er = (long double)eps * (long double)rho;
    long double mm = floorl(er / (2.0L * sqrtl((long double)d)));
    if (mm > 2e9L) mm = 2e9L;
    uint64_t m = (uint64_t)mm;
    while (m > 0 && 4.0L * d * (long double)m * (long double)m > er * er) --m;
    if (m >= 1) g.at = (uint32_t)(m + 1);
    // cell-level cut-off threshold floor((eps (1 + rho'))^2) with the dyadic
    // rho' = floor(rho 2^40) / 2^40 <= rho, exactly in 128-bit integers:
    // X = eps (2^40 + M), X = q 2^40 + r, X^2 / 2^80 = q^2 + (2 q r + r^2 / 2^40) / 2^40
    const long double rr = (long double)rho * 1099511627776.0L;
    const u128 M = (u128)floorl(rr);
    const u128 X = (u128)eps * (((u128)1 << 40) + M);
    const u128 q = X >> 40, r = X & (((u128)1 << 40) - 1);
    const u128 T = q * q + ((2 * q * r + ((r * r) >> 40)) >> 40);
    const u128 lim = ((u128)1 << 60) / (u128)d;
    if (M > 0 && T < lim) {
      g.eps2_apx = (uint64_t)T;
      g.apxc = (uint32_t)std::min<u128>(isqrt_u128(T) + 1, 0xffffffffu);
    }
  }

  tm.stage(DBSCAN_STAGE_BBOX);
  const int32_t* dpts = pts;
  if (!dev_io) {
    int32_t* p = c.alloc<int32_t>((size_t)n * d);
    // Concurrent host-path calls copy their inputs one at a time: the copy
    // engine would interleave them, so every call's input would arrive late
    // and all the calls would compute at the end together. In turn, each
    // call computes while the next one's input is in flight.
    static std::mutex h2d_mu;
    std::lock_guard<std::mutex> lk(h2d_mu);
    DB_CUDA(cudaMemcpyAsync(p, pts, sizeof(int32_t) * (size_t)n * d, cudaMemcpyHostToDevice, st));
    DB_CUDA(cudaStreamSynchronize(st));
    dpts = p;
  }
  int32_t* lohi_d = c.alloc<int32_t>(17);
  bbox(c, dpts, n, d, g.s, lohi_d);
  alloc_outputs();
  int32_t lohi[17];
  const int32_t* lohi_h = c.fetch(lohi_d, 17);
  c.sync();
  std::memcpy(lohi, lohi_h, sizeof(lohi));
  uint32_t bits = 0;
  for (int k = d - 1; k >= 0; --k) {  // axis 0 most significant
    const uint64_t span = (uint64_t)((int64_t)lohi[8 + k] - (int64_t)lohi[k]);
    const uint64_t maxc = span / s;
    g.lo[k] = lohi[k];
    g.maxc[k] = (uint32_t)maxc;
    g.width[k] = (uint32_t)bit_width(maxc);
    g.shift[k] = bits;
    bits += g.width[k];
  }
  if (bits > 63) throw Error(DBSCAN_ERANGE, "packed cell key needs more than 63 bits");
  g.bits = bits;
  const bool key64 = bits > 32;

  // ---- a1-a4: group the points by cell. Few distinct cells: hash-table
  // counting sort (group.cu); otherwise keys + LSD radix sort + segmentation.
  tm.stage(DBSCAN_STAGE_KEYS);
  int32_t* Ps = c.alloc<int32_t>((size_t)n * g.D);
  uint32_t* cell_of = c.alloc<uint32_t>(n);
  uint32_t* cell_start = c.alloc<uint32_t>((size_t)n + 1);
  uint64_t* cell_key = c.alloc<uint64_t>(n);
  uint32_t* sidx = nullptr;
  uint32_t* cellmin = nullptr;
  uint32_t ncells = 0;
  int passes = 0;
  bool hash_group = false;
  bool key_ordered = true;  // cell ids follow key order (the radix path always)
  // the hash table (<= 2^20 slots) always fits n <= 2^19 cells; beyond that
  // try it only if the sample saw repeated cells
  const bool try_hash = !(flags & (DBSCAN_F_RADIX_GROUP | DBSCAN_F_LATTICE_GROUP)) &&
                        (n <= (1 << 19) || lohi[16] >= 16);
  if (try_hash) {
    sidx = c.alloc<uint32_t>(n);
    c.inv = c.alloc<uint32_t>(n);  // inverse permutation (labels by input index)
    const bool sparse_ok = d <= 3 && !(flags & (DBSCAN_F_NO_SPARSE | DBSCAN_F_FORCE_STENCIL | DBSCAN_F_FORCE_TREE));
    const int sparse_mode = !sparse_ok ? 0 : ((flags & DBSCAN_F_FORCE_SPARSE) ? 2 : 1);
    hash_group = group_by_hash(c, dpts, n, g, sparse_mode, Ps, sidx, cell_of, cell_start, cell_key, &cellmin,
                               &ncells, &key_ordered);
    if (!hash_group) c.inv = nullptr;
  }
  // many cells, d <= 3, small padded lattice: counting sort over the lattice
  // (group.cu), which also yields the sparse path's rank directory and the
  // largest cell for Alg 2's global bound
  bool lat_group = false, no_core = false;
  const uint4* lat_dir = nullptr;
  if (!hash_group && !(flags & DBSCAN_F_RADIX_GROUP) && lattice_applicable(g, n)) {
    if (!sidx) sidx = c.alloc<uint32_t>(n);
    const uint64_t bound_cells = stencil_offsets(g).size() / (size_t)d + 1;
    const int r = lattice_group(c, dpts, n, g, bound_cells, min_pts, Ps, sidx, cell_of, cell_start, cell_key,
                                &lat_dir, &ncells);
    lat_group = r == LAT_OK;
    no_core = r == LAT_ALL_NOISE;
  }
  if (!hash_group && !lat_group && !no_core) {
    void* skeys;
    cell_keys_and_sort(c, dpts, n, g, key64, &skeys, &sidx, &passes);
    tm.stage(DBSCAN_STAGE_SEGMENT);
    ncells = segment_and_gather(c, skeys, key64, sidx, dpts, n, g, Ps, cell_of, cell_start, cell_key);
  }
  // how a9 finds each cell's smallest core index: first point (stable radix
  // sort + stable partition), per-cell minima (hash), or a scan of the cell's
  // core points (lattice counting sort; sparse cells)
  int min_mode = hash_group ? LABEL_MIN_ARRAY : (lat_group ? LABEL_MIN_SCAN : LABEL_MIN_FIRST);
  QTrees qtrees;

  // ---- regime: CSR path (neighbour lists) or the cell-centric sparse path
  const bool tree = (flags & DBSCAN_F_FORCE_TREE) || (d >= 4 && !(flags & DBSCAN_F_FORCE_STENCIL));
  const bool sparse = !no_core && !tree && key_ordered && !(flags & DBSCAN_F_NO_SPARSE) &&
                      !(flags & DBSCAN_F_FORCE_STENCIL) &&
                      sparse_applicable(g, n, ncells, flags & DBSCAN_F_FORCE_SPARSE);
  const bool waves = !(flags & DBSCAN_F_NO_WAVES);

  // device counters: [0] core cells, [1] mixed cells, [2] clusters, [3] core points
  uint32_t* cnt32 = c.alloc<uint32_t>(4);
  unsigned long long* cnt64 = c.alloc<unsigned long long>(3);  // [0] tested pairs, [1] border pts, [2] pairs
  c.zero(cnt32, 16);
  c.zero(cnt64, 24);
  uint8_t* core_s = c.alloc<uint8_t>(n);
  uint32_t* core_cnt = c.alloc<uint32_t>(ncells);

  uint64_t nbr_total = 0;
  bool dense_dir = false;
  unsigned long long* qb_decided = nullptr;  // points proved core by the sub-cell bounds
  CellsView cv{ncells, cell_start, cell_key, cell_of, nullptr, nullptr, nullptr};
  SparseOut so;
  struct SpGuard { SparseOut* o; ~SpGuard() { sparse_release(o); } } sp_guard{&so};
  uint32_t core_cells = 0;
  if (no_core) {
    // Alg 2's global bound: no point can be core (nothing was grouped)
  } else if (sparse) {
    // ---- a4 + a6 + a7 on the rank directory
    tm.stage(DBSCAN_STAGE_MARKCORE);
    so.flags = flags;
    so.counters = c.alloc<uint32_t>(6);
    c.zero(so.counters, 24);
    core_cells = sparse_pipeline(c, g, cv, Ps, sidx, core_s, core_cnt, n, min_pts, wide, lat_dir,
                                 !(flags & DBSCAN_F_NO_BRICK), &so);
  } else {
    // ---- a4-a5: cell lookup + neighbour CSR (+ MarkCore bound ub)
    uint64_t* nbr_off;
    uint32_t* nbr;
    uint32_t* ub;
    tm.stage(DBSCAN_STAGE_NEIGHBORS);
    if (!tree)
      neighbors_stencil(c, g, cell_key, cell_start, ncells, n, &nbr_off, &nbr, &ub, &nbr_total, &dense_dir,
                        &cv.ccls);
    else
      neighbors_tree(c, g, cell_key, cell_start, ncells, &nbr_off, &nbr, &ub, &nbr_total,
                     !(flags & DBSCAN_F_FORCE_TREE), &cv.ccls);
    cv.nbr_off = nbr_off;
    cv.nbr = nbr;
    cv.ub = ub;
    // ---- row f2 (our-exact-qt): per-cell range-count trees for big cells
    if (flags & DBSCAN_F_QUADTREE) {
      build_qtrees(c, g, cv, Ps, sidx, n, &qtrees);
      if (min_mode == LABEL_MIN_FIRST) min_mode = LABEL_MIN_SCAN;  // cells are no longer stable
    }
    // ---- a6: MarkCore (large minPts: sub-cell lower bounds first, row f2)
    tm.stage(DBSCAN_STAGE_MARKCORE);
    const bool bounds = !(flags & DBSCAN_F_QUADTREE) && !(flags & DBSCAN_F_NO_QBOUND) &&
                        (min_pts >= QB_MIN_PTS || (flags & DBSCAN_F_FORCE_QBOUND));
    if (bounds) {
      qb_decided = c.alloc<unsigned long long>(1);
      c.zero(qb_decided, sizeof(unsigned long long));
      c.zero(core_s, (size_t)n);
      mark_core_bounds(c, g, cv, Ps, sidx, n, min_pts, core_s, qb_decided);
      if (min_mode == LABEL_MIN_FIRST) min_mode = LABEL_MIN_SCAN;  // cells are no longer stable
    }
    mark_core(c, g, cv, Ps, n, min_pts, wide, core_s, &qtrees, bounds);
    // ---- a7: core-first compaction
    tm.stage(DBSCAN_STAGE_COMPACT);
    compact_core(c, g, cv, Ps, sidx, core_s, n, min_pts, core_cnt, cnt32);
    // no host read here: with no core cell the later stages produce the
    // all-noise result by themselves (the count is read with the final stats)
    core_cells = UINT32_MAX;
  }

  cudaStream_t side = c.side;
  cudaEvent_t ev_labels = evs.e[2], ev_side = evs.e[3];
  bool side_used = false;
  uint8_t* core_d = dev_io ? out->core : c.alloc<uint8_t>(n);
  int32_t* cluster_d = dev_io ? out->cluster : c.alloc<int32_t>(n);
  int64_t* off_d = dev_io ? out->border_off : c.alloc<int64_t>((size_t)n + 1);
  int64_t nnz = 0;
  // final counters (read with the call's last synchronisation)
  const uint32_t* h32_h = nullptr;
  const unsigned long long* h64_h = nullptr;
  const unsigned long long* hqb = nullptr;
  const uint64_t* hnbr = nullptr;
  auto fetch_counters = [&]() {
    h32_h = c.fetch(cnt32, 4);
    h64_h = c.fetch(cnt64, 3);
    hqb = qb_decided ? c.fetch(qb_decided, 1) : nullptr;
    hnbr = c.nbr_total_d ? c.fetch(c.nbr_total_d, 1) : nullptr;
  };
  if (core_cells == 0) {
    // no core point: no cluster, every point is noise
    tm.stage(DBSCAN_STAGE_LABELS);
    DB_CUDA(cudaMemsetAsync(core_d, 0, (size_t)n, st));
    DB_CUDA(cudaMemsetAsync(cluster_d, 0xff, sizeof(int32_t) * (size_t)n, st));
    DB_CUDA(cudaMemsetAsync(off_d, 0, sizeof(int64_t) * (size_t)(n + 1), st));
    out->border_ids = ids_alloc(0);
  } else {
    // ---- a8: ClusterCore
    tm.stage(DBSCAN_STAGE_CLUSTER);
    uint32_t* parent = c.alloc<uint32_t>(ncells);
    if (sparse) sparse_cluster(c, g, cv, Ps, core_cnt, wide, parent, cnt64, &so);
    else cluster_core(c, g, cv, Ps, core_cnt, wide, waves, nbr_total, parent, cnt64, cnt64 + 2, &qtrees);

    // ---- a9: labels, scattered to input order
    tm.stage(DBSCAN_STAGE_LABELS);
    uint32_t* cell_label = c.alloc<uint32_t>(ncells);
    labels(c, cv, sidx, core_s, core_cnt, min_mode, cellmin, sparse ? so.core_list : nullptr, so.ncore, parent,
           n, cell_label, core_d, cluster_d, cnt32 + 2);

    // host path: core flags and labels are final; copy them out on the side
    // stream while ClusterBorder runs
    if (!dev_io) {
      DB_CUDA(cudaEventRecord(ev_labels, st));
      DB_CUDA(cudaStreamWaitEvent(side, ev_labels, 0));
      DB_CUDA(cudaMemcpyAsync(out->core, core_d, (size_t)n, cudaMemcpyDeviceToHost, side));
      DB_CUDA(cudaMemcpyAsync(out->cluster, cluster_d, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToHost,
                              side));
      side_used = true;
    }

    // ---- a10: ClusterBorder
    tm.stage(DBSCAN_STAGE_BORDER);
    if (sparse) sparse_border(c, g, cell_label, cluster_d, n, wide, off_d, cnt64 + 1, &so);
    else border_count(c, g, cv, Ps, sidx, core_cnt, cell_label, cluster_d, n, wide, off_d, cnt64 + 1);
    // one synchronisation gives nnz = border_off[n] (the size of border_ids)
    // and the final counters; with no border point the device work ends here
    const int64_t* nnz_h = c.fetch(off_d + n, 1);
    fetch_counters();
    if (c.tracing) c.mark("border sync");
    c.sync();
    nnz = *nnz_h;
    if (!dev_io && nnz == 0) host_fill(out->border_off, 0, sizeof(int64_t) * (size_t)(n + 1));
    else if (!dev_io)
      DB_CUDA(cudaMemcpyAsync(out->border_off, off_d, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyDeviceToHost,
                              side));
    if (c.tracing) c.mark("border nnz known");
    out->border_ids = ids_alloc(nnz);
    if (c.tracing) c.mark("ids alloc");
    int32_t* ids_d = dev_io ? out->border_ids : c.alloc<int32_t>(nnz);
    if (nnz > 0) {
      if (sparse) sparse_border_fill(c, g, wide, off_d, ids_d, &so);
      else border_fill(c, g, cv, Ps, sidx, core_cnt, cell_label, wide, off_d, ids_d);
    }
    if (!dev_io && nnz > 0)
      DB_CUDA(cudaMemcpyAsync(out->border_ids, ids_d, sizeof(int32_t) * (size_t)nnz,
                              cudaMemcpyDeviceToHost, st));
  }

  if (!dev_io && !side_used) {  // no core point: core 0, cluster -1, border_off 0
    host_fill(out->core, 0, (size_t)n);
    host_fill(out->cluster, 0xff, sizeof(int32_t) * (size_t)n);
    host_fill(out->border_off, 0, sizeof(int64_t) * (size_t)(n + 1));
  }
  if (side_used) {  // the temporaries stay alive until the side copies are done
    DB_CUDA(cudaEventRecord(ev_side, side));
    DB_CUDA(cudaStreamWaitEvent(st, ev_side, 0));
  }
  uint32_t h32[4];
  unsigned long long h64[3];
  if (!h32_h) fetch_counters();
  tm.close();  // (the last event; read after the stream is idle)
  c.free_all();
  if (c.tracing) c.mark("final sync");
  DB_CUDA(cudaStreamSynchronize(st));
  tm.finish(out->stage_ms);
  c.finish();
  std::memcpy(h32, h32_h, sizeof(h32));
  std::memcpy(h64, h64_h, sizeof(h64));
  if (counting_build())
    for (WorkIo fn : work_fns()) fn(hw, st);
  if (c.tracing) {
    c.mark("end");
    const double t0 = c.trace.front().second;
    for (auto& e : c.trace) fprintf(stderr, "  %9.1f us  %s %d\n", e.second - t0, e.first.first, e.first.second);
  }

  out->nnz = nnz;
  out->n_core = h32[3];
  out->n_clusters = h32[2];
  out->n_border = (int64_t)h64[1];
  out->n_noise = n - out->n_core - out->n_border;
  out->stats[DBSCAN_STAT_NCELLS] = ncells;
  out->stats[DBSCAN_STAT_KEY_BITS] = bits;
  out->stats[DBSCAN_STAT_SORT_PASSES] = passes;
  out->stats[DBSCAN_STAT_NBR_ENTRIES] = hnbr ? (int64_t)*hnbr : (int64_t)nbr_total;
  out->stats[DBSCAN_STAT_CORE_CELLS] = core_cells == UINT32_MAX ? h32[0] : core_cells;
  out->stats[DBSCAN_STAT_PAIRS] = (int64_t)h64[2];
  out->stats[DBSCAN_STAT_PAIRS_TESTED] = (int64_t)h64[0];
  out->stats[DBSCAN_STAT_LAUNCHES] = c.launches;
  out->stats[DBSCAN_STAT_WIDE] = wide;
  out->stats[DBSCAN_STAT_TREE] = tree;
  out->stats[DBSCAN_STAT_CELL_SIDE] = (int64_t)s;
  out->stats[DBSCAN_STAT_DENSE_DIR] = dense_dir;
  out->stats[DBSCAN_STAT_SPARSE] = sparse;
  out->stats[DBSCAN_STAT_HASH_GROUP] = hash_group ? 1 : (lat_group ? 2 : 0);
  out->stats[DBSCAN_STAT_MARKCORE_TESTS] = (int64_t)hw[0];
  out->stats[DBSCAN_STAT_BCP_TESTS] = (int64_t)hw[1];
  out->stats[DBSCAN_STAT_BORDER_TESTS] = (int64_t)hw[2];
  out->stats[DBSCAN_STAT_MARKCORE_ALG2] = (int64_t)hw[3];
  out->stats[DBSCAN_STAT_COUNTING_BUILD] = counting_build();
  out->stats[DBSCAN_STAT_QT_NODES] = (int64_t)qtrees.nodes;
  out->stats[DBSCAN_STAT_APPROX_SIDE] = g.at;
  out->stats[DBSCAN_STAT_BRICK] = so.brick;
  out->stats[DBSCAN_STAT_POINT_BORDER] = so.point_border;
  out->stats[DBSCAN_STAT_SPARSE_PASSES] = so.passes;
  out->stats[DBSCAN_STAT_QB_DECIDED] = hqb ? (int64_t)*hqb : -1;
  return DBSCAN_OK;
}

}  // namespace db

using namespace db;

static void free_priv(dbscan_result* r) {
  Priv* p = (Priv*)r->priv;
  if (!p) return;
  void* ptrs[4] = {p->core, p->cluster, p->border_off, p->border_ids};
  for (void* q : ptrs) {
    if (!q) continue;
    if (p->dev) cudaFreeAsync(q, p->st);
    else std::free(q);
  }
  if (p->core) r->core = nullptr;
  if (p->cluster) r->cluster = nullptr;
  if (p->border_off) r->border_off = nullptr;
  if (p->border_ids) r->border_ids = nullptr;
  delete p;
  r->priv = nullptr;
}

extern "C" {

static int dbscan_impl(const int32_t* pts, int64_t n, int32_t d, int64_t eps, int64_t min_pts, uint32_t flags,
                       void* stream, dbscan_result* out, double rho) {
  g_last_error.clear();
  if (!out) { g_last_error = "out is NULL"; return DBSCAN_EINVAL; }
  const bool caller_out = flags & DBSCAN_F_CALLER_OUT;
  uint8_t* ucore = out->core;
  int32_t* ucl = out->cluster;
  int64_t* uoff = out->border_off;
  int32_t* uids = caller_out ? out->border_ids : nullptr;  // optional, capacity in out->nnz
  const int64_t ucap = caller_out && uids ? out->nnz : 0;
  std::memset(out, 0, sizeof(*out));
  if (caller_out) { out->core = ucore; out->cluster = ucl; out->border_off = uoff; }
  out->n = n;
  out->flags = flags;
  const char* bad = nullptr;
  if (n < 0 || n > INT32_MAX) bad = "n out of range [0, 2^31-1]";
  else if (d < 1 || d > 8) bad = "d out of range [1, 8]";
  else if (eps < 1) bad = "eps < 1";
  else if (min_pts < 1) bad = "min_pts < 1";
  else if (!pts && n > 0) bad = "pts is NULL";
  else if ((flags & DBSCAN_F_FORCE_STENCIL) && (flags & DBSCAN_F_FORCE_TREE)) bad = "FORCE_STENCIL with FORCE_TREE";
  else if (caller_out && (!uoff || (n > 0 && (!ucore || !ucl)))) bad = "F_CALLER_OUT with NULL output";
  else if ((flags & DBSCAN_F_FORCE_STENCIL) && d > 6) bad = "FORCE_STENCIL limited to d <= 6";
  else if ((flags & DBSCAN_F_RADIX_GROUP) && (flags & DBSCAN_F_LATTICE_GROUP)) bad = "RADIX_GROUP with LATTICE_GROUP";
  if (bad) { g_last_error = bad; return DBSCAN_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  try {
    return run(pts, n, d, eps, min_pts, flags, st, out, uids, ucap, rho);
  } catch (const Error& e) {
    g_last_error = e.what();
    // (the call's stream and its side stream were synchronised by ~Ctx)
    (void)cudaGetLastError();
    free_priv(out);
    if (!caller_out) { out->core = nullptr; out->cluster = nullptr; out->border_off = nullptr; }
    out->border_ids = nullptr;
    out->nnz = 0;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    free_priv(out);
    return DBSCAN_ECUDA;
  }
}

int dbscan(const int32_t* pts, int64_t n, int32_t d, int64_t eps, int64_t min_pts, uint32_t flags,
           void* stream, dbscan_result* out) {
  return dbscan_impl(pts, n, d, eps, min_pts, flags, stream, out, 0.0);
}

int dbscan_approx(const int32_t* pts, int64_t n, int32_t d, int64_t eps, int64_t min_pts, double rho,
                  uint32_t flags, void* stream, dbscan_result* out) {
  if (!(rho > 0) || rho > 1e6) {
    g_last_error = "rho must be in (0, 1e6]";
    if (out) std::memset(out, 0, sizeof(*out));
    return DBSCAN_EINVAL;
  }
  return dbscan_impl(pts, n, d, eps, min_pts, flags, stream, out, rho);
}

void dbscan_result_free(dbscan_result* r) {
  if (!r) return;
  free_priv(r);
}

void dbscan_release_workspace(void) { ws_release_idle(); }

const char* dbscan_error_string(int code) {
  static thread_local std::string s;
  const char* base = "unknown error";
  switch (code) {
    case DBSCAN_OK: base = "ok"; break;
    case DBSCAN_EINVAL: base = "invalid argument"; break;
    case DBSCAN_ERANGE: base = "value out of supported range"; break;
    case DBSCAN_ENOMEM: base = "out of memory"; break;
    case DBSCAN_ECUDA: base = "CUDA error"; break;
  }
  s = base;
  if (code != DBSCAN_OK && !g_last_error.empty()) s += ": " + g_last_error;
  return s.c_str();
}

const char* dbscan_stage_name(int i) {
  static const char* names[DBSCAN_NSTAGES] = {"bbox",     "keys+sort", "sort",    "segment",
                                              "hash",     "neighbors", "markcore", "compact",
                                              "cluster",  "labels",    "border",  "total"};
  return (i >= 0 && i < DBSCAN_NSTAGES) ? names[i] : "?";
}

int dbscan_version(void) { return 100; }

}  // extern "C"
