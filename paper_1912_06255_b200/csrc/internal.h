// internal.h — host-side interfaces between the stage files of the B200 path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dbscan.h"
#include "common.cuh"

namespace db {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
#define DB_CUDA(call) ::db::cuda_check((call), #call)

// A block of device or pinned host memory of a workspace (see Ctx::alloc, dbscan.cu).
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
};
void arena_grow(Arena& a, size_t need, cudaStream_t st);  // (after the stream is idle)

// Per-call context: stream, stream-ordered temporaries, launch counter.
struct Ctx {
  cudaStream_t st = nullptr;
  // stage timer hook (begin stage s; no-op without F_TIMING)
  void (*stage_fn)(void*, int) = nullptr;
  void* stage_obj = nullptr;
  // a second stream for independent work (set by the caller with two events
  // for the fork and the join)
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  void fork() {  // side waits for everything queued on st so far
    DB_CUDA(cudaEventRecord(fork_ev, st));
    DB_CUDA(cudaStreamWaitEvent(side, fork_ev, 0));
  }
  void join() {  // st waits for everything queued on side so far
    DB_CUDA(cudaEventRecord(join_ev, side));
    DB_CUDA(cudaStreamWaitEvent(st, join_ev, 0));
  }
  void stage(int s) {
    if (stage_fn) stage_fn(stage_obj, s);
    if (tracing) mark("stage", s);
  }
  // host-side trace (DB_TRACE=1 in the environment): what the host thread
  // does when, to find where the GPU waits for it
  bool tracing = false;
  uint32_t flags = 0;  // the call's DBSCAN_F_* flags (path switches read by the stages)
  std::vector<std::pair<std::pair<const char*, int>, double>> trace;
  void mark(const char* what, int v = -1) {
    trace.push_back({{what, v}, std::chrono::duration<double, std::micro>(
                                    std::chrono::steady_clock::now().time_since_epoch()).count()});
  }
  std::vector<void*> temps;
  int64_t launches = 0;
  int sms = 148;
  uint32_t* dense_dir = nullptr;  // dense cell directory, when built
  // inverse permutation (input index -> sorted position) when the grouping
  // wrote it; the kernels that move points inside cells keep it current
  uint32_t* inv = nullptr;
  const uint64_t* nbr_total_d = nullptr;  // exact neighbour-CSR size (device), when only bounded on the host
  uint64_t dense_lat[3] = {0, 0, 0};
  // Temporaries come out of the call's workspace (one device allocation kept
  // across calls: no allocator call per temporary); past its end they fall
  // back to stream-ordered allocations and the workspace is regrown once the
  // call has finished (finish()).
  Arena* ar = nullptr;
  size_t used = 0;
  bool finished = false;
  // Small host<->device transfers go through pinned host staging (workspace):
  // from pageable memory each one is a synchronous staged copy of ~10-20 us.
  Arena* pin = nullptr;
  size_t pin_used = 0;
  void* pin_take(size_t bytes) {
    bytes = (bytes + 15) & ~(size_t)15;
    if (!pin || pin_used + bytes > pin->cap) return nullptr;
    void* p = pin->base + pin_used;
    pin_used += bytes;
    return p;
  }
  template <typename T>
  void upload(T* dst, const T* src, size_t count) {
    const size_t bytes = sizeof(T) * count;
    void* h = pin_take(bytes);
    if (h) std::memcpy(h, src, bytes);
    DB_CUDA(cudaMemcpyAsync(dst, h ? h : (const void*)src, bytes, cudaMemcpyHostToDevice, st));
  }
  // device -> host, complete after the next sync(): returns the host copy
  template <typename T>
  const T* fetch(const T* dsrc, size_t count) {
    T* h = static_cast<T*>(pin_take(sizeof(T) * count));
    if (!h) {
      fetch_spill.emplace_back(sizeof(T) * count);
      h = reinterpret_cast<T*>(fetch_spill.back().data());
    }
    DB_CUDA(cudaMemcpyAsync(h, dsrc, sizeof(T) * count, cudaMemcpyDeviceToHost, st));
    return h;
  }
  std::vector<std::vector<char>> fetch_spill;

  template <typename T>
  T* alloc(size_t count) {
    size_t bytes = count * sizeof(T);
    bytes = (bytes + 255) & ~(size_t)255;
    if (bytes == 0) bytes = 256;
    if (ar && used + bytes <= ar->cap) {
      void* p = ar->base + used;
      used += bytes;
      return static_cast<T*>(p);
    }
    used += bytes;  // (the size the workspace should have had)
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, st);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      throw Error(-3, std::string("cudaMallocAsync failed: ") + cudaGetErrorString(e));
    }
    temps.push_back(p);
    return static_cast<T*>(p);
  }
  void zero(void* p, size_t bytes) { DB_CUDA(cudaMemsetAsync(p, 0, bytes, st)); }
  void launched() {
    ++launches;
    if (tracing) mark("launch", (int)launches);
#ifdef DB_DEBUG_SYNC
    DB_CUDA(cudaStreamSynchronize(st));
#endif
    DB_CUDA(cudaGetLastError());
  }
  void free_all() {
    for (void* p : temps) cudaFreeAsync(p, st);
    temps.clear();
  }
  // after the call's final synchronisation: regrow an undersized workspace
  void finish() {
    finished = true;
    if (ar && used > ar->cap) arena_grow(*ar, used, st);
  }
  ~Ctx() {  // error paths: the streams may still use the workspace; wait for both
    // before the workspace goes back to the pool (Ctx is destroyed before WsGuard)
    if (!finished && st) (void)cudaStreamSynchronize(st);
    if (!finished && side) (void)cudaStreamSynchronize(side);
    (void)cudaGetLastError();
    free_all();
  }
  // Read a small device value (synchronises the stream).
  void sync() {
    if (tracing) mark("sync");
    DB_CUDA(cudaStreamSynchronize(st));
    if (tracing) mark("sync done");
  }
  template <typename T>
  T read(const T* dptr) {
    if (tracing) mark("read");
    const T* h = fetch(dptr, 1);
    DB_CUDA(cudaStreamSynchronize(st));
    if (tracing) mark("read done");
    return *h;
  }
};

// Work counters of the measurement build (common.cuh DB_WORK): every
// translation unit registers a function that reads (and zeroes) its counters.
typedef void (*WorkIo)(unsigned long long* add_to /* [4] */, cudaStream_t st);
void work_register(WorkIo fn);
#ifdef DB_COUNT_WORK
namespace {
void db_work_io(unsigned long long* add_to, cudaStream_t st) {
  unsigned long long h[4] = {0, 0, 0, 0};
  DB_CUDA(cudaMemcpyFromSymbolAsync(h, db_work_ctr, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
  DB_CUDA(cudaStreamSynchronize(st));
  for (int i = 0; i < 4; ++i) add_to[i] += h[i];
  const unsigned long long z[4] = {0, 0, 0, 0};
  DB_CUDA(cudaMemcpyToSymbolAsync(db_work_ctr, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
}
struct DbWorkReg {
  DbWorkReg() { work_register(&db_work_io); }
} db_work_reg;
}  // namespace
#endif

// ---- scan.cu ----
// out[0..n] = exclusive prefix sums of in[0..n-1]; out[n] = total.
void exclusive_scan_u32_u64(Ctx& c, const uint32_t* in, uint64_t* out, int64_t n);
void exclusive_scan_u32_i64(Ctx& c, const uint32_t* in, int64_t* out, int64_t n,
                            const unsigned long long* zero_if = nullptr /* device: 0 => all outputs 0 */);
void exclusive_scan_u32_u32(Ctx& c, const uint32_t* in, uint32_t* out, int64_t n);
// same, with in[i] read as 0 where mask[i] >= 0 (in[i] is then never read)
void exclusive_scan_u32_i64_masked(Ctx& c, const uint32_t* in, const int32_t* mask, int64_t* out, int64_t n,
                                   const unsigned long long* zero_if = nullptr);

// ---- radix.cu (a2) ----
// LSD passes over the low `passes` 8-bit digits; hist = [passes][256] global digit
// histograms; the sorted pairs end in *ko/*vo (one of the two buffers).
void radix_sort_pairs_u32(Ctx& c, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint32_t n,
                          int passes, const uint32_t* hist, uint32_t** ko, uint32_t** vo);
void radix_sort_pairs_u64(Ctx& c, uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, uint32_t n,
                          int passes, const uint32_t* hist, uint64_t** ko, uint32_t** vo);

// ---- grid.cu (a1-a4) ----
// lohi[0..7] per-axis minimum, [8..15] maximum, [16] sampled cell collisions
// (see keys.cu) for the grouping choice; lohi must hold 17 int32.
void bbox(Ctx& c, const int32_t* pts, int64_t n, int d, uint32_t s, int32_t* lohi);
// keys + LSD radix sort; on return keys/idx hold the sorted (key, input index) pairs
// in *sorted_keys / *sorted_idx (either buffer of the ping-pong pair).
void cell_keys_and_sort(Ctx& c, const int32_t* pts, int64_t n, const Geo& g, bool key64,
                        void** sorted_keys, uint32_t** sorted_idx, int* passes);
// generic u64-key radix sort used by the cell tree (Morton order)
void radix_sort_u64(Ctx& c, uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                    int64_t n, int bits, uint64_t** out_keys, uint32_t** out_vals);
// segmentation + gather: writes padded sorted points Ps[n*D], cell_of[n],
// cell_start[ncells+1], cell_key[ncells]; returns ncells (synchronises).
uint32_t segment_and_gather(Ctx& c, const void* sorted_keys, bool key64, const uint32_t* sorted_idx,
                            const int32_t* pts, int64_t n, const Geo& g, int32_t* Ps,
                            uint32_t* cell_of, uint32_t* cell_start, uint64_t* cell_key);
// counting-sort grouping through a hash table of the distinct keys (group.cu):
// writes Ps, idx (input index per sorted position), cell_of, cell_start,
// cell_key and *cellmin (minimum input index per cell); returns false (nothing
// written) when the keys do not fit its table, and the caller sorts instead.
// sparse_mode (whether the sparse path, which needs cell ids in key order,
// may run): 0 no, 1 if the lattice turns out sparse, 2 forced.
bool group_by_hash(Ctx& c, const int32_t* pts, int64_t n, const Geo& g, int sparse_mode, int32_t* Ps,
                   uint32_t* idx, uint32_t* cell_of, uint32_t* cell_start, uint64_t* cell_key,
                   uint32_t** cellmin, uint32_t* ncells, bool* ordered /* ids in key order */);
// lattice counting sort for d <= 3 when the padded lattice has at most
// LAT_PER_POINT cells per point (group.cu): writes Ps, idx, cell_of,
// cell_start, cell_key (cell ids in key order) and the sparse path's rank
// directory (*dir, 16 B per 32 lattice cells). Returns LAT_OK; LAT_FALLBACK
// (a cell has more than 255 points: nothing written, sort instead); or
// LAT_ALL_NOISE when (largest cell) x bound_cells < min_pts (no core point is
// possible; nothing written).
constexpr uint64_t LAT_PER_POINT = 8;
enum { LAT_OK = 0, LAT_FALLBACK = 1, LAT_ALL_NOISE = 2 };
bool lattice_applicable(const Geo& g, int64_t n);
int lattice_group(Ctx& c, const int32_t* pts, int64_t n, const Geo& g, uint64_t bound_cells, int64_t min_pts,
                  int32_t* Ps, uint32_t* idx, uint32_t* cell_of, uint32_t* cell_start, uint64_t* cell_key,
                  const uint4** dir, uint32_t* ncells);
// open-addressing table of the ncells keys; returns mask (capacity-1).
uint64_t build_hash(Ctx& c, const uint64_t* cell_key, uint32_t ncells, Slot** table);

// ---- neighbors.cu (a5) ----
// neighbour-cell CSR excluding the cell itself: nbr_off[ncells+1] (device), nbr list.
// Both build the CSR and ub[g] = sum of the neighbours' sizes (MarkCore bound).
// *total: the CSR size, or an upper bound of it (exact count then in c.nbr_total_d).
// d <= 3 (or forced): builds a dense cell directory or a hash table itself.
void neighbors_stencil(Ctx& c, const Geo& g, const uint64_t* cell_key, const uint32_t* cell_start,
                       uint32_t ncells, int64_t n, uint64_t** nbr_off, uint32_t** nbr,
                       uint32_t** ub, uint64_t* total, bool* dense, const uint32_t** ccls);
// d >= 4: all-pairs over cells when there are few (<= 16384), else the cell tree
// (allow_brute = false forces the tree).
void neighbors_tree(Ctx& c, const Geo& g, const uint64_t* cell_key, const uint32_t* cell_start,
                    uint32_t ncells, uint64_t** nbr_off, uint32_t** nbr, uint32_t** ub,
                    uint64_t* total, bool allow_brute, const uint32_t** ccls /* NULL unless class-sorted */);
// host: exact stencil offsets (Delta != 0 with sum gap^2 <= eps^2), flat [count*d] int8
std::vector<int8_t> stencil_offsets(const Geo& g);

// ---- core.cu (a6, a7) ----
struct CellsView {
  uint32_t ncells;
  const uint32_t* cell_start;
  const uint64_t* cell_key;
  const uint32_t* cell_of;
  const uint64_t* nbr_off;
  const uint32_t* nbr;
  const uint32_t* ub;  // sum of neighbour-cell sizes (saturating)
  // rows sorted by class (lattice L1 distance 1, 2, >= 3; the all-pairs
  // neighbour path): per cell the class-1 and class-2 counts, [2][ncells]; or NULL
  const uint32_t* ccls = nullptr;
};
// Per-cell range-count trees (qtree.cu, row f2): cells with >= QT_MIN points;
// node_off[c] = first node of cell c's implicit binary tree (heap order),
// box[node] = {lo[D], hi[D]} of its points, cnt[node] = their number.
struct QTrees {
  const uint64_t* node_off = nullptr;
  const int32_t* box = nullptr;
  const uint32_t* cnt = nullptr;
  uint64_t nodes = 0;
};
// Orders the points of tree cells by Morton code inside the cell (Ps, idx
// permuted within each cell) and builds the trees.
void build_qtrees(Ctx& c, const Geo& g, const CellsView& cv, int32_t* Ps, uint32_t* idx, int64_t n, QTrees* qt);
// pre: core_s already holds 1 for points proved core by mark_core_bounds
// (0 elsewhere); those points are skipped.
void mark_core(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps, int64_t n,
               int64_t min_pts, bool wide, uint8_t* core_s, const QTrees* qt = nullptr, bool pre = false);
// Row f2, large minPts: points proved core by lower bounds from sub-cell
// counts (qtree.cu; reorders the points of cells with >= 256 points by
// sub-cell). core_s must be zeroed; *decided (device) += points proved core.
constexpr int64_t QB_MIN_PTS = 2000;  // minPts from which the bounds run by default
void mark_core_bounds(Ctx& c, const Geo& g, const CellsView& cv, int32_t* Ps, uint32_t* idx, int64_t n,
                      int64_t min_pts, uint8_t* core_s, unsigned long long* decided);
// core-first stable partition inside each mixed cell (Ps, idx, core_s permuted in
// place); core_cnt[ncells]; counters[0] += core cells, counters[1] += mixed cells.
void compact_core(Ctx& c, const Geo& g, const CellsView& cv, int32_t* Ps, uint32_t* idx,
                  uint8_t* core_s, int64_t n, int64_t min_pts, uint32_t* core_cnt,
                  uint32_t* counters /*device [2], zeroed*/);

// stable core-first partition of the listed cells (count on the device)
void partition_mixed(Ctx& c, const Geo& g, const CellsView& cv, const uint32_t* mixed,
                     const uint32_t* nmixed, const uint32_t* core_cnt, int32_t* Ps, uint32_t* idx,
                     uint8_t* core_s, int64_t n);

// ---- sparse.cu (cell-centric path for sparse lattices, d <= 3) ----
constexpr uint64_t SPARSE_MEAN_PER_CELL = 4;  // n / ncells at or below: sparse path
struct SparseOut {
  uint32_t* counters = nullptr;  // device [6]: -, brick overflow, large pairs, mixed, core cells, core points
  void* stash = nullptr;         // kernel arguments kept between the stages
  const uint32_t* core_list = nullptr;  // cells holding core points, linear order
  uint32_t ncore = 0;
  int brick = 0;                 // MarkCore: 1 brick kernel, 2 with overflowed bricks
  bool point_border = false;     // ClusterBorder from the non-core points (few of them)
  int passes = 0;                // ClusterCore pair-search launches (stats[DBSCAN_STAT_SPARSE_PASSES])
  uint32_t flags = 0;            // the call's DBSCAN_F_* flags
};
bool sparse_applicable(const Geo& g, int64_t n, uint32_t ncells, bool forced);
// a4 + a6 + a7 on the rank directories: core flags, core-first compaction,
// core_cnt, the core-cell directory; returns the number of core cells (0 =
// no core point, the caller takes the all-noise exit; synchronises).
// dir: the rank directory from the lattice counting sort, or NULL (built here).
// brick_ok: the brick MarkCore may run (DBSCAN_F_NO_BRICK unset).
uint32_t sparse_pipeline(Ctx& c, const Geo& g, const CellsView& cv, int32_t* Ps, uint32_t* idx,
                         uint8_t* core_s, uint32_t* core_cnt, int64_t n, int64_t min_pts, bool wide,
                         const uint4* dir, bool brick_ok, SparseOut* o);
void sparse_cluster(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps,
                    const uint32_t* core_cnt, bool wide, uint32_t* parent,
                    unsigned long long* tested, SparseOut* o);
void sparse_border(Ctx& c, const Geo& g, const uint32_t* cell_label, const int32_t* cluster, int64_t n,
                   bool wide, int64_t* border_off, unsigned long long* nborder, SparseOut* o);
void sparse_border_fill(Ctx& c, const Geo& g, bool wide, const int64_t* border_off,
                        int32_t* border_ids, SparseOut* o);
void sparse_release(SparseOut* o);

// ---- cluster.cu (a8, a9) ----
void uf_init_list(Ctx& c, uint32_t* parent, const uint32_t* list, uint32_t m);  // list[0..m) only
void uf_flatten(Ctx& c, uint32_t* parent, const uint32_t* list, uint32_t m);  // parent[x] = Find(x)
void uf_init(Ctx& c, uint32_t* parent, uint32_t n);
// warp-per-pair BCP over list[0 .. min(*count, cap)) with Link on success
void bcp_large(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps, const uint32_t* core_cnt,
               uint32_t* parent, const uint2* list, const uint32_t* count, uint32_t cap, bool wide,
               const struct QTrees* qt = nullptr);
// *tested (device) counts pairs that survived the Find check of their wave;
// *npairs (device) receives the number of candidate pairs. nbr_total = CSR
// entries (bounds the pairs; no host synchronisation).
void cluster_core(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps, const uint32_t* core_cnt,
                  bool wide, bool waves, uint64_t nbr_total, uint32_t* parent,
                  unsigned long long* tested /*device, zeroed*/, unsigned long long* npairs,
                  const struct QTrees* qt = nullptr);
// Smallest core input index of a cell: its first point (stable radix sort and
// stable partition), cellmin[] for all-core cells (hash grouping: order inside
// a cell is arbitrary), or a scan of its core points (lattice counting sort).
enum { LABEL_MIN_FIRST = 0, LABEL_MIN_ARRAY = 1, LABEL_MIN_SCAN = 2 };
// core_list (optional): the ncore cells holding core points; the kernels then
// visit only those (cell_label of other cells is left unset: never read).
void labels(Ctx& c, const CellsView& cv, const uint32_t* idx, const uint8_t* core_s,
            const uint32_t* core_cnt, int min_mode, const uint32_t* cellmin, const uint32_t* core_list,
            uint32_t ncore, uint32_t* parent, int64_t n, uint32_t* cell_label,
            uint8_t* core_out, int32_t* cluster_out, uint32_t* counters /*device [4]*/);

// ---- border.cu (a10) ----
// count pass -> border_off (exclusive scan in input order, device int64[n+1],
// core points read as 0 through cluster[] >= 0); nnz = border_off[n] (no
// host synchronisation: the caller reads it).
void border_count(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps,
                     const uint32_t* idx, const uint32_t* core_cnt, const uint32_t* cell_label,
                     const int32_t* cluster, int64_t n, bool wide, int64_t* border_off,
                     unsigned long long* nborder /*device counter, zeroed*/);
void border_fill(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps,
                 const uint32_t* idx, const uint32_t* core_cnt, const uint32_t* cell_label, bool wide,
                 const int64_t* border_off, int32_t* border_ids);

// Dispatch on padded dimension D in {2,4,8} and the WIDE distance path.
template <typename F>
void dispatch(int D, bool wide, F&& f) {
  if (D == 2) { if (wide) f.template operator()<2, true>(); else f.template operator()<2, false>(); }
  else if (D == 4) { if (wide) f.template operator()<4, true>(); else f.template operator()<4, false>(); }
  else { if (wide) f.template operator()<8, true>(); else f.template operator()<8, false>(); }
}

inline unsigned grid_for(int64_t work, int threads, int cap) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

}  // namespace db
