// border.cu — ClusterBorder, Alg 4, PAPER.md P:L876-904:
// every non-core point p (they only live in cells with |g| < minPts)
// joins the cluster of every core point q in g or a neighbouring cell with
// d(p, q) <= eps; border points may belong to several clusters
// (P:L214-215). Output: a CSR over all points in input order, each row the
// ascending distinct cluster ids (reading 10).
// Shortcuts that do not change the output: all core points of one cell carry
// one label, so a core point in p's own cell gives that label without a
// distance test (same cell => within eps), and a neighbouring
// cell whose label is already in p's set is not scanned; within a cell the
// scan stops at the first core point within eps.
#include "internal.h"

namespace db {

constexpr int MAXL = 32;  // register-resident label set; larger sets use the slow path

struct LabelSet {
  uint32_t v[MAXL];
  int n = 0;
  bool overflow = false;
  __device__ bool has(uint32_t x) const {
    for (int i = 0; i < n; ++i)
      if (v[i] == x) return true;
    return false;
  }
  __device__ void add(uint32_t x) {  // keeps v[0..n) ascending
    if (n == MAXL) { overflow = true; return; }
    int i = n++;
    while (i > 0 && v[i - 1] > x) { v[i] = v[i - 1]; --i; }
    v[i] = x;
  }
};

template <int D, bool WIDE>
__device__ __forceinline__ bool cell_has_core_within(const int32_t* p, uint32_t h,
                                                     const CellsView& cv,
                                                     const int32_t* __restrict__ Ps,
                                                     const uint32_t* __restrict__ core_cnt,
                                                     uint32_t clampc, uint64_t eps2) {
  const uint32_t s = cv.cell_start[h], e = s + core_cnt[h];
  int32_t q[D];
  for (uint32_t u = s; u < e; ++u) {
    PtLoad<D>::load(Ps, u, q);
    DB_WORK(2);
    if (within<D, WIDE>(p, q, clampc, eps2)) return true;
  }
  return false;
}

// Smallest label > `after` among the clusters within eps of p (slow path for
// points with more than MAXL distinct labels); 0xffffffff if none.
template <int D, bool WIDE>
__device__ uint32_t next_label(const int32_t* p, uint32_t g, int64_t after, const CellsView& cv,
                               const int32_t* __restrict__ Ps, const uint32_t* __restrict__ core_cnt,
                               const uint32_t* __restrict__ cell_label, uint32_t clampc,
                               uint64_t eps2) {
  uint32_t best = 0xffffffffu;
  if (core_cnt[g] > 0 && (int64_t)cell_label[g] > after) best = cell_label[g];
  for (uint64_t t = cv.nbr_off[g]; t < cv.nbr_off[g + 1]; ++t) {
    const uint32_t h = cv.nbr[t];
    if (core_cnt[h] == 0) continue;
    const uint32_t lab = cell_label[h];
    if ((int64_t)lab <= after || lab >= best) continue;
    if (cell_has_core_within<D, WIDE>(p, h, cv, Ps, core_cnt, clampc, eps2)) best = lab;
  }
  return best;
}

// One non-core point j (sorted order): label set, then its CSR count (fill =
// 0) or row (fill = 1). Returns whether it is a border point.
template <int D, bool WIDE>
__device__ __forceinline__ bool border_point(int fill, uint32_t j, const CellsView& cv,
                                             const int32_t* __restrict__ Ps, const uint32_t* __restrict__ idx,
                                             const uint32_t* __restrict__ core_cnt,
                                             const uint32_t* __restrict__ cell_label, uint32_t clampc,
                                             uint64_t eps2, uint32_t* __restrict__ bcnt,
                                             const int64_t* __restrict__ border_off,
                                             int32_t* __restrict__ border_ids) {
  const uint32_t g = cv.cell_of[j];  // (the caller's cell; cell_of keeps this self-contained)
  int32_t p[D];
  PtLoad<D>::load(Ps, j, p);
  LabelSet L;
  if (core_cnt[g] > 0) L.add(cell_label[g]);
  for (uint64_t t = cv.nbr_off[g]; t < cv.nbr_off[g + 1] && !L.overflow; ++t) {
    const uint32_t h = cv.nbr[t];
    if (core_cnt[h] == 0) continue;
    const uint32_t lab = cell_label[h];
    if (L.has(lab)) continue;
    if (cell_has_core_within<D, WIDE>(p, h, cv, Ps, core_cnt, clampc, eps2)) L.add(lab);
  }
  const uint32_t i = idx[j];
  if (!L.overflow) {
    if (!fill) {
      bcnt[i] = (uint32_t)L.n;
    } else {
      int32_t* out = border_ids + border_off[i];
      for (int k = 0; k < L.n; ++k) out[k] = (int32_t)L.v[k];
    }
    return L.n > 0;
  }
  // slow path: enumerate labels in ascending order without storage
  uint32_t cnt = 0;
  int64_t after = -1;
  while (true) {
    const uint32_t nx = next_label<D, WIDE>(p, g, after, cv, Ps, core_cnt, cell_label, clampc, eps2);
    if (nx == 0xffffffffu) break;
    if (fill) border_ids[border_off[i] + cnt] = (int32_t)nx;
    ++cnt;
    after = nx;
  }
  if (!fill) bcnt[i] = cnt;
  return cnt > 0;
}

// Warp per cell (grid-stride), lanes over the cell's non-core points, which
// follow its core points (a7) and exist only in cells with |g| < minPts
// (P:L883); cells without non-core points cost one load.
template <int D, bool WIDE>
__global__ void __launch_bounds__(256, 4) border_kernel(
    int fill, CellsView cv, const int32_t* __restrict__ Ps, const uint32_t* __restrict__ idx,
    const uint32_t* __restrict__ core_cnt, const uint32_t* __restrict__ cell_label, uint32_t clampc,
    uint64_t eps2, uint32_t* __restrict__ bcnt, const int64_t* __restrict__ border_off,
    int32_t* __restrict__ border_ids, unsigned long long* nborder) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t nb = 0;
  for (uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < cv.ncells; g += nwarps) {
    const uint32_t e = cv.cell_start[g + 1];
    for (uint32_t j = cv.cell_start[g] + core_cnt[g] + lane; j < e; j += 32)
      nb += border_point<D, WIDE>(fill, j, cv, Ps, idx, core_cnt, cell_label, clampc, eps2, bcnt, border_off,
                                  border_ids);
  }
  if (!fill) block_add_u64(nb, nborder);
}

// Counts per non-core point (scattered to input order), then border_off =
// exclusive scan over all points with core points read as 0 (cluster >= 0),
// so the counts need no clearing; no border point at all: border_off = 0.
void border_count(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps,
                     const uint32_t* idx, const uint32_t* core_cnt, const uint32_t* cell_label,
                     const int32_t* cluster, int64_t n, bool wide, int64_t* border_off,
                     unsigned long long* nborder) {
  uint32_t* bcnt = c.alloc<uint32_t>(n);
  const unsigned grid = grid_for((int64_t)cv.ncells * 32, 256, c.sms * 16);
  dispatch(g.D, wide, [&]<int D, bool W>() {
    border_kernel<D, W><<<grid, 256, 0, c.st>>>(0, cv, Ps, idx, core_cnt, cell_label, g.clampc, g.eps2, bcnt,
                                                nullptr, nullptr, nborder);
  });
  c.launched();
  // (no border point at all: the scan writes zeros without reading the counts)
  exclusive_scan_u32_i64_masked(c, bcnt, cluster, border_off, n, nborder);
}

void border_fill(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps,
                 const uint32_t* idx, const uint32_t* core_cnt, const uint32_t* cell_label, bool wide,
                 const int64_t* border_off, int32_t* border_ids) {
  const unsigned grid = grid_for((int64_t)cv.ncells * 32, 256, c.sms * 16);
  dispatch(g.D, wide, [&]<int D, bool W>() {
    border_kernel<D, W><<<grid, 256, 0, c.st>>>(1, cv, Ps, idx, core_cnt, cell_label, g.clampc, g.eps2, nullptr,
                                                border_off, border_ids, nullptr);
  });
  c.launched();
}

}  // namespace db
