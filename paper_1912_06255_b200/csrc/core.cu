// core.cu — MarkCore and core compaction (a7).
//
// Alg 2: a cell with |g| >= minPts is all core
// (same cell => within eps); otherwise each point p
// counts |g| (its own cell, no distance test) plus RangeCount over the
// neighbouring cells and is core iff count >= minPts.
// Two output-preserving shortcuts (reading 13): counting stops once
// count >= minPts, and a sparse cell whose upper bound |g| + sum_h |h| is
// below minPts is all non-core without any distance test.
#include "internal.h"

namespace db {

enum : uint8_t { CELL_DENSE = 0, CELL_COUNT = 1, CELL_NONCORE = 2 };

__global__ void cell_class_kernel(CellsView cv, int64_t min_pts, uint8_t* __restrict__ cls) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= cv.ncells) return;
  const int64_t cnt = cv.cell_start[g + 1] - cv.cell_start[g];
  if (cnt >= min_pts) { cls[g] = CELL_DENSE; return; }
  int64_t ub = cnt;
  for (uint64_t t = cv.nbr_off[g]; t < cv.nbr_off[g + 1] && ub < min_pts; ++t) {
    uint32_t h = cv.nbr[t];
    ub += cv.cell_start[h + 1] - cv.cell_start[h];
  }
  cls[g] = ub >= min_pts ? CELL_COUNT : CELL_NONCORE;
}

// Thread per sorted point. Threads of one warp are consecutive points of the
// same or adjacent cells, so their neighbour-cell scans mostly read the same
// points (broadcast loads through L1).
template <int D, bool WIDE>
__global__ void __launch_bounds__(256) mark_core_kernel(CellsView cv, const uint8_t* __restrict__ cls,
                                                        const int32_t* __restrict__ Ps, uint32_t n,
                                                        int64_t min_pts, uint32_t clampc,
                                                        uint64_t eps2, uint8_t* __restrict__ core_s) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t g = cv.cell_of[j];
  const uint8_t c = cls[g];
  if (c != CELL_COUNT) { core_s[j] = c == CELL_DENSE; return; }
  int32_t p[D], q[D];
  PtLoad<D>::load(Ps, j, p);
  int64_t count = cv.cell_start[g + 1] - cv.cell_start[g];
  for (uint64_t t = cv.nbr_off[g]; t < cv.nbr_off[g + 1] && count < min_pts; ++t) {
    const uint32_t h = cv.nbr[t];
    const uint32_t e = cv.cell_start[h + 1];
    for (uint32_t u = cv.cell_start[h]; u < e; ++u) {
      PtLoad<D>::load(Ps, u, q);
      count += within<D, WIDE>(p, q, clampc, eps2);
      if (count >= min_pts) break;
    }
  }
  core_s[j] = count >= min_pts;
}

void mark_core(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps, int64_t n,
               int64_t min_pts, bool wide, uint8_t* core_s) {
  uint8_t* cls = c.alloc<uint8_t>(cv.ncells);
  cell_class_kernel<<<grid_for(cv.ncells, 256, 1 << 30), 256, 0, c.st>>>(cv, min_pts, cls);
  c.launched();
  dispatch(g.D, wide, [&]<int D, bool W>() {
    mark_core_kernel<D, W><<<grid_for(n, 256, 1 << 30), 256, 0, c.st>>>(
        cv, cls, Ps, (uint32_t)n, min_pts, g.clampc, g.eps2, core_s);
  });
  c.launched();
}

// ---------------------------------------------------------------- a7
// core_cnt[g] = number of core points in g. Cells with |g| >= minPts are all
// core; only cells with fewer points can be mixed.
__global__ void core_count_kernel(CellsView cv, const uint8_t* __restrict__ core_s, int64_t min_pts,
                                  uint32_t* __restrict__ core_cnt, uint32_t* __restrict__ mixed,
                                  uint32_t* __restrict__ counters) {
  uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  bool is_core_cell = false;
  if (g < cv.ncells) {
    const uint32_t s = cv.cell_start[g], e = cv.cell_start[g + 1];
    uint32_t k;
    if ((int64_t)(e - s) >= min_pts) {
      k = e - s;
    } else {
      k = 0;
      for (uint32_t u = s; u < e; ++u) k += core_s[u];
      if (k > 0 && k < e - s) {
        uint32_t slot = atomicAdd(counters + 1, 1u);
        mixed[slot] = g;
      }
    }
    core_cnt[g] = k;
    is_core_cell = k > 0;
  }
  uint32_t b = __ballot_sync(DB_FULL, is_core_cell);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(counters, __popc(b));
}

// Stable partition of one mixed cell: core points first, each group in its
// original (input-index) order. Thread per mixed cell via a scratch copy.
template <int D>
__global__ void partition_kernel(CellsView cv, const uint32_t* __restrict__ mixed,
                                 const uint32_t* __restrict__ nmixed, int32_t* __restrict__ Ps,
                                 uint32_t* __restrict__ idx, uint8_t* __restrict__ core_s,
                                 int32_t* __restrict__ scratchP, uint32_t* __restrict__ scratchI) {
  const uint32_t m = *nmixed;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
    const uint32_t g = mixed[t];
    const uint32_t s = cv.cell_start[g], e = cv.cell_start[g + 1];
    for (uint32_t u = s; u < e; ++u) {
      for (int k = 0; k < D; ++k) scratchP[(size_t)u * D + k] = Ps[(size_t)u * D + k];
      scratchI[u] = idx[u] | ((uint32_t)core_s[u] << 31);
    }
    uint32_t w = s;
    for (int pass = 1; pass >= 0; --pass)
      for (uint32_t u = s; u < e; ++u) {
        uint32_t v = scratchI[u];
        if ((v >> 31) != (uint32_t)pass) continue;
        for (int k = 0; k < D; ++k) Ps[(size_t)w * D + k] = scratchP[(size_t)u * D + k];
        idx[w] = v & 0x7fffffffu;
        core_s[w] = (uint8_t)pass;
        ++w;
      }
  }
}

void compact_core(Ctx& c, const Geo& g, const CellsView& cv, int32_t* Ps, uint32_t* idx,
                  uint8_t* core_s, int64_t n, int64_t min_pts, uint32_t* core_cnt,
                  uint32_t* counters) {
  uint32_t* mixed = c.alloc<uint32_t>(cv.ncells);
  core_count_kernel<<<grid_for(cv.ncells, 256, 1 << 30), 256, 0, c.st>>>(cv, core_s, min_pts,
                                                                          core_cnt, mixed, counters);
  c.launched();
  int32_t* sP = c.alloc<int32_t>((size_t)n * g.D);
  uint32_t* sI = c.alloc<uint32_t>(n);
  auto go = [&](auto Dc) {
    constexpr int D = decltype(Dc)::value;
    partition_kernel<D><<<c.sms * 4, 128, 0, c.st>>>(cv, mixed, counters + 1, Ps, idx, core_s, sP, sI);
  };
  if (g.D == 2) go(std::integral_constant<int, 2>());
  else if (g.D == 4) go(std::integral_constant<int, 4>());
  else go(std::integral_constant<int, 8>());
  c.launched();
}

}  // namespace db
