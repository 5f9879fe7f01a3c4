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

// Candidate points of one query (sum of neighbour-cell sizes, ub[g]) at or
// below this are scanned by one thread; above it by one warp.
constexpr uint32_t WARP_CANDIDATES = 32;
// Such a cell with at least this many points goes to the cell-tile kernel
// (a warp per cell, lanes over its points) instead of a warp per point.
constexpr int64_t TILE_MIN_POINTS = 4;
// (and the per-point kernel's point-box filter of neighbour cells: both pay
// from d = 6 on, ncu on SS-varden 5D / 7D and the BASELINE 5D / 7D configs)
constexpr int TILE_MIN_D = 6;

// Warp per cell (grid-stride), lanes over its points. With cnt = |g| and
// ub = sum of the neighbours' sizes (from the neighbour stage): cnt >= minPts
// -> all core (dense cell); cnt + ub < minPts -> none core without any
// distance test (the count can only be lower); otherwise count, in the lane
// if ub is small, else queue the point for the warp kernel.
template <int D, bool WIDE>
__global__ void __launch_bounds__(256) mark_core_kernel(CellsView cv, const int32_t* __restrict__ Ps,
                                                        int64_t min_pts, uint32_t clampc, uint64_t eps2,
                                                        uint8_t* __restrict__ core_s,
                                                        uint32_t* __restrict__ queue,
                                                        uint32_t* __restrict__ qcount,
                                                        uint32_t* __restrict__ cqueue,
                                                        uint32_t* __restrict__ cqcount, bool pre) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < cv.ncells; g += nwarps) {
    const uint32_t s = cv.cell_start[g], e = cv.cell_start[g + 1];
    const int64_t cnt = e - s;
    const uint32_t ub = cv.ub[g];
    if (cnt >= min_pts || cnt + (int64_t)ub < min_pts) {
      const uint8_t v = cnt >= min_pts;
      for (uint32_t u = s + lane; u < e; u += 32) core_s[u] = v;
      continue;
    }
    if (cqueue && ub > WARP_CANDIDATES && cnt >= TILE_MIN_POINTS) {  // the whole cell to the tile kernel
      if (lane == 0) cqueue[atomicAdd(cqcount, 1u)] = g;
      continue;
    }
    for (uint32_t j0 = s; j0 < e; j0 += 32) {
      const uint32_t j = j0 + lane;
      // (pre: points the sub-cell bounds proved core are set already)
      const bool valid = j < e && !(pre && core_s[j]);
      const bool enqueue = valid && ub > WARP_CANDIDATES;
      if (valid && !enqueue) {
        int32_t p[D], q[D];
        PtLoad<D>::load(Ps, j, p);
        int64_t count = cnt;
        for (uint64_t t = cv.nbr_off[g]; t < cv.nbr_off[g + 1] && count < min_pts; ++t) {
          const uint32_t h = cv.nbr[t];
          const uint32_t he = cv.cell_start[h + 1];
          for (uint32_t u = cv.cell_start[h]; u < he; ++u) {
            PtLoad<D>::load(Ps, u, q);
            DB_WORK(0);
            DB_WORK(3);
            count += within<D, WIDE>(p, q, clampc, eps2);
            if (count >= min_pts) break;
          }
        }
        core_s[j] = count >= min_pts;
      }
      // warp-aggregated append to the warp-kernel queue
      const uint32_t b = __ballot_sync(DB_FULL, enqueue);
      if (b) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(qcount, (uint32_t)__popc(b));
        base = __shfl_sync(DB_FULL, base, 0);
        if (enqueue) queue[base + __popc(b & lanemask_lt())] = j;
      }
    }
  }
}

// Warp per queued query point. The candidates (points of the neighbouring
// cells, 32 cells at a time) are flattened by a warp prefix sum over the cell
// sizes; lane l tests candidate t0 + l, found by a 5-step binary search over
// the lanes' exclusive offsets. Consecutive candidates of one cell are
// consecutive points, so the loads coalesce. The count is warp-uniform, so
// the exit at minPts is a uniform branch.
template <int D, bool WIDE>
__global__ void __launch_bounds__(256) mark_core_warp_kernel(CellsView cv, const int32_t* __restrict__ Ps,
                                                             const uint32_t* __restrict__ queue,
                                                             const uint32_t* __restrict__ qcount,
                                                             int64_t min_pts, Geo geo,
                                                             uint8_t* __restrict__ core_s, bool prune) {
  const int lane = threadIdx.x & 31;
  const uint32_t clampc = geo.clampc;
  const uint64_t eps2 = geo.eps2;
  const uint32_t m = *qcount;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < m; w += nwarps) {
    const uint32_t j = queue[w];
    const uint32_t g = cv.cell_of[j];
    int32_t p[D], q[D];
    PtLoad<D>::load(Ps, j, p);
    int64_t count = cv.cell_start[g + 1] - cv.cell_start[g];
    const uint64_t nb0 = cv.nbr_off[g], nb1 = cv.nbr_off[g + 1];
    for (uint64_t cb = nb0; cb < nb1 && count < min_pts; cb += 32) {
      const uint64_t t = cb + lane;
      uint32_t sz = 0, st = 0;
      if (t < nb1) {
        // (a neighbour cell whose box is beyond eps of p holds no candidate)
        const uint32_t h = cv.nbr[t];
        st = cv.cell_start[h];
        sz = cv.cell_start[h + 1] - st;
        if (prune && cb > nb0) {  // (from the second block of 32 cells: most points stop in the first)
          int64_t blo[D];
          cell_box_lo<D>(cv.cell_key[h], geo, blo);
          if (!near_box<D>(p, blo, geo)) sz = 0;
        }
      }
      const uint32_t incl = warp_inclusive_scan(sz);
      const uint32_t total = __shfl_sync(DB_FULL, incl, 31);
      const uint32_t excl = incl - sz;
      for (uint32_t t0 = 0; t0 < total && count < min_pts; t0 += 32) {
        const uint32_t tt = t0 + lane;
        int lo = 0;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          const uint32_t e = __shfl_sync(DB_FULL, excl, lo + s);
          if (e <= tt) lo += s;
        }
        const uint32_t ost = __shfl_sync(DB_FULL, st, lo);
        const uint32_t oex = __shfl_sync(DB_FULL, excl, lo);
        bool hit = false;
        if (tt < total) {
          DB_WORK(0);
          DB_WORK(3);
          PtLoad<D>::load(Ps, ost + (tt - oex), q);
          hit = within<D, WIDE>(p, q, clampc, eps2);
        }
        count += __popc(__ballot_sync(DB_FULL, hit));
      }
    }
    if (lane == 0) core_s[j] = count >= min_pts;
  }
}

// Cell-tile variant (CSR path): a warp per queued cell, a lane per point of
// the cell (32 at a time). The candidates — the points of the neighbouring
// cells, 32 cells at a time, flattened by a prefix sum as in the warp kernel
// — are staged 32 at a time in a per-warp shared-memory tile, one load per
// lane, and every lane tests its own point against each staged candidate
// (broadcast reads): a candidate load serves all the cell's points. Counting
// stops when every lane has reached minPts (Alg 2; reading 13).
template <int D>
__device__ __forceinline__ void tile_put(int32_t* t, const int32_t* q) {
  if constexpr (D == 2) {
    *reinterpret_cast<int2*>(t) = make_int2(q[0], q[1]);
  } else {
#pragma unroll
    for (int k = 0; k < D; k += 4) *reinterpret_cast<int4*>(t + k) = make_int4(q[k], q[k + 1], q[k + 2], q[k + 3]);
  }
}
template <int D>
__device__ __forceinline__ void tile_get(const int32_t* t, int32_t* q) {
  if constexpr (D == 2) {
    const int2 v = *reinterpret_cast<const int2*>(t);
    q[0] = v.x; q[1] = v.y;
  } else {
#pragma unroll
    for (int k = 0; k < D; k += 4) {
      const int4 v = *reinterpret_cast<const int4*>(t + k);
      q[k] = v.x; q[k + 1] = v.y; q[k + 2] = v.z; q[k + 3] = v.w;
    }
  }
}

template <int D, bool WIDE>
__global__ void __launch_bounds__(256, 4) mark_core_tile_kernel(CellsView cv, const int32_t* __restrict__ Ps,
                                                             const uint32_t* __restrict__ cqueue,
                                                             const uint32_t* __restrict__ cqcount,
                                                             int64_t min_pts, Geo geo,
                                                             uint8_t* __restrict__ core_s, bool pre) {
  const uint32_t clampc = geo.clampc;
  const uint64_t eps2 = geo.eps2;
  __shared__ __align__(16) int32_t tile[8][32 * D];
  const int lane = threadIdx.x & 31;
  int32_t* T = tile[threadIdx.x >> 5];
  const uint32_t m = *cqcount;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t need = (uint32_t)min(min_pts, (int64_t)0xffffffff);
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < m; w += nwarps) {
    const uint32_t g = cqueue[w];
    const uint32_t s = cv.cell_start[g], e = cv.cell_start[g + 1];
    const uint64_t nb0 = cv.nbr_off[g], nb1 = cv.nbr_off[g + 1];
    for (uint32_t j0 = s; j0 < e; j0 += 32) {
      const uint32_t j = j0 + lane;
      const bool live = j < e && !(pre && core_s[j]);
      if (!__any_sync(DB_FULL, live)) continue;
      int32_t p[D];
#pragma unroll
      for (int k = 0; k < D; ++k) p[k] = 0;
      if (live) PtLoad<D>::load(Ps, j, p);
      // bounding box of the live points: neighbour cells beyond eps of it are skipped
      int32_t qlo[D], qhi[D];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        qlo[k] = __reduce_min_sync(DB_FULL, live ? p[k] : INT32_MAX);
        qhi[k] = __reduce_max_sync(DB_FULL, live ? p[k] : INT32_MIN);
      }
      uint32_t count = e - s;  // its own cell (< minPts: not a dense cell)
      bool done = !live;
      for (uint64_t cb = nb0; cb < nb1; cb += 32) {
        const uint64_t t = cb + lane;
        uint32_t sz = 0, st = 0;
        if (t < nb1) {
          const uint32_t h = cv.nbr[t];
          int64_t blo[D];
          cell_box_lo<D>(cv.cell_key[h], geo, blo);
          if (near_box2<D>(qlo, qhi, blo, geo)) {
            st = cv.cell_start[h];
            sz = cv.cell_start[h + 1] - st;
          }
        }
        const uint32_t incl = warp_inclusive_scan(sz);
        const uint32_t total = __shfl_sync(DB_FULL, incl, 31);
        const uint32_t excl = incl - sz;
        for (uint32_t t0 = 0; t0 < total; t0 += 32) {
          const uint32_t tt = t0 + lane;
          int lo = 0;
#pragma unroll
          for (int sh = 16; sh >= 1; sh >>= 1) {
            const uint32_t ex = __shfl_sync(DB_FULL, excl, lo + sh);
            if (ex <= tt) lo += sh;
          }
          const uint32_t ost = __shfl_sync(DB_FULL, st, lo);
          const uint32_t oex = __shfl_sync(DB_FULL, excl, lo);
          if (tt < total) {
            int32_t q[D];
            PtLoad<D>::load(Ps, ost + (tt - oex), q);
            tile_put<D>(T + lane * D, q);
          }
          __syncwarp();
          const uint32_t nt = min(32u, total - t0);
          if (!done) {
            for (uint32_t u = 0; u < nt; ++u) {
              int32_t q[D];
              tile_get<D>(T + u * D, q);
              DB_WORK(0);
              DB_WORK(3);
              count += within<D, WIDE>(p, q, clampc, eps2) ? 1u : 0u;
            }
            done = count >= need;
          }
          __syncwarp();
          if (__all_sync(DB_FULL, done)) break;
        }
        if (__all_sync(DB_FULL, done)) break;
      }
      if (live) core_s[j] = count >= need;
    }
  }
}

// Tree variant of the warp kernel (row f2, our-exact-qt): neighbour cells
// with a tree are searched by a traversal of their tree instead
// of a scan: a node whose box is out of reach is skipped, a node whose box
// lies inside the eps-ball adds its count with no distance test (exact), a
// leaf's 32 points are tested by the lanes. Cells without a tree are scanned
// as in mark_core_warp_kernel. Decisions are warp-uniform.
constexpr uint32_t QT_MIN_CELL = 256;  // = QT_MIN in qtree.cu

template <int D>
__device__ __forceinline__ void box_dist2(const int32_t* p, const int32_t* __restrict__ bx, const Geo& g,
                                          uint64_t* dmin, uint64_t* dmax) {
  uint64_t mn = 0, mx = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < g.d) {
      const int64_t x = p[k], lo = bx[k], hi = bx[D + k];
      uint64_t a = (uint64_t)(x < lo ? lo - x : (x > hi ? x - hi : 0));
      uint64_t b = (uint64_t)max(x - lo, hi - x);
      if (a > g.clampc) a = g.clampc;
      if (b > g.clampc) b = g.clampc;
      mn += a * a;
      mx += b * b;
    }
  }
  *dmin = mn;
  *dmax = mx;
}

template <int D, bool WIDE>
__global__ void __launch_bounds__(256, 4) mark_core_qt_kernel(CellsView cv, const int32_t* __restrict__ Ps,
                                                           const uint32_t* __restrict__ queue,
                                                           const uint32_t* __restrict__ qcount, int64_t min_pts,
                                                           Geo g, QTrees qt, uint8_t* __restrict__ core_s) {
  const int lane = threadIdx.x & 31;
  const uint32_t m = *qcount;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < m; w += nwarps) {
    const uint32_t j = queue[w];
    const uint32_t gc = cv.cell_of[j];
    int32_t p[D], q[D];
    PtLoad<D>::load(Ps, j, p);
    int64_t count = cv.cell_start[gc + 1] - cv.cell_start[gc];
    const uint64_t nb1 = cv.nbr_off[gc + 1];
    for (uint64_t cb = cv.nbr_off[gc]; cb < nb1 && count < min_pts; cb += 32) {
      const uint64_t t = cb + lane;
      uint32_t sz = 0, st = 0, h = 0;
      bool tree = false;
      if (t < nb1) {
        h = cv.nbr[t];
        st = cv.cell_start[h];
        sz = cv.cell_start[h + 1] - st;
        tree = sz >= QT_MIN_CELL;
        if (tree) sz = 0;
      }
      // cells without a tree: flattened scan
      const uint32_t incl = warp_inclusive_scan(sz);
      const uint32_t total = __shfl_sync(DB_FULL, incl, 31);
      const uint32_t excl = incl - sz;
      for (uint32_t t0 = 0; t0 < total && count < min_pts; t0 += 32) {
        const uint32_t tt = t0 + lane;
        int lo = 0;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          const uint32_t e = __shfl_sync(DB_FULL, excl, lo + s);
          if (e <= tt) lo += s;
        }
        const uint32_t ost = __shfl_sync(DB_FULL, st, lo);
        const uint32_t oex = __shfl_sync(DB_FULL, excl, lo);
        bool hit = false;
        if (tt < total) {
          PtLoad<D>::load(Ps, ost + (tt - oex), q);
          DB_WORK(0);
          DB_WORK(3);
          hit = within<D, WIDE>(p, q, g.clampc, g.eps2);
        }
        count += __popc(__ballot_sync(DB_FULL, hit));
      }
      // cells with a tree: one traversal each
      uint32_t tm = __ballot_sync(DB_FULL, tree);
      while (tm && count < min_pts) {
        const int src = __ffs(tm) - 1;
        tm &= tm - 1;
        const uint32_t hc = __shfl_sync(DB_FULL, h, src);
        const uint32_t s0 = cv.cell_start[hc], e0 = cv.cell_start[hc + 1];
        uint32_t L = (e0 - s0 + 31) / 32, P2 = 1;
        while (P2 < L) P2 <<= 1;
        const uint64_t base = qt.node_off[hc];
        uint32_t stack[64];
        int sp = 0;
        stack[sp++] = 0;
        while (sp > 0 && count < min_pts) {
          const uint32_t node = stack[--sp];
          if (node >= P2 - 1) {  // leaf: lanes test its points
            const uint32_t u = s0 + (node - (P2 - 1)) * 32 + lane;
            bool hit = false;
            if (u < e0) {
              PtLoad<D>::load(Ps, u, q);
              DB_WORK(0);
              DB_WORK(3);
          hit = within<D, WIDE>(p, q, g.clampc, g.eps2);
            }
            count += __popc(__ballot_sync(DB_FULL, hit));
            continue;
          }
          for (uint32_t ch = 2 * node + 2; ch >= 2 * node + 1; --ch) {  // left child on top
            const uint32_t nc = qt.cnt[base + ch];
            if (nc == 0) continue;
            uint64_t dmin, dmax;
            box_dist2<D>(p, qt.box + (base + ch) * 2 * D, g, &dmin, &dmax);
            if (dmin > g.eps2) continue;
            if (dmax <= g.eps2) { count += nc; continue; }  // box inside the ball
            stack[sp++] = ch;
          }
        }
      }
    }
    if (lane == 0) core_s[j] = count >= min_pts;
  }
}

void mark_core(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps, int64_t n,
               int64_t min_pts, bool wide, uint8_t* core_s, const QTrees* qt, bool pre) {
  uint32_t* queue = c.alloc<uint32_t>(n);
  uint32_t* qcount = c.alloc<uint32_t>(2);  // [0] points, [1] cells
  const bool use_qt = qt && qt->nodes;
  // the cell tiles pay where a point needs many candidates to reach minPts:
  // high d, where the eps-ball fills a small part of its neighbour cells
  const bool tiles = !use_qt && g.d >= TILE_MIN_D;
  uint32_t* cqueue = tiles ? c.alloc<uint32_t>(cv.ncells) : nullptr;
  c.zero(qcount, 2 * sizeof(uint32_t));
  dispatch(g.D, wide, [&]<int D, bool W>() {
    mark_core_kernel<D, W><<<grid_for((int64_t)cv.ncells * 32, 256, c.sms * 16), 256, 0, c.st>>>(
        cv, Ps, min_pts, g.clampc, g.eps2, core_s, queue, qcount, cqueue, qcount + 1, pre);
    c.launched();
    if (use_qt) {
      mark_core_qt_kernel<D, W><<<c.sms * 16, 256, 0, c.st>>>(cv, Ps, queue, qcount, min_pts, g, *qt, core_s);
    } else {
      if (tiles) {
        mark_core_tile_kernel<D, W><<<c.sms * 8, 256, 0, c.st>>>(cv, Ps, cqueue, qcount + 1, min_pts, g, core_s,
                                                                 pre);
        c.launched();
      }
      mark_core_warp_kernel<D, W><<<c.sms * 16, 256, 0, c.st>>>(cv, Ps, queue, qcount, min_pts, g, core_s,
                                                                 g.d >= TILE_MIN_D);
    }
    c.launched();
  });
}

// ---------------------------------------------------------------- a7
// core_cnt[g] = number of core points in g. Cells with |g| >= minPts are all
// core; only cells with fewer points can be mixed.
__global__ void __launch_bounds__(256) core_count_kernel(CellsView cv, const uint8_t* __restrict__ core_s,
                                                         int64_t min_pts, uint32_t* __restrict__ core_cnt,
                                                         uint32_t* __restrict__ mixed,
                                                         uint32_t* __restrict__ counters) {
  __shared__ uint32_t s_scan[33];
  __shared__ uint32_t s_base;
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  bool is_core_cell = false, is_mixed = false;
  uint32_t s = 0, e = 0, k = 0;
  bool big = false;  // more than 64 points below minPts: counted by the whole warp
  if (g < cv.ncells) {
    s = cv.cell_start[g];
    e = cv.cell_start[g + 1];
    if ((int64_t)(e - s) >= min_pts) {
      k = e - s;
    } else if (e - s > 64) {
      big = true;
    } else {
      for (uint32_t u = s; u < e; ++u) k += core_s[u];
    }
  }
  // the block's large cells, spread over its warps (a warp per cell)
  __shared__ uint32_t s_nbig, s_big[256], s_k[256];
  if (threadIdx.x == 0) s_nbig = 0;
  __syncthreads();
  if (big) s_big[atomicAdd(&s_nbig, 1u)] = threadIdx.x;
  __syncthreads();
  for (uint32_t q = threadIdx.x >> 5; q < s_nbig; q += blockDim.x >> 5) {
    const uint32_t gg = blockIdx.x * blockDim.x + s_big[q];
    const uint32_t cs = cv.cell_start[gg], ce = cv.cell_start[gg + 1];
    uint32_t part = 0;
    for (uint32_t u = cs + (threadIdx.x & 31u); u < ce; u += 32) part += core_s[u];
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(DB_FULL, part, o);
    if ((threadIdx.x & 31u) == 0) s_k[s_big[q]] = part;
  }
  __syncthreads();
  if (big) k = s_k[threadIdx.x];
  if (g < cv.ncells) {
    if ((int64_t)(e - s) < min_pts) is_mixed = k > 0 && k < e - s;
    core_cnt[g] = k;
    is_core_cell = k > 0;
  }
  const uint32_t b = __syncthreads_count(is_core_cell);  // one atomic per block
  if (threadIdx.x == 0 && b) atomicAdd(counters, b);
  uint32_t nm;
  const uint32_t ex = block_exclusive_scan<uint32_t>(is_mixed ? 1u : 0u, s_scan, &nm);
  if (threadIdx.x == 0 && nm) s_base = atomicAdd(counters + 1, nm);
  __syncthreads();
  if (is_mixed) mixed[s_base + ex] = g;
}

// Stable partition of the mixed cells: core points first, each group in its
// original (input-index) order. A warp takes 32 mixed cells: a cell of <= 8
// points is partitioned by its lane in registers (sparse lattices); the
// larger ones by the whole warp, one after the other — 32 points per step
// to their places in a scratch copy (ballot ranks: the core ones from the
// cell start, the others after its core_cnt core points), then copied back
// coalesced. (A thread per large cell made SS-simden 3D at minPts 3e4 spend
// 11.5 ms here: cells of tens of thousands of points done serially.)
template <int D>
__global__ void partition_kernel(CellsView cv, const uint32_t* __restrict__ mixed,
                                 const uint32_t* __restrict__ nmixed, const uint32_t* __restrict__ core_cnt,
                                 int32_t* __restrict__ Ps, uint32_t* __restrict__ idx,
                                 uint8_t* __restrict__ core_s, int32_t* __restrict__ scratchP,
                                 uint32_t* __restrict__ scratchI, uint32_t* __restrict__ inv) {
  const uint32_t m = *nmixed;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = lanemask_lt();
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  // the small cells (<= 8 points, D <= 4), a lane per cell over chunks of 32
  if constexpr (D <= 4)
  for (uint32_t t0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; t0 < m; t0 += nwarps * 32) {
    const uint32_t t = t0 + lane;
    uint32_t g = 0, s = 0, e = 0;
    if (t < m) {
      g = mixed[t];
      s = cv.cell_start[g];
      e = cv.cell_start[g + 1];
    }
    if constexpr (D <= 4) {
      const bool big = t < m && e - s > 8;
      if (t < m && !big) {  // small cell: in registers, no scratch round trip
        constexpr int SM = 8;
        int32_t P[SM][D];
        uint32_t I[SM];
        uint8_t C[SM];
        const uint32_t nn = e - s;
#pragma unroll
        for (int q = 0; q < SM; ++q)
          if ((uint32_t)q < nn) {
            PtLoad<D>::load(Ps, s + q, P[q]);
            I[q] = idx[s + q];
            C[q] = core_s[s + q];
          }
        uint32_t w = s;
#pragma unroll
        for (int pass = 1; pass >= 0; --pass)
#pragma unroll
          for (int q = 0; q < SM; ++q)
            if ((uint32_t)q < nn && C[q] == pass) {
              if constexpr (D == 2) reinterpret_cast<int2*>(Ps)[w] = make_int2(P[q][0], P[q][1]);
              else reinterpret_cast<int4*>(Ps)[w] = make_int4(P[q][0], P[q][1], P[q][2], P[q][3]);
              idx[w] = I[q];
              core_s[w] = (uint8_t)pass;
              if (inv) inv[I[q]] = w;
              ++w;
            }
      }
    }
  }
  // the large cells (> 8 points; all of them for D = 8), a warp per cell
  for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < m; t += nwarps) {
    {
      const uint32_t gs = mixed[t];
      const uint32_t cs = cv.cell_start[gs], ce = cv.cell_start[gs + 1];
      if (D <= 4 && ce - cs <= 8) continue;  // (warp-uniform)
      const uint32_t kc = core_cnt[gs];
      uint32_t nc = 0, nn = 0;  // core / other points placed so far
      for (uint32_t u0 = cs; u0 < ce; u0 += 32) {
        const uint32_t u = u0 + lane;
        const bool valid = u < ce;
        const uint32_t c = valid ? core_s[u] : 0u;
        int32_t P[D];
        uint32_t I = 0;
        if (valid) {
          PtLoad<D>::load(Ps, u, P);
          I = idx[u];
        }
        const uint32_t bc = __ballot_sync(DB_FULL, valid && c), bn = __ballot_sync(DB_FULL, valid && !c);
        if (valid) {
          const uint32_t pos = c ? cs + nc + __popc(bc & lt) : cs + kc + nn + __popc(bn & lt);
#pragma unroll
          for (int k = 0; k < D; ++k) scratchP[(size_t)pos * D + k] = P[k];
          scratchI[pos] = I | (c << 31);
        }
        nc += __popc(bc);
        nn += __popc(bn);
      }
      __syncwarp();
      for (uint32_t u = cs + lane; u < ce; u += 32) {
        const uint32_t v = scratchI[u];
#pragma unroll
        for (int k = 0; k < D; ++k) Ps[(size_t)u * D + k] = scratchP[(size_t)u * D + k];
        idx[u] = v & 0x7fffffffu;
        core_s[u] = (uint8_t)(v >> 31);
        if (inv) inv[v & 0x7fffffffu] = u;
      }
      __syncwarp();
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
  partition_mixed(c, g, cv, mixed, counters + 1, core_cnt, Ps, idx, core_s, n);
}

void partition_mixed(Ctx& c, const Geo& g, const CellsView& cv, const uint32_t* mixed,
                     const uint32_t* nmixed, const uint32_t* core_cnt, int32_t* Ps, uint32_t* idx,
                     uint8_t* core_s, int64_t n) {
  int32_t* sP = c.alloc<int32_t>((size_t)n * g.D);
  uint32_t* sI = c.alloc<uint32_t>(n);
  auto go = [&](auto Dc) {
    constexpr int D = decltype(Dc)::value;
    partition_kernel<D><<<c.sms * 16, 256, 0, c.st>>>(cv, mixed, nmixed, core_cnt, Ps, idx, core_s, sP, sI, c.inv);
  };
  if (g.D == 2) go(std::integral_constant<int, 2>());
  else if (g.D == 4) go(std::integral_constant<int, 4>());
  else go(std::integral_constant<int, 8>());
  c.launched();
}

}  // namespace db
