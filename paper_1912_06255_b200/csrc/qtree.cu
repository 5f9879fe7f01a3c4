// qtree.cu — per-cell trees for RangeCount (the paper's
// our-exact-qt: PAPER.md §"Range Counting").
//
// The paper divides each cell (side eps/sqrt(d)) recursively into 2^d
// sub-cells until they are empty or small, each node storing its point count
// (P:L960-967), builds the trees in parallel by integer-sorting the points of
// a node by sub-cell, and answers RangeCount(p, eps, h) by a
// traversal that descends only into sub-cells intersecting the eps-ball of p
// and counts points explicitly at the leaves.
//
// GPU form (DESIGN.md §5 f2): the points of every cell with at least QT_MIN
// points are ordered by sub-cell of the 2^d-ary subdivision B levels deep
// (Morton order of the sub-cells, d B <= 12) with a counting sort per cell in
// shared memory; the tree over that order is implicit and
// binary — leaves of QT_LEAF consecutive points, a complete binary tree above
// them (node i has children 2i+1, 2i+2) — so every node is a run of points
// sharing a Morton prefix, i.e. a union of quadtree sub-cells. Each node keeps
// the integer bounding box of its points and their count. A query visits a
// node only if its box intersects the eps-ball; a node whose box lies inside
// the ball adds its count without any distance test (exact: every point of
// the box is within eps); leaves test their points, a warp's lanes at once.
#include <algorithm>

#include "internal.h"

namespace db {

constexpr uint32_t QT_MIN = 256;   // cells with at least this many points get a tree
constexpr int QT_LEAF = 32;        // points per leaf (a warp tests a leaf at once)

__device__ __forceinline__ uint32_t qt_leaves(uint32_t m) {
  uint32_t L = (m + QT_LEAF - 1) / QT_LEAF, P2 = 1;
  while (P2 < L) P2 <<= 1;
  return P2;
}

// Block per tree cell: counting sort of its points by sub-cell (the top B
// levels of the 2^d-ary subdivision, d B <= 12: up to 4096 sub-cells), the
// paper's per-node integer sort on sub-cell keys done once for
// B levels; then copied back in place. Order inside a sub-cell is the atomics'.
constexpr int QT_SUB_BITS = 12;

// (qstart != NULL: also writes, for cell c with tree index tidx[c], the
// cell-relative start of each of its 2^(B d) sub-cells and the cell size at
// qstart[tidx[c] * (2^(B d) + 1) ..], the per-node counts of the bounds below)
template <int D>
__global__ void __launch_bounds__(1024) qt_sort_cells_kernel(int32_t* __restrict__ Ps, uint32_t* __restrict__ idx,
                                                             const uint32_t* __restrict__ cell_start,
                                                             const uint64_t* __restrict__ cell_key, uint32_t ncells,
                                                             Geo g, int B, int32_t* __restrict__ Ps2,
                                                             uint32_t* __restrict__ idx2, uint32_t min_size,
                                                             const uint32_t* __restrict__ tidx,
                                                             uint32_t* __restrict__ qstart,
                                                             uint32_t* __restrict__ inv) {
  __shared__ uint32_t hist[1 << QT_SUB_BITS];
  __shared__ uint32_t s_scan[33];
  const int NB = 1 << (B * g.d);
  for (uint32_t c = blockIdx.x; c < ncells; c += gridDim.x) {
    const uint32_t s = cell_start[c], e = cell_start[c + 1];
    if (e - s < min_size) continue;  // uniform per block
    const uint64_t key = cell_key[c];
    int64_t base[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      base[k] = k < g.d ? (int64_t)g.lo[k] + (int64_t)cell_coord(key, g, k) * (int64_t)g.s : 0;
    auto sub_of = [&](const int32_t* x) -> uint32_t {
      uint32_t q[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        q[k] = k < g.d ? (uint32_t)((((uint64_t)((int64_t)x[k] - base[k])) << B) / g.s) : 0u;
      uint32_t code = 0;
      for (int b = B - 1; b >= 0; --b)
        for (int k = 0; k < g.d; ++k) code = (code << 1) | ((q[k] >> b) & 1u);
      return code;
    };
    for (int i = threadIdx.x; i < NB; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (uint32_t j = s + threadIdx.x; j < e; j += blockDim.x) {
      int32_t x[D];
      PtLoad<D>::load(Ps, j, x);
      atomicAdd(hist + sub_of(x), 1u);
    }
    __syncthreads();
    // exclusive scan of hist (blockDim = 1024 threads x 4 bins)
    {
      const int per = (NB + (int)blockDim.x - 1) / (int)blockDim.x;
      uint32_t v[4] = {0, 0, 0, 0}, sum = 0;
      for (int t = 0; t < per && t < 4; ++t) {
        const int i = threadIdx.x * per + t;
        v[t] = i < NB ? hist[i] : 0u;
        sum += v[t];
      }
      uint32_t tot;
      uint32_t ex = block_exclusive_scan<uint32_t>(sum, s_scan, &tot);
      uint32_t* qs = qstart ? qstart + (size_t)tidx[c] * (NB + 1) : nullptr;
      for (int t = 0; t < per && t < 4; ++t) {
        const int i = threadIdx.x * per + t;
        if (i < NB) {
          hist[i] = ex;
          if (qs) qs[i] = ex;
        }
        ex += v[t];
      }
      if (qs && threadIdx.x == 0) qs[NB] = e - s;
    }
    __syncthreads();
    for (uint32_t j = s + threadIdx.x; j < e; j += blockDim.x) {
      int32_t x[D];
      PtLoad<D>::load(Ps, j, x);
      const uint32_t pos = s + atomicAdd(hist + sub_of(x), 1u);
#pragma unroll
      for (int k = 0; k < D; ++k) Ps2[(size_t)pos * D + k] = x[k];
      idx2[pos] = idx[j];
    }
    __syncthreads();
    __threadfence_block();
    for (uint32_t j = s + threadIdx.x; j < e; j += blockDim.x) {
#pragma unroll
      for (int k = 0; k < D; ++k) Ps[(size_t)j * D + k] = Ps2[(size_t)j * D + k];
      idx[j] = idx2[j];
      if (inv) inv[idx2[j]] = j;
    }
    __syncthreads();
  }
}

__global__ void qt_nodes_count_kernel(const uint32_t* __restrict__ cell_start, uint32_t ncells,
                                      uint32_t* __restrict__ nnodes) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const uint32_t m = cell_start[c + 1] - cell_start[c];
  nnodes[c] = m >= QT_MIN ? 2 * qt_leaves(m) - 1 : 0;
}

// Warp per leaf slot of every tree cell: the leaf's box and count, then the
// lane-0 thread climbs: the second child to arrive at a node builds it.
template <int D>
__global__ void __launch_bounds__(256) qt_build_kernel(const int32_t* __restrict__ Ps,
                                                       const uint32_t* __restrict__ cell_start, uint32_t ncells,
                                                       const uint64_t* __restrict__ node_off, int d,
                                                       int32_t* box, uint32_t* cnt, uint32_t* flags,
                                                       const uint32_t* __restrict__ leaf_cell,
                                                       const uint32_t* __restrict__ leaf_idx, uint64_t nleaves) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nleaves; w += nwarps) {
    const uint32_t c = leaf_cell[w], lf = leaf_idx[w];
    const uint32_t s = cell_start[c], e = cell_start[c + 1];
    const uint32_t P2 = qt_leaves(e - s);
    const uint64_t base = node_off[c];
    const uint32_t u = s + lf * QT_LEAF + lane;
    const bool ok = u < e && lf * QT_LEAF < e - s;
    int32_t x[D];
    if (ok) PtLoad<D>::load(Ps, u, x);
    int32_t lo[D], hi[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      int32_t l = ok ? x[k] : INT32_MAX, h = ok ? x[k] : INT32_MIN;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        l = min(l, __shfl_xor_sync(DB_FULL, l, o));
        h = max(h, __shfl_xor_sync(DB_FULL, h, o));
      }
      lo[k] = l; hi[k] = h;
    }
    const uint32_t nl = (uint32_t)__popc(__ballot_sync(DB_FULL, ok));
    if (lane == 0) {
      uint64_t node = P2 - 1 + lf;
      for (int k = 0; k < D; ++k) { box[(base + node) * 2 * D + k] = lo[k]; box[(base + node) * 2 * D + D + k] = hi[k]; }
      cnt[base + node] = nl;
      uint32_t cnt_acc = nl;
      while (node > 0) {
        __threadfence();
        const uint64_t parent = (node - 1) >> 1;
        if (atomicAdd(flags + base + parent, 1u) == 0) break;  // the sibling builds it
        __threadfence();
        const uint64_t sib = (node & 1) ? node + 1 : node - 1;
        const volatile int32_t* sb = box + (base + sib) * 2 * D;
        for (int k = 0; k < D; ++k) { lo[k] = min(lo[k], sb[k]); hi[k] = max(hi[k], sb[D + k]); }
        cnt_acc += ((volatile uint32_t*)cnt)[base + sib];
        for (int k = 0; k < D; ++k) {
          box[(base + parent) * 2 * D + k] = lo[k];
          box[(base + parent) * 2 * D + D + k] = hi[k];
        }
        cnt[base + parent] = cnt_acc;
        node = parent;
      }
    }
    __syncwarp();
  }
  (void)d;
  (void)ncells;
}

__global__ void qt_leaf_list_kernel(const uint32_t* __restrict__ cell_start, uint32_t ncells,
                                    const uint64_t* __restrict__ leaf_off, uint32_t* __restrict__ leaf_cell,
                                    uint32_t* __restrict__ leaf_idx) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const uint32_t m = cell_start[c + 1] - cell_start[c];
  if (m < QT_MIN) return;
  const uint32_t P2 = qt_leaves(m);
  const uint64_t o = leaf_off[c];
  for (uint32_t l = 0; l < P2; ++l) { leaf_cell[o + l] = c; leaf_idx[o + l] = l; }
}

__global__ void qt_leaf_count_kernel(const uint32_t* __restrict__ cell_start, uint32_t ncells,
                                     uint32_t* __restrict__ nl) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const uint32_t m = cell_start[c + 1] - cell_start[c];
  nl[c] = m >= QT_MIN ? qt_leaves(m) : 0;
}

void build_qtrees(Ctx& c, const Geo& g, const CellsView& cv, int32_t* Ps, uint32_t* idx, int64_t n, QTrees* qt) {
  const uint32_t nc = cv.ncells;
  // 1. order the points of every tree cell by sub-cell (block per cell)
  const int B = std::max(1, QT_SUB_BITS / g.d);
  int32_t* Ps2 = c.alloc<int32_t>((size_t)n * g.D);
  uint32_t* idx2 = c.alloc<uint32_t>(n);
  auto byD = [&](auto f) {
    if (g.D == 2) f(std::integral_constant<int, 2>());
    else if (g.D == 4) f(std::integral_constant<int, 4>());
    else f(std::integral_constant<int, 8>());
  };
  byD([&](auto Dc) {
    constexpr int D = decltype(Dc)::value;
    qt_sort_cells_kernel<D><<<std::min<uint32_t>(nc, (uint32_t)c.sms * 8), 1024, 0, c.st>>>(
        Ps, idx, cv.cell_start, cv.cell_key, nc, g, B, Ps2, idx2, QT_MIN, nullptr, nullptr, c.inv);
  });
  c.launched();
  // 2. node offsets and leaf lists
  uint32_t* nn = c.alloc<uint32_t>(nc);
  uint64_t* node_off = c.alloc<uint64_t>((size_t)nc + 1);
  qt_nodes_count_kernel<<<grid_for(nc, 256, 1 << 30), 256, 0, c.st>>>(cv.cell_start, nc, nn);
  c.launched();
  exclusive_scan_u32_u64(c, nn, node_off, nc);
  uint32_t* nl = c.alloc<uint32_t>(nc);
  uint64_t* leaf_off = c.alloc<uint64_t>((size_t)nc + 1);
  qt_leaf_count_kernel<<<grid_for(nc, 256, 1 << 30), 256, 0, c.st>>>(cv.cell_start, nc, nl);
  c.launched();
  exclusive_scan_u32_u64(c, nl, leaf_off, nc);
  uint64_t tot[2];
  const uint64_t* t0 = c.fetch(node_off + nc, 1);
  const uint64_t* t1 = c.fetch(leaf_off + nc, 1);
  c.sync();
  tot[0] = *t0;
  tot[1] = *t1;
  qt->node_off = node_off;
  qt->nodes = tot[0];
  if (tot[0] == 0) { qt->box = nullptr; qt->cnt = nullptr; return; }
  int32_t* box = c.alloc<int32_t>(tot[0] * 2 * g.D);
  uint32_t* cnt = c.alloc<uint32_t>(tot[0]);
  uint32_t* flags = c.alloc<uint32_t>(tot[0]);
  c.zero(flags, sizeof(uint32_t) * tot[0]);
  uint32_t* leaf_cell = c.alloc<uint32_t>(tot[1]);
  uint32_t* leaf_idx = c.alloc<uint32_t>(tot[1]);
  qt_leaf_list_kernel<<<grid_for(nc, 256, 1 << 30), 256, 0, c.st>>>(cv.cell_start, nc, leaf_off, leaf_cell,
                                                                    leaf_idx);
  c.launched();
  byD([&](auto Dc) {
    constexpr int D = decltype(Dc)::value;
    qt_build_kernel<D><<<grid_for((int64_t)tot[1] * 32, 256, c.sms * 16), 256, 0, c.st>>>(
        Ps, cv.cell_start, nc, node_off, g.d, box, cnt, flags, leaf_cell, leaf_idx, tot[1]);
  });
  c.launched();
  qt->box = box;
  qt->cnt = cnt;
}

// ===========================================================================
// MarkCore lower bounds from sub-cell counts (row f2; the paper's quadtree
// RangeCount: a node whose region lies inside the eps-ball adds
// its count without distance tests). For large minPts, Alg 2's per-point
// count needs up to minPts hits per point; on clustered data
// almost every such point has far more than minPts neighbours (SS-simden 3D
// at minPts = 10^4: 2.8M points to count, 99.9% of them core with > 2.4 10^4
// neighbours). So, before the exact counts:
//  * every cell with >= QB_MIN points is subdivided 2^(B d) ways (its points
//    ordered by sub-cell, Morton order, so every node of the implicit 2^d-ary
//    tree is a run of points, its count a difference of two starts);
//  * a warp per QUERY sub-cell Q (level LQ of a cell that needs counting)
//    accumulates a lower bound L = |g| (own cell: within eps) +
//    the counts of the neighbouring cells and tree nodes whose box lies
//    entirely within eps of Q's box (max box distance <= eps: every point of
//    the node is within eps of every point of Q), descending into nodes that
//    are neither inside nor out of reach, nearest cells first, until
//    L >= minPts: then every point of Q is core (L never exceeds its count).
//  * the points not decided this way are counted exactly by the usual
//    MarkCore kernels.
// ===========================================================================
constexpr uint32_t QB_MIN = 256;   // cells with at least this many points are subdivided
constexpr int QB_BITS = 10;        // at most 2^10 sub-cells per cell
constexpr int QB_FRONT = 1 << QB_BITS;
constexpr uint32_t QB_NONE = 0xffffffffu;

struct QBArgs {
  Geo g;
  CellsView cv;
  const uint32_t* tidx;    // [ncells] tree index or QB_NONE
  const uint32_t* tlist;   // [ntree] cell of each tree index
  const uint32_t* qstart;  // [ntree * (NS + 1)] cell-relative sub-cell starts (level B)
  const uint32_t* ntree;   // device count
  int B, LQ, NS;
  int64_t min_pts;
  uint8_t* core_s;
  unsigned long long* decided;
};

__global__ void qb_flags_kernel(const uint32_t* __restrict__ cell_start, uint32_t ncells, uint32_t* __restrict__ f) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ncells) f[c] = cell_start[c + 1] - cell_start[c] >= QB_MIN ? 1u : 0u;
}

__global__ void qb_index_kernel(const uint32_t* __restrict__ f, const uint32_t* __restrict__ pos, uint32_t ncells,
                                uint32_t* __restrict__ tidx, uint32_t* __restrict__ tlist) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  tidx[c] = f[c] ? pos[c] : QB_NONE;
  if (f[c]) tlist[pos[c]] = c;
}

// lattice box of the sub-cell with Morton prefix P (level l) of the cell with
// lattice coordinates cc: x is in sub-cell j of axis k iff
// floor((x - base_k) 2^l / s) = j, i.e. x - base_k in [ceil(j s / 2^l), ceil((j+1) s / 2^l) - 1]
template <int D>
__device__ __forceinline__ void qb_box(const Geo& g, const uint32_t* cc, uint32_t P, int l, int64_t* lo,
                                       int64_t* hi) {
  uint32_t j[D];
#pragma unroll
  for (int k = 0; k < D; ++k) j[k] = 0;
  for (int i = 0; i < l; ++i)
#pragma unroll
    for (int k = 0; k < D; ++k)
      if (k < g.d) j[k] = (j[k] << 1) | ((P >> ((l - 1 - i) * g.d + (g.d - 1 - k))) & 1u);
  const uint64_t den = 1ull << l;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < g.d) {
      const int64_t base = (int64_t)g.lo[k] + (int64_t)cc[k] * (int64_t)g.s;
      lo[k] = base + (int64_t)(((uint64_t)j[k] * g.s + den - 1) >> l);
      hi[k] = base + (int64_t)((((uint64_t)j[k] + 1) * g.s + den - 1) >> l) - 1;
    } else {
      lo[k] = hi[k] = 0;
    }
  }
}

// 1: every pair of points of the two boxes within eps; -1: no pair; 0: some
template <int D>
__device__ __forceinline__ int qb_classify(const Geo& g, const int64_t* alo, const int64_t* ahi, const int64_t* blo,
                                           const int64_t* bhi) {
  uint64_t mn = 0, mx = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < g.d) {
      int64_t a = blo[k] - ahi[k], b = alo[k] - bhi[k];
      uint64_t t = (uint64_t)max((int64_t)0, max(a, b));
      uint64_t u = (uint64_t)max(bhi[k] - alo[k], ahi[k] - blo[k]);
      if (t > g.clampc) t = g.clampc;
      if (u > g.clampc) u = g.clampc;
      mn += t * t;
      mx += u * u;
    }
  }
  return mx <= g.eps2 ? 1 : (mn > g.eps2 ? -1 : 0);
}

template <int D>
__global__ void __launch_bounds__(256) qb_bound_kernel(QBArgs A) {
  __shared__ uint16_t s_front[8][2][QB_FRONT];
  const int lane = threadIdx.x & 31;
  uint16_t(*F)[QB_FRONT] = s_front[threadIdx.x >> 5];
  const Geo& g = A.g;
  const int d = g.d;
  const uint32_t nq = 1u << (A.LQ * d);
  const uint64_t total = (uint64_t)(*A.ntree) * nq;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int shq = (A.B - A.LQ) * d;
  unsigned long long dec = 0;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < total; w += nw) {
    const uint32_t t = (uint32_t)(w / nq), q = (uint32_t)(w % nq);
    const uint32_t gc = A.tlist[t];
    const uint32_t s0 = A.cv.cell_start[gc], m = A.cv.cell_start[gc + 1] - s0;
    // cells that need no count (dense, or all non-core by the bound ub) are
    // decided by mark_core_kernel
    if ((int64_t)m >= A.min_pts || (int64_t)m + (int64_t)A.cv.ub[gc] < A.min_pts) continue;
    const uint32_t* qs = A.qstart + (size_t)t * (A.NS + 1);
    const uint32_t a0 = qs[q << shq], a1 = qs[(q + 1) << shq];
    if (a0 == a1) continue;
    uint32_t cg[D];
    const uint64_t kg = A.cv.cell_key[gc];
#pragma unroll
    for (int k = 0; k < D; ++k) cg[k] = k < d ? cell_coord(kg, g, k) : 0u;
    int64_t qlo[D], qhi[D];
    qb_box<D>(g, cg, q, A.LQ, qlo, qhi);
    int64_t L = m;
    const uint64_t e1 = A.cv.nbr_off[gc + 1];
    for (uint64_t e = A.cv.nbr_off[gc]; e < e1 && L < A.min_pts; ++e) {
      const uint32_t h = A.cv.nbr[e];
      const uint32_t hm = A.cv.cell_start[h + 1] - A.cv.cell_start[h];
      uint32_t ch[D];
      const uint64_t kh = A.cv.cell_key[h];
#pragma unroll
      for (int k = 0; k < D; ++k) ch[k] = k < d ? cell_coord(kh, g, k) : 0u;
      int64_t blo[D], bhi[D];
      qb_box<D>(g, ch, 0, 0, blo, bhi);
      const int cls = qb_classify<D>(g, qlo, qhi, blo, bhi);
      if (cls > 0) { L += hm; continue; }
      if (cls < 0) continue;
      const uint32_t th = A.tidx[h];
      if (th == QB_NONE) continue;
      const uint32_t* hs = A.qstart + (size_t)th * (A.NS + 1);
      // descend level by level; F[cur] holds the partial nodes of level l-1
      int cur = 0;
      uint32_t nf = 1;
      if (lane == 0) F[0][0] = 0;
      __syncwarp();
      for (int l = 1; l <= A.B && nf && L < A.min_pts; ++l) {
        const int sh = (A.B - l) * d;
        const uint32_t items = nf << d;
        uint32_t nn = 0;
        for (uint32_t i0 = 0; i0 < items; i0 += 32) {
          const uint32_t i = i0 + lane;
          uint32_t add = 0, child = 0;
          bool part = false;
          if (i < items) {
            child = ((uint32_t)F[cur][i >> d] << d) | (i & ((1u << d) - 1u));
            const uint32_t c0 = hs[child << sh], c1 = hs[(child + 1) << sh];
            if (c1 > c0) {
              qb_box<D>(g, ch, child, l, blo, bhi);
              const int k2 = qb_classify<D>(g, qlo, qhi, blo, bhi);
              if (k2 > 0) add = c1 - c0;
              else if (k2 == 0 && l < A.B) part = true;
            }
          }
          L += __reduce_add_sync(DB_FULL, add);
          const uint32_t pb = __ballot_sync(DB_FULL, part);
          if (part) F[cur ^ 1][nn + __popc(pb & lanemask_lt())] = (uint16_t)child;
          nn += __popc(pb);
          if (L >= A.min_pts) break;
        }
        __syncwarp();
        cur ^= 1;
        nf = nn;
      }
    }
    if (L >= A.min_pts) {
      for (uint32_t j = s0 + a0 + lane; j < s0 + a1; j += 32) A.core_s[j] = 1;
      if (lane == 0) dec += a1 - a0;
    }
  }
  block_add_u64(dec, A.decided);
}

void mark_core_bounds(Ctx& c, const Geo& g, const CellsView& cv, int32_t* Ps, uint32_t* idx, int64_t n,
                      int64_t min_pts, uint8_t* core_s, unsigned long long* decided) {
  const uint32_t nc = cv.ncells;
  const int B = std::max(1, QB_BITS / g.d);
  const int NS = 1 << (B * g.d);
  const int LQ = std::max(1, std::min(B, 6 / g.d));
  uint32_t* f = c.alloc<uint32_t>(nc);
  uint32_t* pos = c.alloc<uint32_t>((size_t)nc + 1);
  uint32_t* tidx = c.alloc<uint32_t>(nc);
  const uint64_t cap = std::min<uint64_t>(nc, (uint64_t)n / QB_MIN + 1);
  uint32_t* tlist = c.alloc<uint32_t>(cap);
  uint32_t* qstart = c.alloc<uint32_t>(cap * (NS + 1));
  qb_flags_kernel<<<grid_for(nc, 256, 1 << 30), 256, 0, c.st>>>(cv.cell_start, nc, f);
  c.launched();
  exclusive_scan_u32_u32(c, f, pos, nc);
  qb_index_kernel<<<grid_for(nc, 256, 1 << 30), 256, 0, c.st>>>(f, pos, nc, tidx, tlist);
  c.launched();
  int32_t* Ps2 = c.alloc<int32_t>((size_t)n * g.D);
  uint32_t* idx2 = c.alloc<uint32_t>(n);
  QBArgs A{};
  A.g = g;
  A.cv = cv;
  A.tidx = tidx;
  A.tlist = tlist;
  A.qstart = qstart;
  A.ntree = pos + nc;
  A.B = B;
  A.LQ = LQ;
  A.NS = NS;
  A.min_pts = min_pts;
  A.core_s = core_s;
  A.decided = decided;
  auto byD = [&](auto fn) {
    if (g.D == 2) fn(std::integral_constant<int, 2>());
    else if (g.D == 4) fn(std::integral_constant<int, 4>());
    else fn(std::integral_constant<int, 8>());
  };
  byD([&](auto Dc) {
    constexpr int D = decltype(Dc)::value;
    qt_sort_cells_kernel<D><<<std::min<uint32_t>(nc, (uint32_t)c.sms * 8), 1024, 0, c.st>>>(
        Ps, idx, cv.cell_start, cv.cell_key, nc, g, B, Ps2, idx2, QB_MIN, tidx, qstart, c.inv);
    c.launched();
    qb_bound_kernel<D><<<c.sms * 16, 256, 0, c.st>>>(A);
    c.launched();
  });
}

}  // namespace db
