// cluster.cu — ClusterCore and canonical labels (a9).
//
// Alg 3: for core cells g and core neighbours h with
// g > h ("the cell with higher ID [is] responsible") and
// Find(g) != Find(h), test Connected(g, h) — is the bichromatic
// closest pair of their core points within eps — and Link on
// success; a lock-free union-find keeps the components on the fly.
// BCP: points further than eps from the other cell are filtered out first
// (P:L640-641), the search stops at the first pair within eps,
// and the work is done in fixed-size blocks of points: here a
// warp holds 32 points of g in registers and streams 32-point blocks of h,
// exiting on a warp vote.
// Bucketing ("process each batch in parallel before moving to the
// next batch") becomes gap-ordered waves: pairs whose lattice offset has L1
// norm 1 (face-adjacent) first, then 2, then the rest; each wave re-checks
// Find before any BCP, so later waves are mostly pruned.
// Labels: the paper stores uf.Find(g); its value depends on the
// schedule, so the cluster id is canonicalised to the minimum input index of
// the cluster's core points (reading 8).
#include "internal.h"

namespace db {

constexpr int NWAVES = 3;
constexpr uint32_t SMALL_PAIR = 64;  // |A|*|B| at or below: one thread per pair

__device__ __forceinline__ int wave_of(uint64_t kg, uint64_t kh, const Geo& g) {
  uint32_t l1 = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (k < g.d) {
      uint32_t a = cell_coord(kg, g, k), b = cell_coord(kh, g, k);
      l1 += a > b ? a - b : b - a;
    }
  return l1 <= 1 ? 0 : (l1 == 2 ? 1 : 2);
}

// distance from p to the integer box [lo, hi] within eps?
template <int D>
__device__ __forceinline__ bool near_range(const int32_t* p, const int32_t* lo, const int32_t* hi,
                                           int d, uint32_t clampc, uint64_t eps2, uint32_t slack = 0) {
  uint64_t acc = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < d) {
      int64_t x = p[k];
      int64_t t = x < lo[k] ? (int64_t)lo[k] - x : (x > hi[k] ? x - (int64_t)hi[k] : 0);
      t = t > (int64_t)slack ? t - (int64_t)slack : 0;
      uint64_t u = (uint64_t)t;
      if (u > clampc) u = clampc;
      acc += u * u;
    }
  }
  return acc <= eps2;
}

// Warp-cooperative BCP of one pair (warp-uniform arguments and result).
// Lanes hold up to 32 core points of g (filtered against h's box);
// 32-point blocks of h's core points are loaded one point per lane, filtered
// against the bounding box of the current g block, and the survivors are
// broadcast by shuffle and tested against every lane's point; the first pair
// within eps ends the search. Between g blocks, a Find check
// stops early when another warp has connected the pair meanwhile.
template <int D, bool WIDE, bool APX>
__device__ bool warp_bcp(uint2 p, const CellsView& cv, const Geo& g, const int32_t* __restrict__ Ps,
                         const uint32_t* __restrict__ core_cnt, uint32_t* parent) {
  const int lane = threadIdx.x & 31;
  const uint32_t sa = cv.cell_start[p.x], ea = sa + core_cnt[p.x];
  const uint32_t sb = cv.cell_start[p.y], eb = sb + core_cnt[p.y];
  int64_t boxh[D];
  cell_box_lo<D>(cv.cell_key[p.y], g, boxh);
  for (uint32_t a0 = sa; a0 < ea; a0 += 32) {
    const uint32_t u = a0 + lane;
    int32_t a[D];
    bool keep = false;
    if (u < ea) {
      PtLoad<D>::load(Ps, u, a);
      keep = near_box<D>(a, boxh, g, APX ? 2 * (g.at - 1) : 0);  // (approximate: both sub-cell boxes)
    }
    if (!__any_sync(DB_FULL, keep)) continue;
    int32_t qa[D];
    if (APX) connect_prep<D>(a, g, qa);
    // bounding box of the kept block
    int32_t lo[D], hi[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      int32_t l = keep ? a[k] : INT32_MAX, h = keep ? a[k] : INT32_MIN;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        l = min(l, __shfl_xor_sync(DB_FULL, l, o));
        h = max(h, __shfl_xor_sync(DB_FULL, h, o));
      }
      lo[k] = l; hi[k] = h;
    }
    for (uint32_t b0 = sb; b0 < eb; b0 += 32) {
      const uint32_t v = b0 + lane;
      int32_t b[D];
      bool kb = false;
      if (v < eb) {
        PtLoad<D>::load(Ps, v, b);
        // (approximate: both sub-cell boxes reach up to t-1 past their points)
        kb = near_range<D>(b, lo, hi, g.d, g.clampc, g.eps2, APX ? 2 * (g.at - 1) : 0);
        if (APX) connect_prep<D>(b, g, b);
      }
      uint32_t mb = __ballot_sync(DB_FULL, kb);
      bool mine = false;
      while (mb) {
        const int src = __ffs(mb) - 1;
        mb &= mb - 1;
        int32_t q[D];
#pragma unroll
        for (int k = 0; k < D; ++k) q[k] = __shfl_sync(DB_FULL, b[k], src);
        if (keep) DB_WORK(1);
        mine |= keep && (APX ? connect_q<D, WIDE>(qa, q, g) : within<D, WIDE>(a, q, g.clampc, g.eps2));
      }
      if (__any_sync(DB_FULL, mine)) return true;
    }
    bool dn = false;
    if (lane == 0) dn = uf_same(parent, p.x, p.y);
    if (__shfl_sync(DB_FULL, dn, 0)) return false;
  }
  return false;
}

// Tree variant (row f2: "for each core point p in g, issue a
// RangeCount query to h and connect if non-zero"): h's points are all core
// and ordered under a range-count tree (qtree.cu). For each 32-point block of
// g's core points (lanes), one warp-uniform traversal of h's tree: a node is
// entered if its box is within eps of some lane's point; a node whose box
// lies within eps of some lane's point in full proves a pair within eps (the
// node holds >= 1 point, all core) and ends the search; leaves are tested 32
// x 32 by shuffles.
template <int D, bool WIDE>
__device__ bool warp_bcp_tree(uint32_t ga, uint32_t hb, const CellsView& cv, const Geo& g,
                              const int32_t* __restrict__ Ps, const uint32_t* __restrict__ core_cnt,
                              const QTrees& qt) {
  const int lane = threadIdx.x & 31;
  const uint32_t sa = cv.cell_start[ga], ea = sa + core_cnt[ga];
  const uint32_t sb = cv.cell_start[hb], eb = cv.cell_start[hb + 1];
  uint32_t L = (eb - sb + 31) / 32, P2 = 1;
  while (P2 < L) P2 <<= 1;
  const uint64_t base = qt.node_off[hb];
  int64_t boxh[D];
  cell_box_lo<D>(cv.cell_key[hb], g, boxh);
  for (uint32_t a0 = sa; a0 < ea; a0 += 32) {
    const uint32_t u = a0 + lane;
    int32_t a[D];
    bool keep = false;
    if (u < ea) {
      PtLoad<D>::load(Ps, u, a);
      keep = near_box<D>(a, boxh, g);
    }
    if (!__any_sync(DB_FULL, keep)) continue;
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
      const uint32_t node = stack[--sp];
      if (node >= P2 - 1) {
        const uint32_t v = sb + (node - (P2 - 1)) * 32 + lane;
        int32_t b[D];
        const bool vb = v < eb;
        if (vb) PtLoad<D>::load(Ps, v, b);
        uint32_t mb = __ballot_sync(DB_FULL, vb);
        bool mine = false;
        while (mb) {
          const int src = __ffs(mb) - 1;
          mb &= mb - 1;
          int32_t q[D];
#pragma unroll
          for (int k = 0; k < D; ++k) q[k] = __shfl_sync(DB_FULL, b[k], src);
          if (keep) DB_WORK(1);
          mine |= keep && within<D, WIDE>(a, q, g.clampc, g.eps2);
        }
        if (__any_sync(DB_FULL, mine)) return true;
        continue;
      }
      for (uint32_t ch = 2 * node + 2; ch >= 2 * node + 1; --ch) {
        if (qt.cnt[base + ch] == 0) continue;
        const int32_t* bx = qt.box + (base + ch) * 2 * D;
        uint64_t mn = 0, mx = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if (k < g.d) {
            const int64_t x = a[k], lo = bx[k], hi = bx[D + k];
            uint64_t p = (uint64_t)(x < lo ? lo - x : (x > hi ? x - hi : 0));
            uint64_t f = (uint64_t)max(x - lo, hi - x);
            if (p > g.clampc) p = g.clampc;
            if (f > g.clampc) f = g.clampc;
            mn += p * p;
            mx += f * f;
          }
        }
        if (__any_sync(DB_FULL, keep && mx <= g.eps2)) return true;  // a pair within eps exists
        if (__any_sync(DB_FULL, keep && mn <= g.eps2)) stack[sp++] = ch;
      }
    }
  }
  return false;
}

// Warp per pair over list[0 .. min(*count, cap)) (the sparse path's queue).
// MODE 0: exact; 1: exact with range-count trees (row f2); 2: approximate
// connectivity (row f4). Separate instantiations keep the exact kernel lean.
template <int D, bool WIDE, int MODE>
__global__ void __launch_bounds__(256, 2) bcp_large_kernel(const uint2* __restrict__ list,
                                                        const uint32_t* __restrict__ count,
                                                        CellsView cv, Geo g,
                                                        const int32_t* __restrict__ Ps,
                                                        const uint32_t* __restrict__ core_cnt,
                                                        uint32_t* parent, uint32_t cap, QTrees qt) {
  const int lane = threadIdx.x & 31;
  const uint32_t m = min(*count, cap);
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < m; i += nwarps) {
    const uint2 p = list[i];
    bool done = false;
    if (lane == 0) done = uf_same(parent, p.x, p.y);
    if (__shfl_sync(DB_FULL, done, 0)) continue;
    // a tree on an all-core side (f2): search it; else the block BCP
    bool hit;
    bool ty = false, tx = false;
    if (MODE == 1) {
      ty = qt.node_off[p.y + 1] > qt.node_off[p.y] &&
           core_cnt[p.y] == cv.cell_start[p.y + 1] - cv.cell_start[p.y];
      tx = qt.node_off[p.x + 1] > qt.node_off[p.x] &&
           core_cnt[p.x] == cv.cell_start[p.x + 1] - cv.cell_start[p.x];
    }
    if (MODE == 1 && ty) hit = warp_bcp_tree<D, WIDE>(p.x, p.y, cv, g, Ps, core_cnt, qt);
    else if (MODE == 1 && tx) hit = warp_bcp_tree<D, WIDE>(p.y, p.x, cv, g, Ps, core_cnt, qt);
    else hit = warp_bcp<D, WIDE, MODE == 2>(p, cv, g, Ps, core_cnt, parent);
    if (hit && lane == 0) uf_link(parent, p.x, p.y);
    __syncwarp();
  }
}

// One wave of ClusterCore straight from the neighbour CSR (no pair list):
// a group of G lanes per core cell g, lanes over its row; an entry h is a
// candidate of wave w if h < g ("g > h"), h holds core points and
// the pair's lattice L1 distance falls in the wave. Find filter, small BCPs in
// the lane and the queue of large ones as in wave_kernel. Counts candidate
// pairs in *npairs (every wave once). G < 32 serves short rows (the face
// segment of class-sorted rows holds at most 2d cells): each group walks its
// own cells and the warp runs until all of its groups are done.
template <int D, bool WIDE, bool APX, int G>
__global__ void __launch_bounds__(256, 4) wave_csr_kernel(int wave, int nwaves, bool flat, CellsView cv, Geo g,
                                                       const int32_t* __restrict__ Ps,
                                                       const uint32_t* __restrict__ core_cnt, uint32_t* parent,
                                                       uint2* __restrict__ large, uint32_t* __restrict__ nlarge,
                                                       unsigned long long* tested, unsigned long long* npairs) {
  static_assert(G == 8 || G == 16 || G == 32, "group size");
  const int lane = threadIdx.x & 31, gl = lane & (G - 1);
  constexpr uint32_t NG = 32 / G;
  const uint32_t gstride = ((gridDim.x * blockDim.x) >> 5) * NG;
  const bool by_class = cv.ccls && nwaves == NWAVES;  // class-sorted rows: the wave's segment only
  uint32_t mine = 0, cand = 0;
  uint32_t gc = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * NG + lane / G;
  uint32_t kg = 0, rg = 0;
  uint64_t key_g = 0, t0 = 0, r1 = 0;
  // waves after the first (class-sorted rows; the host flattens the forest
  // before each): a pair whose h has the ancestor rg of g as its parent is
  // connected with one load (a cached parent is stale at worst, and then
  // still an ancestor: components only merge)
  const bool hop = by_class && wave > 0 && flat;
  // move the group to its next core cell with a non-empty segment
  auto seek = [&]() {
    for (; gc < cv.ncells; gc += gstride) {
      kg = core_cnt[gc];
      if (kg == 0) continue;
      uint64_t r0 = cv.nbr_off[gc];
      r1 = cv.nbr_off[gc + 1];
      if (by_class) {
        const uint32_t c1 = cv.ccls[gc], c2 = cv.ccls[cv.ncells + gc];
        if (wave == 0) r1 = r0 + c1;
        else if (wave == 1) { r0 += c1; r1 = r0 + c2; }
        else r0 += c1 + c2;
      }
      if (r0 < r1) {
        t0 = r0;
        if (!by_class && nwaves > 1) key_g = cv.cell_key[gc];
        if (hop) rg = uf_root_cached(parent, gc);
        return;
      }
    }
  };
  seek();
  while (__any_sync(DB_FULL, gc < cv.ncells)) {
    const bool act = gc < cv.ncells;
    const uint64_t t = t0 + gl;
    uint2 p = make_uint2(gc, 0);
    bool is = false, need = false, small = false;
    if (act && t < r1) {
      const uint32_t h = cv.nbr[t];
      p.y = h;
      if (h < gc && hop && __ldca(parent + h) == rg) {
        is = true;  // (h is core: a cell without core points is never linked)
      } else if (h < gc) {
        const uint32_t kh = core_cnt[h];
        is = kh > 0 && (by_class || nwaves == 1 || wave_of(key_g, cv.cell_key[h], g) == wave);
        if (is) {
          need = !uf_same(parent, gc, h);
          if (APX && need && apx_cells_within(cv.cell_key[gc], cv.cell_key[h], g)) {
            uf_link(parent, gc, h);  // (rho-approximate: no point test needed)
            need = false;
          }
          small = need && (uint64_t)kg * kh <= SMALL_PAIR;
        }
      }
    }
    cand += is;
    mine += need;
    const uint32_t lm = __ballot_sync(DB_FULL, need && !small);
    if (lm) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(nlarge, (uint32_t)__popc(lm));
      base = __shfl_sync(DB_FULL, base, 0);
      if (need && !small) large[base + __popc(lm & lanemask_lt())] = p;
    }
    if (small) {
      const uint32_t sa = cv.cell_start[p.x], ea = sa + kg;
      const uint32_t sb = cv.cell_start[p.y], eb = sb + core_cnt[p.y];
      bool hit = false;
      int32_t a[D], q[D];
      for (uint32_t u = sa; u < ea && !hit; ++u) {
        PtLoad<D>::load(Ps, u, a);
        if (APX) connect_prep<D>(a, g, a);
        for (uint32_t v = sb; v < eb; ++v) {
          PtLoad<D>::load(Ps, v, q);
          if (APX) connect_prep<D>(q, g, q);
          DB_WORK(1);
          if (APX ? connect_q<D, WIDE>(a, q, g) : within<D, WIDE>(a, q, g.clampc, g.eps2)) { hit = true; break; }
        }
      }
      if (hit) uf_link(parent, p.x, p.y);
    }
    if (act) {
      t0 += G;
      if (t0 >= r1) {
        gc += gstride;
        seek();
      }
    }
  }
  block_add_u64(mine, tested);
  block_add_u64(cand, npairs);
}

__global__ void uf_init_kernel(uint32_t* parent, uint32_t n) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) parent[i] = i;
}

void uf_init(Ctx& c, uint32_t* parent, uint32_t n) {
  uf_init_kernel<<<grid_for(n, 256, 1 << 30), 256, 0, c.st>>>(parent, n);
  c.launched();
}

// only the listed cells (the sparse path's union-find touches core cells only)
__global__ void uf_init_list_kernel(uint32_t* parent, const uint32_t* __restrict__ list, uint32_t m) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) parent[list[t]] = list[t];
}

void uf_init_list(Ctx& c, uint32_t* parent, const uint32_t* list, uint32_t m) {
  if (m == 0) return;
  uf_init_list_kernel<<<grid_for(m, 256, 1 << 30), 256, 0, c.st>>>(parent, list, m);
  c.launched();
}

// parent[x] = Find(x) for the listed cells (all when list is null), between
// passes, so that the next pass's parent comparison (uf_same_hop) settles
// most pairs in one hop (a concurrent Link only moves a root below another
// root, so the stored value stays an ancestor).
__global__ void uf_flatten_kernel(uint32_t* parent, const uint32_t* __restrict__ list, uint32_t m) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
    const uint32_t x = list ? list[t] : t;
    const uint32_t r = uf_find(parent, x);
    if (r != x) parent[x] = r;
  }
}

void uf_flatten(Ctx& c, uint32_t* parent, const uint32_t* list, uint32_t m) {
  if (m == 0) return;
  uf_flatten_kernel<<<grid_for(m, 256, c.sms * 8), 256, 0, c.st>>>(parent, list, m);
  c.launched();
}

void bcp_large(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps, const uint32_t* core_cnt,
               uint32_t* parent, const uint2* list, const uint32_t* count, uint32_t cap, bool wide,
               const QTrees* qt) {
  const QTrees none;
  const QTrees& q = qt ? *qt : none;
  dispatch(g.D, wide, [&]<int D, bool W>() {
    if (g.at)
      bcp_large_kernel<D, W, 2><<<c.sms * 8, 256, 0, c.st>>>(list, count, cv, g, Ps, core_cnt, parent, cap, q);
    else if (q.nodes)
      bcp_large_kernel<D, W, 1><<<c.sms * 8, 256, 0, c.st>>>(list, count, cv, g, Ps, core_cnt, parent, cap, q);
    else
      bcp_large_kernel<D, W, 0><<<c.sms * 8, 256, 0, c.st>>>(list, count, cv, g, Ps, core_cnt, parent, cap, q);
  });
  c.launched();
}

void cluster_core(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps, const uint32_t* core_cnt,
                  bool wide, bool waves, uint64_t nbr_total, uint32_t* parent, unsigned long long* tested,
                  unsigned long long* npairs_out, const QTrees* qt) {
  const uint32_t nc = cv.ncells;
  const int nw = waves ? NWAVES : 1;
  uf_init(c, parent, nc);
  if (nbr_total == 0) return;
  // large pairs of a wave: at most one per CSR entry
  uint2* large = c.alloc<uint2>(nbr_total);
  uint32_t* nlarge = c.alloc<uint32_t>(NWAVES);
  c.zero(nlarge, sizeof(uint32_t) * NWAVES);
  for (int w = 0; w < nw; ++w) {
    // the face segment of class-sorted rows is short (<= 2d cells): groups of 8
    const bool narrow = cv.ccls && nw == NWAVES && w == 0;
    // long rows (the crowded high-d lattices): flatten the forest before the
    // later waves, whose pairs then mostly settle with one load
    const bool flat = cv.ccls && nw == NWAVES && w > 0 && nbr_total >= 256ull * nc;
    if (flat) uf_flatten(c, parent, nullptr, nc);
    const unsigned wgrid = grid_for((int64_t)nc * (narrow ? 8 : 32), 256, c.sms * 16);
    dispatch(g.D, wide, [&]<int D, bool W>() {
      if (g.at) {
        if (narrow)
          wave_csr_kernel<D, W, true, 8><<<wgrid, 256, 0, c.st>>>(w, nw, flat, cv, g, Ps, core_cnt, parent, large,
                                                                  nlarge + w, tested, npairs_out);
        else
          wave_csr_kernel<D, W, true, 32><<<wgrid, 256, 0, c.st>>>(w, nw, flat, cv, g, Ps, core_cnt, parent, large,
                                                                   nlarge + w, tested, npairs_out);
      } else {
        if (narrow)
          wave_csr_kernel<D, W, false, 8><<<wgrid, 256, 0, c.st>>>(w, nw, flat, cv, g, Ps, core_cnt, parent, large,
                                                                   nlarge + w, tested, npairs_out);
        else
          wave_csr_kernel<D, W, false, 32><<<wgrid, 256, 0, c.st>>>(w, nw, flat, cv, g, Ps, core_cnt, parent, large,
                                                                    nlarge + w, tested, npairs_out);
      }
    });
    c.launched();
    bcp_large(c, g, cv, Ps, core_cnt, parent, large, nlarge + w, (uint32_t)nbr_total, wide, qt);
  }
}

// ---------------------------------------------------------------- a9: labels
// Cells are t = 0..nc-1, or list[t] when a list of the cells with core
// points is given (sparse lattices: 733K of 8.9M cells on c5).
__device__ __forceinline__ uint32_t cell_at(const uint32_t* __restrict__ list, uint32_t t) {
  return list ? list[t] : t;
}

__global__ void label_roots_kernel(uint32_t nc, const uint32_t* __restrict__ list,
                                   const uint32_t* __restrict__ core_cnt,
                                   const uint32_t* __restrict__ cell_start,
                                   const uint32_t* __restrict__ idx, int min_mode,
                                   const uint32_t* __restrict__ cellmin, uint32_t* parent,
                                   uint32_t* comp_min, uint32_t* counters) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t g = t < nc ? cell_at(list, t) : 0;
  bool root = false;
  const bool has = t < nc && core_cnt[g] > 0;
  const uint32_t hm = __ballot_sync(DB_FULL, has);
  if (has) {
    const uint32_t r = uf_find(parent, g);
    const uint32_t s = cell_start[g], k = core_cnt[g];
    uint32_t mn;
    if (min_mode == LABEL_MIN_FIRST) {
      // stable sort + stable core-first partition: the first point of a cell
      // has the smallest input index among its core points
      mn = idx[s];
    } else if (min_mode == LABEL_MIN_ARRAY && k == cell_start[g + 1] - s) {
      mn = cellmin[g];  // all core: the cell's minimum
    } else {
      // mixed cell (fewer than minPts points), or any cell of the lattice
      // counting sort (sparse cells): minimum over its core points
      mn = 0xffffffffu;
      for (uint32_t u = s; u < s + k; ++u) mn = min(mn, idx[u]);
    }
    // lanes of one component share one atomic (a component over millions of
    // cells would otherwise serialise millions of same-address atomics)
    const uint32_t peers = __match_any_sync(hm, r);
    mn = __reduce_min_sync(peers, mn);
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicMin(comp_min + r, mn);
    root = r == g;
  }
  const uint32_t b = __syncthreads_count(root);  // one atomic per block, not per warp
  if (threadIdx.x == 0 && b) atomicAdd(counters, b);
}

__global__ void cell_label_kernel(uint32_t nc, const uint32_t* __restrict__ list,
                                  const uint32_t* __restrict__ core_cnt, uint32_t* parent,
                                  const uint32_t* __restrict__ comp_min, uint32_t* __restrict__ cell_label) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nc) return;
  const uint32_t g = cell_at(list, t);
  cell_label[g] = core_cnt[g] > 0 ? comp_min[uf_find(parent, g)] : 0xffffffffu;
}

// Scatter the labels to input order (a9). Core points are the first
// core_cnt[g] points of their cell (a7).
//  * per position (few large cells): thread per sorted position, -1 for
//    non-core points, so cluster[] needs no clearing; 10^7 independent
//    threads hide the latency of the idx load before each scattered store;
//  * per cell (many small cells, or the list of cells holding core points):
//    cluster[] was set to -1 first and only core points are written (8% of
//    the points on c5).
__global__ void __launch_bounds__(256) write_positions_kernel(uint32_t n, const uint32_t* __restrict__ idx,
                                                              const uint32_t* __restrict__ cell_of,
                                                              const uint32_t* __restrict__ cell_start,
                                                              const uint32_t* __restrict__ core_cnt,
                                                              const uint32_t* __restrict__ cell_label,
                                                              int32_t* __restrict__ cluster_out,
                                                              uint32_t* counters) {
  // grid-stride over a bounded grid: one atomic per block (same-address
  // atomics from n/256 blocks serialise: ~25 us at n = 10M)
  unsigned long long nc = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t g = cell_of[j];
    const bool is_core = j - cell_start[g] < core_cnt[g];
    cluster_out[idx[j]] = is_core ? (int32_t)cell_label[g] : -1;
    nc += is_core;
  }
  __shared__ unsigned long long s_c;
  if (threadIdx.x == 0) s_c = 0;
  __syncthreads();
  nc = __reduce_add_sync(DB_FULL, (uint32_t)nc);
  if ((threadIdx.x & 31) == 0 && nc) atomicAdd(&s_c, nc);
  __syncthreads();
  if (threadIdx.x == 0 && s_c) atomicAdd(counters + 1, (uint32_t)s_c);
}

// By input index (the grouping kept the inverse permutation inv): thread i
// reads its sorted position and cell, and writes cluster[i] and core[i] —
// coalesced stores instead of a scatter through idx (write_positions), the
// random reads (cell_of at the sorted position) hitting L2.
__global__ void __launch_bounds__(256) write_input_kernel(uint32_t n, const uint32_t* __restrict__ inv,
                                                          const uint32_t* __restrict__ cell_of,
                                                          const uint32_t* __restrict__ cell_start,
                                                          const uint32_t* __restrict__ core_cnt,
                                                          const uint32_t* __restrict__ cell_label,
                                                          int32_t* __restrict__ cluster_out,
                                                          uint8_t* __restrict__ core_out, uint32_t* counters) {
  unsigned long long nc = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t j = inv[i];
    const uint32_t g = cell_of[j];
    const bool is_core = j - cell_start[g] < core_cnt[g];
    cluster_out[i] = is_core ? (int32_t)cell_label[g] : -1;
    core_out[i] = is_core;
    nc += is_core;
  }
  __shared__ unsigned long long s_c;
  if (threadIdx.x == 0) s_c = 0;
  __syncthreads();
  nc = __reduce_add_sync(DB_FULL, (uint32_t)nc);
  if ((threadIdx.x & 31) == 0 && nc) atomicAdd(&s_c, nc);
  __syncthreads();
  if (threadIdx.x == 0 && s_c) atomicAdd(counters + 1, (uint32_t)s_c);
}

// (also sets cell_label: the cell's component minimum, ~0 without core points)
__global__ void __launch_bounds__(256) write_points_kernel(uint32_t nc, const uint32_t* __restrict__ list,
                                                           const uint32_t* __restrict__ idx,
                                                           const uint32_t* __restrict__ cell_start,
                                                           const uint32_t* __restrict__ core_cnt,
                                                           uint32_t* parent, const uint32_t* __restrict__ comp_min,
                                                           uint32_t* __restrict__ cell_label,
                                                           int32_t* __restrict__ cluster_out, uint32_t* counters) {
  unsigned long long ncore = 0;
  const uint32_t lane = threadIdx.x & 31u;
  // (warp-uniform trip count: the cells with more than 32 core points are
  // written by the whole warp)
  for (uint32_t t0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; t0 < nc; t0 += gridDim.x * blockDim.x) {
    const uint32_t t = t0 + lane;
    uint32_t k = 0, s = 0;
    int32_t lab = -1;
    if (t < nc) {
      const uint32_t g = cell_at(list, t);
      k = core_cnt[g];
      if (!k) {
        cell_label[g] = 0xffffffffu;
      } else {
        lab = (int32_t)comp_min[uf_find(parent, g)];
        cell_label[g] = (uint32_t)lab;
        s = cell_start[g];
        if (k <= 32)
          for (uint32_t u = s; u < s + k; ++u) cluster_out[idx[u]] = lab;
        ncore += k;
      }
    }
    for (uint32_t bm = __ballot_sync(DB_FULL, k > 32); bm; bm &= bm - 1) {
      const int src = __ffs(bm) - 1;
      const uint32_t bs = __shfl_sync(DB_FULL, s, src), bk = __shfl_sync(DB_FULL, k, src);
      const int32_t bl = __shfl_sync(DB_FULL, lab, src);
      for (uint32_t u = bs + lane; u < bs + bk; u += 32) cluster_out[idx[u]] = bl;
    }
  }
  __shared__ unsigned long long s_part[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) ncore += __shfl_xor_sync(DB_FULL, ncore, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = ncore;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_part[w];
    if (t) atomicAdd(counters + 1, (uint32_t)t);  // core points (< 2^31)
  }
}

// core[i] = cluster[i] >= 0, in input order (coalesced, 4 points per thread).
__global__ void core_from_cluster_kernel(uint32_t n, const int32_t* __restrict__ cluster,
                                         uint8_t* __restrict__ core) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t i = 4 * q;
  if (i + 3 < n && (reinterpret_cast<uintptr_t>(core) & 3) == 0) {
    const int4 v = reinterpret_cast<const int4*>(cluster)[q];
    const uint32_t w = (uint32_t)(v.x >= 0) | ((uint32_t)(v.y >= 0) << 8) |
                       ((uint32_t)(v.z >= 0) << 16) | ((uint32_t)(v.w >= 0) << 24);
    reinterpret_cast<uint32_t*>(core)[q] = w;
  } else {
    for (uint32_t k = i; k < min(i + 4, n); ++k) core[k] = cluster[k] >= 0;
  }
}

void labels(Ctx& c, const CellsView& cv, const uint32_t* idx, const uint8_t* core_s,
            const uint32_t* core_cnt, int min_mode, const uint32_t* cellmin, const uint32_t* core_list,
            uint32_t ncore, uint32_t* parent, int64_t n, uint32_t* cell_label,
            uint8_t* core_out, int32_t* cluster_out, uint32_t* counters) {
  const uint32_t nc = cv.ncells;
  const uint32_t m = core_list ? ncore : nc;  // cells the kernels visit
  uint32_t* comp_min = c.alloc<uint32_t>(nc);
  DB_CUDA(cudaMemsetAsync(comp_min, 0xff, sizeof(uint32_t) * nc, c.st));
  label_roots_kernel<<<grid_for(m, 256, 1 << 30), 256, 0, c.st>>>(m, core_list, core_cnt, cv.cell_start, idx,
                                                                    min_mode, cellmin, parent, comp_min,
                                                                    counters);
  c.launched();
  if (!core_list && (int64_t)nc * 32 <= n && c.inv) {
    cell_label_kernel<<<grid_for(m, 256, 1 << 30), 256, 0, c.st>>>(m, core_list, core_cnt, parent, comp_min,
                                                                    cell_label);
    c.launched();
    write_input_kernel<<<grid_for(n, 256, c.sms * 16), 256, 0, c.st>>>(
        (uint32_t)n, c.inv, cv.cell_of, cv.cell_start, core_cnt, cell_label, cluster_out, core_out, counters);
    c.launched();
    return;  // (core[] written too)
  }
  if (!core_list && (int64_t)nc * 32 <= n) {
    cell_label_kernel<<<grid_for(m, 256, 1 << 30), 256, 0, c.st>>>(m, core_list, core_cnt, parent, comp_min,
                                                                    cell_label);
    c.launched();
    write_positions_kernel<<<grid_for(n, 256, c.sms * 16), 256, 0, c.st>>>(
        (uint32_t)n, idx, cv.cell_of, cv.cell_start, core_cnt, cell_label, cluster_out, counters);
  } else {
    DB_CUDA(cudaMemsetAsync(cluster_out, 0xff, sizeof(int32_t) * (size_t)n, c.st));
    write_points_kernel<<<grid_for(m, 256, c.sms * 16), 256, 0, c.st>>>(
        m, core_list, idx, cv.cell_start, core_cnt, parent, comp_min, cell_label, cluster_out, counters);
  }
  c.launched();
  core_from_cluster_kernel<<<grid_for((n + 3) / 4, 256, 1 << 30), 256, 0, c.st>>>((uint32_t)n, cluster_out,
                                                                                  core_out);
  c.launched();
}

}  // namespace db
