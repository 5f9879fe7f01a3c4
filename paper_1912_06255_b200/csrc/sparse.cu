// sparse.cu — the cell-centric path for sparse lattices (d <= 3, few points
// per cell, e.g. BASELINE configs[4] "3D uniform fill": 8.9M cells of ~1.1
// points). It computes exactly what the CSR path computes (rows a5-a10 of
// SURVEY §8(a)) but never materialises neighbour lists: with ~26 non-empty
// neighbours of ~1 point per cell, building and re-reading a CSR costs more
// than walking the stencil again.
//
//  * Cell lookup (a4): a rank directory over the lattice padded by R cells:
//    an occupancy bitmap plus a per-32-cell exclusive prefix count (2 bits per
//    lattice cell; L2-resident at these sizes). Cell ids follow key order,
//    which is the lattice's linear order, so id = prefix[w] + popc(bits below).
//    Out-of-range neighbours land in the padding (no range checks).
//  * MarkCore (a6, Alg 2): a thread per point probes every
//    stencil offset without divergence (consecutive lanes probe adjacent
//    directory words), lists the cells found in L1-resident local memory, then
//    counts over those ~26 cells only, nearest first, stopping at minPts; a
//    thread per cell then counts core points (a7) and mixed cells are
//    partitioned core-first.
//  * ClusterCore (a8, Alg 3): per wave (offsets of lattice L1 norm
//    1, 2, >= 3, each with a negative linear offset so h < g, "g > h",
//    P:L847-849), a warp takes 32 cells and, for each core cell among them,
//    lanes probe the wave's offsets, skip pairs with equal Find, run small
//    BCPs inline with early exit and queue large ones for the warp BCP kernel
//    (cluster.cu).
//  * ClusterBorder (a10, Alg 4): a thread per non-core point,
//    the same two phases restricted to cells with core points, label sets of
//    up to SP_MAXL in registers staged per sorted position; larger sets are
//    enumerated without storage in ascending order.
#include <algorithm>
#include <map>

#include "internal.h"

namespace db {

constexpr int SP_MAXL = 4;
constexpr int SP_MAX_OFFS = 1024;
constexpr uint32_t MISS = 0xffffffffu;

struct SpArgs {
  Geo g;
  uint64_t stride[3];
  const uint32_t* bm;
  const uint32_t* pre;
  const long long* coff;     // stencil columns: start offset (padded linear units), nearest first
  const uint32_t* cmask;     // stencil columns: (1 << width) - 1
  int ncols;
  const long long* bcoff;    // back columns (cells before g in linear order)
  const uint32_t* bcmask;
  int nbcols;
  uint32_t ncells;
  const uint32_t* cell_start;
  const uint64_t* cell_key;
  const uint32_t* cell_of;
  int32_t* Ps;
  uint32_t* idx;
  uint8_t* core_s;
  uint32_t* core_cnt;
  int64_t min_pts;
  uint32_t* counters;        // [0] core cells, [1] unused, [2] large pairs, [3] mixed cells
  uint32_t* mixed_list;
  const uint32_t* cell_label;
  uint32_t* parent;
  uint2* large;
  uint32_t large_cap;
  uint32_t* bcnt;            // [n] input order
  uint32_t* tmp_lab;         // [n*SP_MAXL] sorted order
  uint8_t* tmp_n;            // [n] sorted order; 0xff = overflow
  unsigned long long* nborder;
  int64_t n;
};

__device__ __forceinline__ uint32_t rd_lookup(const uint32_t* __restrict__ bm,
                                              const uint32_t* __restrict__ pre, uint64_t lin) {
  const uint32_t w = __ldg(bm + (lin >> 5));
  const uint32_t b = (uint32_t)lin & 31u;
  if (!((w >> b) & 1u)) return MISS;
  return __ldg(pre + (lin >> 5)) + __popc(w & ((1u << b) - 1u));
}

// A stencil column: the lattice cells base + off .. base + off + width - 1,
// consecutive along the last axis (the exact stencil is a union of such
// columns). The cells present in it have consecutive ids (ids
// follow the lattice's linear order), so one 64-bit window of the bitmap
// gives how many there are and one prefix word gives the first id; their
// points are one contiguous range of Ps. Returns the number of cells.
__device__ __forceinline__ uint32_t col_probe(const uint32_t* __restrict__ bm,
                                              const uint32_t* __restrict__ pre, uint64_t start,
                                              uint32_t mask, uint32_t* id0) {
  const uint64_t w0 = start >> 5;
  const uint32_t b0 = (uint32_t)start & 31u;
  const uint32_t lo = __ldg(bm + w0), hi = __ldg(bm + w0 + 1);
  const uint32_t bits = __funnelshift_r(lo, hi, b0) & mask;
  if (!bits) return 0;
  *id0 = __ldg(pre + w0) + __popc(lo & ((1u << b0) - 1u));
  return __popc(bits);
}

template <int DIM>
__device__ __forceinline__ uint64_t cell_lin(uint64_t key, const SpArgs& a) {
  uint64_t lin = 0;
#pragma unroll
  for (int k = 0; k < DIM; ++k) lin += (uint64_t)(cell_coord(key, a.g, k) + a.g.R) * a.stride[k];
  return lin;
}

template <int D>
__device__ __forceinline__ void load_pt(const int32_t* __restrict__ Ps, uint32_t j, int32_t* x) {
  PtLoad<D>::load(Ps, j, x);
}

template <int D>
__device__ __forceinline__ void shfl_pt(const int32_t* src, int from, int32_t* dst) {
#pragma unroll
  for (int k = 0; k < D; ++k) dst[k] = __shfl_sync(DB_FULL, src[k], from);
}

// Flattened candidates of one batch: lane l owns cell (st_l, sz_l); candidate
// tt lives in the lane o with excl_o <= tt < excl_o + sz_o.
struct Batch {
  uint32_t st, excl, total;
};

__device__ __forceinline__ Batch make_batch(uint32_t st, uint32_t sz) {
  const uint32_t incl = warp_inclusive_scan(sz);
  Batch b;
  b.st = st;
  b.excl = incl - sz;
  b.total = __shfl_sync(DB_FULL, incl, 31);
  return b;
}

// owner lane and point index of candidate tt (all lanes call; tt may be >= total)
__device__ __forceinline__ uint32_t batch_point(const Batch& b, uint32_t tt, int* owner) {
  int lo = 0;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t e = __shfl_sync(DB_FULL, b.excl, lo + s);
    if (e <= tt) lo += s;
  }
  *owner = lo;
  const uint32_t ost = __shfl_sync(DB_FULL, b.st, lo);
  const uint32_t oex = __shfl_sync(DB_FULL, b.excl, lo);
  return ost + (tt - oex);
}

// ------------------------------------------------------------- directory
__global__ void rd_set_kernel(const uint64_t* __restrict__ cell_key, uint32_t ncells, SpArgs a,
                              uint32_t* bm) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncells) return;
  const uint64_t key = cell_key[i];
  uint64_t lin = 0;
  for (int k = 0; k < a.g.d; ++k) lin += (uint64_t)(cell_coord(key, a.g, k) + a.g.R) * a.stride[k];
  atomicOr(bm + (lin >> 5), 1u << (lin & 31));
}

// largest cell size (block max, one atomic per block)
__global__ void __launch_bounds__(256) cell_max_kernel(const uint32_t* __restrict__ cell_start,
                                                       uint32_t ncells, uint32_t* mx) {
  uint32_t m = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += gridDim.x * blockDim.x)
    m = max(m, cell_start[i + 1] - cell_start[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(DB_FULL, m, o));
  __shared__ uint32_t sm[8];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, sm[w]);
    atomicMax(mx, m);
  }
}

__global__ void popc_kernel(const uint32_t* __restrict__ bm, uint64_t words, uint32_t* __restrict__ cnt) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < words) cnt[i] = __popc(bm[i]);
}

// ------------------------------------------------------------ MarkCore (a6)
// Thread per sorted point (Alg 2): a dense cell (|g| >= minPts)
// is all core; otherwise count the points within eps over the
// stencil columns, nearest column first, stopping at minPts. The own cell
// lies in the central column and is counted by the same test (same cell =>
// within eps, so the test always passes there; p counts itself).
// Consecutive lanes hold consecutive sorted points (mostly one cell or its
// last-axis neighbours), so their column probes and point loads coalesce.
constexpr int SP_MAX_COLS = 64;

template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_core_kernel(SpArgs a) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  for (int i = threadIdx.x; i < a.ncols; i += blockDim.x) { s_off[i] = a.coff[i]; s_mask[i] = a.cmask[i]; }
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  const uint32_t g = a.cell_of[j];
  const uint32_t m = a.cell_start[g + 1] - a.cell_start[g];
  if ((int64_t)m >= a.min_pts) { a.core_s[j] = 1; return; }  // dense cell
  const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
  int32_t p[D];
  load_pt<D>(a.Ps, j, p);
  int64_t count = 0;
  for (int c = 0; c < a.ncols && count < a.min_pts; ++c) {
    uint32_t id0;
    const uint32_t nc = col_probe(a.bm, a.pre, base + (uint64_t)s_off[c], s_mask[c], &id0);
    if (!nc) continue;
    const uint32_t ue = a.cell_start[id0 + nc];
    for (uint32_t u = a.cell_start[id0]; u < ue; ++u) {
      int32_t q[D];
      load_pt<D>(a.Ps, u, q);
      count += within<D, WIDE>(p, q, a.g.clampc, a.g.eps2);
      if (count >= a.min_pts) break;
    }
  }
  a.core_s[j] = count >= a.min_pts;
}

// Thread per cell: core count (a7); mixed cells are listed for the partition.
__global__ void __launch_bounds__(256) sp_cells_kernel(SpArgs a) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  bool core_cell = false, mixed = false;
  if (g < a.ncells) {
    const uint32_t s = a.cell_start[g], e = a.cell_start[g + 1], m = e - s;
    uint32_t k = 0;
    if ((int64_t)m >= a.min_pts) k = m;
    else
      for (uint32_t u = s; u < e; ++u) k += a.core_s[u];
    a.core_cnt[g] = k;
    core_cell = k > 0;
    mixed = k > 0 && k < m;
  }
  const uint32_t cb = __syncthreads_count(core_cell);
  if (threadIdx.x == 0 && cb) atomicAdd(a.counters + 0, cb);
  const uint32_t mb = __ballot_sync(DB_FULL, mixed);
  if (mb) {
    const int lane = threadIdx.x & 31, leader = __ffs(mb) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(a.counters + 3, (uint32_t)__popc(mb));
    base = __shfl_sync(DB_FULL, base, leader);
    if (mixed) a.mixed_list[base + __popc(mb & lanemask_lt())] = g;
  }
}

// ---------------------------------------------------------- ClusterCore (a8)
// One pass over the "back" stencil columns (cells h before g in the lattice's
// linear order, i.e. h < g: "the cell with higher ID checks").
// A warp takes 32 consecutive cells; its lanes then run over the (core cell,
// back column) items of the chunk. For a core cell h found in a column:
//  * small pairs (|A| |B| <= SP_SMALL core points; ~1x1 on sparse lattices):
//    the BCP test itself is cheaper than the two Finds that could prune it,
//    so it runs directly (early exit at the first pair within eps,
//    P:L642-644) and Links on success;
//  * larger pairs are skipped if Find(g) == Find(h) and queued
//    for the warp BCP kernel (cluster.cu), which re-checks Find first.
constexpr uint32_t SP_SMALL = 64;

template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_pairs_kernel(SpArgs a, unsigned long long* tested) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  const int nb = a.nbcols;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) { s_off[i] = a.bcoff[i]; s_mask[i] = a.bcmask[i]; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t mine = 0;
  for (uint32_t c0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; c0 < a.ncells;
       c0 += nwarps * 32) {
    const uint32_t gl = c0 + lane;
    const uint32_t kl = gl < a.ncells ? a.core_cnt[gl] : 0;
    const uint32_t cm = __ballot_sync(DB_FULL, kl > 0);
    const uint32_t items = (uint32_t)__popc(cm) * (uint32_t)nb;
    for (uint32_t it = lane; it < items; it += 32) {
      const uint32_t ci = it / nb, col = it - ci * nb;
      const uint32_t g = c0 + (uint32_t)(__fns(cm, 0, ci + 1));
      const uint32_t kg = a.core_cnt[g];
      const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
      uint32_t id0;
      const uint32_t nc = col_probe(a.bm, a.pre, base + (uint64_t)s_off[col], s_mask[col], &id0);
      for (uint32_t h = id0; h < id0 + nc; ++h) {
        const uint32_t kh = a.core_cnt[h];
        if (kh == 0) continue;
        if ((uint64_t)kg * kh > SP_SMALL) {
          if (uf_find(a.parent, g) == uf_find(a.parent, h)) continue;
          const uint32_t slot = atomicAdd(a.counters + 2, 1u);
          if (slot < a.large_cap) { a.large[slot] = make_uint2(g, h); continue; }
          // list full: test the pair here (correct, only slower)
        }
        ++mine;
        const uint32_t sg = a.cell_start[g], sh = a.cell_start[h];
        bool hit = false;
        for (uint32_t u = sg; u < sg + kg && !hit; ++u) {
          int32_t p[D];
          load_pt<D>(a.Ps, u, p);
          for (uint32_t v = sh; v < sh + kh; ++v) {
            int32_t q[D];
            load_pt<D>(a.Ps, v, q);
            if (within<D, WIDE>(p, q, a.g.clampc, a.g.eps2)) { hit = true; break; }
          }
        }
        if (hit) uf_link(a.parent, g, h);
      }
    }
  }
  block_add_u64(mine, tested);
}

// --------------------------------------------------------- ClusterBorder (a10)
// Does cell h hold a core point within eps of p? Core points are first in
// their cell (a7), so they are Ps[cell_start[h] .. + core_cnt[h]).
template <int D, bool WIDE>
__device__ __forceinline__ bool sp_core_within(const SpArgs& a, const int32_t* p, uint32_t h, uint32_t kh) {
  const uint32_t sh = a.cell_start[h];
  for (uint32_t v = sh; v < sh + kh; ++v) {
    int32_t q[D];
    load_pt<D>(a.Ps, v, q);
    if (within<D, WIDE>(p, q, a.g.clampc, a.g.eps2)) return true;
  }
  return false;
}

// Smallest label > `after` among clusters with a core point within eps of p
// (storage-free enumeration for points with more than SP_MAXL labels).
template <int DIM, int D, bool WIDE>
__device__ uint32_t sp_next_label(const SpArgs& a, const long long* s_off, const uint32_t* s_mask,
                                  const int32_t* p, uint32_t g, uint64_t base, int64_t after) {
  uint32_t best = MISS;
  for (int c = 0; c < a.ncols; ++c) {
    uint32_t id0;
    const uint32_t nc = col_probe(a.bm, a.pre, base + (uint64_t)s_off[c], s_mask[c], &id0);
    for (uint32_t h = id0; h < id0 + nc; ++h) {
      const uint32_t kh = a.core_cnt[h];
      if (kh == 0) continue;
      const uint32_t lab = a.cell_label[h];
      if ((int64_t)lab <= after || lab >= best) continue;
      if (h == g || sp_core_within<D, WIDE>(a, p, h, kh)) best = lab;
    }
  }
  return best;
}

// Thread per sorted non-core point (Alg 4): walk the stencil
// columns nearest first; for each cell with core points whose label is not
// yet in the set, scan its core points until one is within eps. The own cell
// gives its label with no distance test (same cell => within eps,
// P:L400-403). Up to SP_MAXL labels live in registers (unused = ~0, sorted
// by a 4-input network at the end) and are staged per sorted position for the
// fill pass; larger sets are enumerated without storage in ascending order.
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_border_kernel(SpArgs a) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  for (int i = threadIdx.x; i < a.ncols; i += blockDim.x) { s_off[i] = a.coff[i]; s_mask[i] = a.cmask[i]; }
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  bool bord = false;
  if (j < a.n && !a.core_s[j]) {
    const uint32_t g = a.cell_of[j];
    const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
    int32_t p[D];
    load_pt<D>(a.Ps, j, p);
    uint32_t L0 = MISS, L1 = MISS, L2 = MISS, L3 = MISS;
    int nl = 0;
    bool ovf = false;
    for (int c = 0; c < a.ncols && !ovf; ++c) {
      uint32_t id0;
      const uint32_t nc = col_probe(a.bm, a.pre, base + (uint64_t)s_off[c], s_mask[c], &id0);
      for (uint32_t h = id0; h < id0 + nc; ++h) {
        const uint32_t kh = a.core_cnt[h];
        if (kh == 0) continue;
        const uint32_t lab = a.cell_label[h];
        if (lab == L0 || lab == L1 || lab == L2 || lab == L3) continue;
        if (h != g && !sp_core_within<D, WIDE>(a, p, h, kh)) continue;
        if (nl == 0) L0 = lab;
        else if (nl == 1) L1 = lab;
        else if (nl == 2) L2 = lab;
        else if (nl == 3) L3 = lab;
        else { ovf = true; break; }
        ++nl;
      }
    }
    uint32_t cnt;
    if (!ovf) {
      auto cs = [](uint32_t& x, uint32_t& y) { const uint32_t lo = min(x, y), hi = max(x, y); x = lo; y = hi; };
      cs(L0, L1); cs(L2, L3); cs(L0, L2); cs(L1, L3); cs(L1, L2);
      if (nl) {
        uint32_t* dst = a.tmp_lab + (size_t)j * SP_MAXL;
        dst[0] = L0;
        if (nl > 1) dst[1] = L1;
        if (nl > 2) dst[2] = L2;
        if (nl > 3) dst[3] = L3;
      }
      a.tmp_n[j] = (uint8_t)nl;
      cnt = (uint32_t)nl;
    } else {
      int64_t after = -1;
      cnt = 0;
      while (true) {
        const uint32_t nx = sp_next_label<DIM, D, WIDE>(a, s_off, s_mask, p, g, base, after);
        if (nx == MISS) break;
        ++cnt;
        after = nx;
      }
      a.tmp_n[j] = 0xff;
    }
    a.bcnt[a.idx[j]] = cnt;
    bord = cnt > 0;
  }
  const uint32_t nb = __syncthreads_count(bord);
  if (threadIdx.x == 0 && nb) atomicAdd(a.nborder, (unsigned long long)nb);
}

// Copy the staged label sets into the CSR (thread per sorted point).
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_border_fill_kernel(SpArgs a, const int64_t* __restrict__ border_off,
                                                             int32_t* __restrict__ border_ids) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  for (int i = threadIdx.x; i < a.ncols; i += blockDim.x) { s_off[i] = a.coff[i]; s_mask[i] = a.cmask[i]; }
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n || a.core_s[j]) return;
  const uint8_t nl = a.tmp_n[j];
  if (nl == 0) return;
  const int64_t o = border_off[a.idx[j]];
  if (nl != 0xff) {
    for (int q = 0; q < nl; ++q) border_ids[o + q] = (int32_t)a.tmp_lab[(size_t)j * SP_MAXL + q];
    return;
  }
  const uint32_t g = a.cell_of[j];
  const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
  int32_t p[D];
  load_pt<D>(a.Ps, j, p);
  int64_t after = -1, w = 0;
  while (true) {
    const uint32_t nx = sp_next_label<DIM, D, WIDE>(a, s_off, s_mask, p, g, base, after);
    if (nx == MISS) break;
    border_ids[o + w++] = (int32_t)nx;
    after = nx;
  }
}

// ----------------------------------------------------------------- host
template <typename F>
static void by_dim_sp(int d, bool wide, F&& f) {
  auto w = [&](auto Dm, auto Dp) {
    if (wide) f(Dm, Dp, std::true_type());
    else f(Dm, Dp, std::false_type());
  };
  if (d == 1) w(std::integral_constant<int, 1>(), std::integral_constant<int, 2>());
  else if (d == 2) w(std::integral_constant<int, 2>(), std::integral_constant<int, 2>());
  else w(std::integral_constant<int, 3>(), std::integral_constant<int, 4>());
}

static unsigned __int128 padded_volume(const Geo& g) {
  unsigned __int128 vol = 1;
  for (int k = 0; k < g.d; ++k) vol *= (unsigned __int128)g.maxc[k] + 1 + 2 * (unsigned __int128)g.R;
  return vol;
}

bool sparse_applicable(const Geo& g, int64_t n, uint32_t ncells, bool forced) {
  if (g.d > 3) return false;
  // 2 bits per lattice cell: keep the directory within ~32 bytes per point
  if (padded_volume(g) > (unsigned __int128)128 * n + (1u << 24)) return false;
  if (stencil_offsets(g).size() / g.d + 1 > (size_t)SP_MAX_OFFS) return false;
  if (forced) return true;
  return (uint64_t)n <= (uint64_t)SPARSE_MEAN_PER_CELL * ncells;
}

void sparse_pipeline(Ctx& c, const Geo& g, const CellsView& cv, int32_t* Ps, uint32_t* idx,
                     uint8_t* core_s, uint32_t* core_cnt, int64_t n, int64_t min_pts, bool wide,
                     bool waves, SparseOut* o) {
  (void)waves;
  SpArgs a{};
  a.g = g;
  unsigned __int128 vol = 1;
  for (int k = g.d - 1; k >= 0; --k) {
    a.stride[k] = (uint64_t)vol;
    vol *= (unsigned __int128)g.maxc[k] + 1 + 2 * (unsigned __int128)g.R;
  }
  // stencil offsets in padded linear units, nearest first; back offsets per wave
  std::vector<int8_t> offs = stencil_offsets(g);
  const int noffs = (int)(offs.size() / g.d);
  // Global MarkCore bound (Alg 2's count can never exceed the points of the
  // stencil cells, reading 13): if (stencil cells) x (largest cell) < minPts
  // no point can be core and the caller takes the all-noise exit.
  if ((uint64_t)min_pts > (uint64_t)noffs + 1) {
    uint32_t* mx = c.alloc<uint32_t>(1);
    c.zero(mx, sizeof(uint32_t));
    cell_max_kernel<<<grid_for(cv.ncells, 256, c.sms * 8), 256, 0, c.st>>>(cv.cell_start, cv.ncells, mx);
    c.launched();
    const uint64_t bound = (uint64_t)c.read(mx) * (uint64_t)(noffs + 1);
    if (bound < (uint64_t)min_pts) return;  // counters[0] (core cells) stays 0
  }
  // rank directory
  const uint64_t words = ((uint64_t)vol + 31) / 32 + 1;
  uint32_t* bm = c.alloc<uint32_t>(words);
  uint32_t* wcnt = c.alloc<uint32_t>(words);
  uint32_t* pre = c.alloc<uint32_t>(words + 1);
  c.zero(bm, sizeof(uint32_t) * words);
  a.bm = bm;
  a.pre = pre;
  rd_set_kernel<<<grid_for(cv.ncells, 256, 1 << 30), 256, 0, c.st>>>(cv.cell_key, cv.ncells, a, bm);
  c.launched();
  popc_kernel<<<grid_for((int64_t)words, 256, 1 << 30), 256, 0, c.st>>>(bm, words, wcnt);
  c.launched();
  exclusive_scan_u32_u32(c, wcnt, pre, (int64_t)words);
  // stencil columns: group the offsets (and self) by all but the last axis;
  // each group is |delta_last| <= m, one column of width 2m + 1
  {
    std::map<std::vector<int>, int> colm;
    std::vector<int> zero(g.d > 1 ? g.d - 1 : 0, 0);
    colm[zero] = 0;
    for (int t = 0; t < noffs; ++t) {
      std::vector<int> pfx(offs.begin() + (size_t)t * g.d, offs.begin() + (size_t)t * g.d + g.d - 1);
      const int v = offs[(size_t)t * g.d + g.d - 1];
      int& mm = colm[pfx];
      mm = std::max(mm, v < 0 ? -v : v);
    }
    std::vector<std::pair<unsigned __int128, std::pair<long long, uint32_t>>> cols, bcols;
    for (auto& [pfx, mm] : colm) {
      int first = 0;  // sign of the first non-zero prefix component
      for (int v : pfx)
        if (v) { first = v < 0 ? -1 : 1; break; }
      unsigned __int128 gap = 0;
      long long off = -(long long)mm;
      for (int k = 0; k + 1 < g.d; ++k) {
        const int v = pfx[k] < 0 ? -pfx[k] : pfx[k];
        if (v) { const unsigned __int128 gg = (unsigned __int128)(v - 1) * g.s + 1; gap += gg * gg; }
        off += (long long)pfx[k] * (long long)a.stride[k];
      }
      cols.push_back({gap, {off, (uint32_t)((1ull << (2 * mm + 1)) - 1)}});
      // back columns: every cell precedes g in linear order (prefix < 0), or
      // the cells below g in its own column
      if (first < 0) bcols.push_back({gap, {off, (uint32_t)((1ull << (2 * mm + 1)) - 1)}});
      else if (first == 0 && mm > 0) bcols.push_back({gap, {off, (uint32_t)((1ull << mm) - 1)}});
    }
    std::stable_sort(bcols.begin(), bcols.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    std::stable_sort(cols.begin(), cols.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    if ((int)cols.size() > SP_MAX_COLS) throw Error(-4, "sparse path: too many stencil columns");
    std::vector<long long> co;
    std::vector<uint32_t> cm;
    for (auto& e : cols) { co.push_back(e.second.first); cm.push_back(e.second.second); }
    long long* dco = c.alloc<long long>(co.size());
    uint32_t* dcm = c.alloc<uint32_t>(cm.size());
    DB_CUDA(cudaMemcpyAsync(dco, co.data(), sizeof(long long) * co.size(), cudaMemcpyHostToDevice, c.st));
    DB_CUDA(cudaMemcpyAsync(dcm, cm.data(), sizeof(uint32_t) * cm.size(), cudaMemcpyHostToDevice, c.st));
    a.coff = dco;
    a.cmask = dcm;
    a.ncols = (int)cols.size();
    std::vector<long long> bo;
    std::vector<uint32_t> bmk;
    for (auto& e : bcols) { bo.push_back(e.second.first); bmk.push_back(e.second.second); }
    bo.push_back(0);
    bmk.push_back(0);
    long long* dbo = c.alloc<long long>(bo.size());
    uint32_t* dbm = c.alloc<uint32_t>(bmk.size());
    DB_CUDA(cudaMemcpyAsync(dbo, bo.data(), sizeof(long long) * bo.size(), cudaMemcpyHostToDevice, c.st));
    DB_CUDA(cudaMemcpyAsync(dbm, bmk.data(), sizeof(uint32_t) * bmk.size(), cudaMemcpyHostToDevice, c.st));
    a.bcoff = dbo;
    a.bcmask = dbm;
    a.nbcols = (int)bcols.size();
  }
  a.ncells = cv.ncells;
  a.cell_start = cv.cell_start;
  a.cell_key = cv.cell_key;
  a.cell_of = cv.cell_of;
  a.Ps = Ps;
  a.idx = idx;
  a.core_s = core_s;
  a.core_cnt = core_cnt;
  a.min_pts = min_pts;
  a.n = n;
  a.counters = o->counters;  // [4], zeroed by the caller
  a.mixed_list = c.alloc<uint32_t>(cv.ncells);
  by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
    constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
    constexpr bool W = decltype(Wd)::value;
    sp_core_kernel<DIM, D, W><<<grid_for(n, 256, 1 << 30), 256, 0, c.st>>>(a);
  });
  c.launched();
  sp_cells_kernel<<<grid_for(cv.ncells, 256, 1 << 30), 256, 0, c.st>>>(a);
  c.launched();
  partition_mixed(c, g, cv, a.mixed_list, a.counters + 3, Ps, idx, core_s, n);
  o->stash = new SpArgs(a);
}

void sparse_cluster(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps,
                    const uint32_t* core_cnt, bool wide, bool waves, uint32_t* parent,
                    unsigned long long* tested, SparseOut* o) {
  (void)waves;  // one pass: small pairs are tested without Find (see sp_pairs_kernel)
  SpArgs& a = *(SpArgs*)o->stash;
  a.parent = parent;
  a.large_cap = cv.ncells + 4096;
  a.large = c.alloc<uint2>(a.large_cap);
  uf_init(c, parent, cv.ncells);
  const unsigned grid = grid_for(((int64_t)cv.ncells + 31) / 32 * 32, 256, c.sms * 16);
  c.zero(a.counters + 2, sizeof(uint32_t));
  by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
    constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
    constexpr bool W = decltype(Wd)::value;
    sp_pairs_kernel<DIM, D, W><<<grid, 256, 0, c.st>>>(a, tested);
  });
  c.launched();
  bcp_large(c, g, cv, Ps, core_cnt, parent, a.large, a.counters + 2, a.large_cap, wide);
}

int64_t sparse_border(Ctx& c, const Geo& g, const uint32_t* cell_label, int64_t n, bool wide,
                      int64_t* border_off, unsigned long long* nborder, SparseOut* o) {
  SpArgs& a = *(SpArgs*)o->stash;
  a.cell_label = cell_label;
  a.bcnt = c.alloc<uint32_t>(n);
  a.tmp_lab = c.alloc<uint32_t>((size_t)n * SP_MAXL);
  a.tmp_n = c.alloc<uint8_t>(n);
  a.nborder = nborder;
  c.zero(a.bcnt, sizeof(uint32_t) * n);
  by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
    constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
    constexpr bool W = decltype(Wd)::value;
    sp_border_kernel<DIM, D, W><<<grid_for(n, 256, 1 << 30), 256, 0, c.st>>>(a);
  });
  c.launched();
  exclusive_scan_u32_i64(c, a.bcnt, border_off, n);
  return c.read(border_off + n);
}

void sparse_border_fill(Ctx& c, const Geo& g, bool wide, const int64_t* border_off,
                        int32_t* border_ids, SparseOut* o) {
  SpArgs& a = *(SpArgs*)o->stash;
  by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
    constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
    constexpr bool W = decltype(Wd)::value;
    sp_border_fill_kernel<DIM, D, W><<<grid_for(a.n, 256, 1 << 30), 256, 0, c.st>>>(a, border_off,
                                                                                   border_ids);
  });
  c.launched();
}

void sparse_release(SparseOut* o) {
  delete (SpArgs*)o->stash;
  o->stash = nullptr;
}

}  // namespace db
