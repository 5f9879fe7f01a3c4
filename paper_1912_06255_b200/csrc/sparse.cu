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
  const long long* offs;     // all stencil offsets (padded linear units), nearest first
  int noffs;
  const long long* woffs;    // per-wave back offsets, concatenated
  int wbeg[4];               // wave w: woffs[wbeg[w] .. wbeg[w+1])
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

__global__ void popc_kernel(const uint32_t* __restrict__ bm, uint64_t words, uint32_t* __restrict__ cnt) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < words) cnt[i] = __popc(bm[i]);
}

// ------------------------------------------------------------ MarkCore (a6)
// Thread per sorted point, two phases. (1) probe every stencil offset (no
// divergence: consecutive lanes probe adjacent directory words) and keep the
// cells found in a per-thread list (<= SP_MAX_LIST entries, L1); (2) count
// over those cells only, nearest first, stopping at minPts (Alg 2,
// P:L571-598; own cell without a distance test).
constexpr int SP_MAX_LIST = 128;

template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_core_kernel(SpArgs a) {
  __shared__ long long so[SP_MAX_OFFS];
  for (int i = threadIdx.x; i < a.noffs; i += blockDim.x) so[i] = a.offs[i];
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  const uint32_t g = a.cell_of[j];
  const uint32_t m = a.cell_start[g + 1] - a.cell_start[g];
  if ((int64_t)m >= a.min_pts) { a.core_s[j] = 1; return; }  // dense cell
  const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
  uint32_t list[SP_MAX_LIST];
  int nf = 0;
  for (int t = 0; t < a.noffs; ++t) {
    const uint32_t h = rd_lookup(a.bm, a.pre, base + (uint64_t)so[t]);
    if (h != MISS) list[nf++] = h;
  }
  int32_t p[D];
  load_pt<D>(a.Ps, j, p);
  int64_t count = m;
  for (int f = 0; f < nf && count < a.min_pts; ++f) {
    const uint32_t h = list[f];
    const uint32_t he = a.cell_start[h + 1];
    for (uint32_t u = a.cell_start[h]; u < he; ++u) {
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
  const uint32_t cb = __ballot_sync(DB_FULL, core_cell);
  if ((threadIdx.x & 31) == 0 && cb) atomicAdd(a.counters + 0, (uint32_t)__popc(cb));
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
// Warp per 32-cell chunk; for each core cell of the chunk, lanes probe the
// wave's back offsets; a lane holding a pair (g, h) with Find(g) != Find(h)
// tests it (small: inline BCP with early exit; large: queued).
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_pairs_kernel(SpArgs a, int wave, unsigned long long* tested) {
  __shared__ long long so[SP_MAX_OFFS];
  const int wb = wave >= 0 ? a.wbeg[wave] : a.wbeg[0];
  const int we = wave >= 0 ? a.wbeg[wave + 1] : a.wbeg[3];
  const int nw = we - wb;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) so[i] = a.woffs[wb + i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t mine = 0;
  for (uint32_t c0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; c0 < a.ncells;
       c0 += nwarps * 32) {
    const uint32_t gl = c0 + lane;
    const uint32_t kl = gl < a.ncells ? a.core_cnt[gl] : 0;
    uint32_t cm = __ballot_sync(DB_FULL, kl > 0);
    while (cm) {
      const int src = __ffs(cm) - 1;
      cm &= cm - 1;
      const uint32_t g = c0 + src;
      const uint32_t kg = __shfl_sync(DB_FULL, kl, src);
      const uint32_t sg = a.cell_start[g];
      const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
      for (int t0 = 0; t0 < nw; t0 += 32) {
        const int t = t0 + lane;
        const uint32_t h = t < nw ? rd_lookup(a.bm, a.pre, base + (uint64_t)so[t]) : MISS;
        if (h == MISS) continue;
        const uint32_t kh = a.core_cnt[h];
        if (kh == 0) continue;
        if (uf_find(a.parent, g) == uf_find(a.parent, h)) continue;
        ++mine;
        if ((uint64_t)kg * kh > 64) {
          const uint32_t slot = atomicAdd(a.counters + 2, 1u);
          if (slot < a.large_cap) { a.large[slot] = make_uint2(g, h); continue; }
          // list full: test the pair here (correct, only slower)
        }
        const uint32_t sh = a.cell_start[h];
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
  if (mine) atomicAdd(tested, (unsigned long long)mine);
}

// --------------------------------------------------------- ClusterBorder (a10)
// Smallest label > `after` among clusters with a core point within eps of p
// (storage-free enumeration for points with more than SP_MAXL labels).
template <int DIM, int D, bool WIDE>
__device__ uint32_t sp_next_label(const SpArgs& a, const long long* so, const int32_t* p, uint32_t g,
                                  uint64_t base, int64_t after) {
  uint32_t best = MISS;
  if (a.core_cnt[g] > 0 && (int64_t)a.cell_label[g] > after) best = a.cell_label[g];
  for (int t = 0; t < a.noffs; ++t) {
    const uint32_t h = rd_lookup(a.bm, a.pre, base + (uint64_t)so[t]);
    if (h == MISS) continue;
    const uint32_t kh = a.core_cnt[h];
    if (kh == 0) continue;
    const uint32_t lab = a.cell_label[h];
    if ((int64_t)lab <= after || lab >= best) continue;
    const uint32_t sh = a.cell_start[h];
    for (uint32_t v = sh; v < sh + kh; ++v) {
      int32_t q[D];
      load_pt<D>(a.Ps, v, q);
      if (within<D, WIDE>(p, q, a.g.clampc, a.g.eps2)) { best = lab; break; }
    }
  }
  return best;
}

// Thread per sorted non-core point, two phases as in MarkCore: (1) list the
// stencil cells holding core points; (2) scan their core points, skipping
// cells whose label is already in the set (four registers, unused = ~0,
// sorted by a 4-input network at the end; larger sets are enumerated without
// storage in ascending order). Own-cell core points give their label with no
// distance test.
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_border_kernel(SpArgs a) {
  __shared__ long long so[SP_MAX_OFFS];
  for (int i = threadIdx.x; i < a.noffs; i += blockDim.x) so[i] = a.offs[i];
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  bool bord = false;
  if (j < a.n && !a.core_s[j]) {
    const uint32_t g = a.cell_of[j];
    const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
    uint32_t list[SP_MAX_LIST];
    int nf = 0;
    for (int t = 0; t < a.noffs; ++t) {
      const uint32_t h = rd_lookup(a.bm, a.pre, base + (uint64_t)so[t]);
      if (h != MISS && a.core_cnt[h] > 0) list[nf++] = h;
    }
    int32_t p[D];
    load_pt<D>(a.Ps, j, p);
    uint32_t L0 = MISS, L1 = MISS, L2 = MISS, L3 = MISS;
    int nl = 0;
    bool ovf = false;
    if (a.core_cnt[g] > 0) { L0 = a.cell_label[g]; nl = 1; }
    for (int f = 0; f < nf && !ovf; ++f) {
      const uint32_t h = list[f];
      const uint32_t lab = a.cell_label[h];
      if (lab == L0 || lab == L1 || lab == L2 || lab == L3) continue;
      const uint32_t sh = a.cell_start[h], kh = a.core_cnt[h];
      for (uint32_t v = sh; v < sh + kh; ++v) {
        int32_t q[D];
        load_pt<D>(a.Ps, v, q);
        if (within<D, WIDE>(p, q, a.g.clampc, a.g.eps2)) {
          if (nl == 0) L0 = lab;
          else if (nl == 1) L1 = lab;
          else if (nl == 2) L2 = lab;
          else if (nl == 3) L3 = lab;
          else ovf = true;
          ++nl;
          break;
        }
      }
    }
    uint32_t cnt;
    if (!ovf) {
      auto cs = [](uint32_t& x, uint32_t& y) { const uint32_t lo = min(x, y), hi = max(x, y); x = lo; y = hi; };
      cs(L0, L1); cs(L2, L3); cs(L0, L2); cs(L1, L3); cs(L1, L2);
      uint32_t* dst = a.tmp_lab + (size_t)j * SP_MAXL;
      dst[0] = L0; dst[1] = L1; dst[2] = L2; dst[3] = L3;
      a.tmp_n[j] = (uint8_t)nl;
      cnt = (uint32_t)nl;
    } else {
      int64_t after = -1;
      cnt = 0;
      while (true) {
        const uint32_t nx = sp_next_label<DIM, D, WIDE>(a, so, p, g, base, after);
        if (nx == MISS) break;
        ++cnt;
        after = nx;
      }
      a.tmp_n[j] = 0xff;
    }
    a.bcnt[a.idx[j]] = cnt;
    bord = cnt > 0;
  }
  const uint32_t b = __ballot_sync(DB_FULL, bord);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(a.nborder, (unsigned long long)__popc(b));
}

// Copy the staged label sets into the CSR (thread per sorted point).
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_border_fill_kernel(SpArgs a, const int64_t* __restrict__ border_off,
                                                             int32_t* __restrict__ border_ids) {
  __shared__ long long so[SP_MAX_OFFS];
  for (int i = threadIdx.x; i < a.noffs; i += blockDim.x) so[i] = a.offs[i];
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n || a.core_s[j]) return;
  const uint8_t nl = a.tmp_n[j];
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
    const uint32_t nx = sp_next_label<DIM, D, WIDE>(a, so, p, g, base, after);
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
  if (stencil_offsets(g).size() / g.d > (size_t)SP_MAX_LIST) return false;
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
  // stencil offsets in padded linear units, nearest first; back offsets per wave
  std::vector<int8_t> offs = stencil_offsets(g);
  const int noffs = (int)(offs.size() / g.d);
  std::vector<long long> lin((size_t)noffs + 1, 0), wl[3];
  for (int t = 0; t < noffs; ++t) {
    long long dl = 0;
    int l1 = 0;
    for (int k = 0; k < g.d; ++k) {
      const int v = offs[(size_t)t * g.d + k];
      dl += (long long)v * (long long)a.stride[k];
      l1 += v < 0 ? -v : v;
    }
    lin[t] = dl;
    if (dl < 0) wl[l1 <= 1 ? 0 : (l1 == 2 ? 1 : 2)].push_back(dl);
  }
  std::vector<long long> wall;
  a.wbeg[0] = 0;
  for (int w = 0; w < 3; ++w) {
    wall.insert(wall.end(), wl[w].begin(), wl[w].end());
    a.wbeg[w + 1] = (int)wall.size();
  }
  wall.push_back(0);
  long long* doffs = c.alloc<long long>(lin.size());
  long long* dwoffs = c.alloc<long long>(wall.size());
  DB_CUDA(cudaMemcpyAsync(doffs, lin.data(), sizeof(long long) * lin.size(), cudaMemcpyHostToDevice, c.st));
  DB_CUDA(cudaMemcpyAsync(dwoffs, wall.data(), sizeof(long long) * wall.size(), cudaMemcpyHostToDevice, c.st));
  a.offs = doffs;
  a.noffs = noffs;
  a.woffs = dwoffs;
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
  SpArgs& a = *(SpArgs*)o->stash;
  a.parent = parent;
  a.large_cap = cv.ncells + 4096;
  a.large = c.alloc<uint2>(a.large_cap);
  uf_init(c, parent, cv.ncells);
  // waves: back offsets of lattice L1 norm 1, then 2, then >= 3, each drained
  // (large pairs included) before the next; without waves one launch (-1)
  const int first = waves ? 0 : -1, last = waves ? 2 : -1;
  const unsigned grid = grid_for(((int64_t)cv.ncells + 31) / 32 * 32, 256, c.sms * 16);
  for (int w = first; w <= last; ++w) {
    c.zero(a.counters + 2, sizeof(uint32_t));
    by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
      constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
      constexpr bool W = decltype(Wd)::value;
      sp_pairs_kernel<DIM, D, W><<<grid, 256, 0, c.st>>>(a, w, tested);
    });
    c.launched();
    bcp_large(c, g, cv, Ps, core_cnt, parent, a.large, a.counters + 2, a.large_cap, wide);
  }
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
