// neighbors.cu — NeighborCells, memoised as a CSR
// ("we cache the result on its first query").
//
// Two cells whose lattice coordinates differ by delta can hold a pair within
// eps iff sum_k gap_k^2 <= eps^2 with gap_k = (|delta_k|-1) s + 1 for
// delta_k != 0 (the closest integer coordinates of the two cells; DESIGN.md
// reading 7). This predicate is exact (complete and tight), so every stage
// that scans "neighbouring cells" sees exactly the cells that can
// matter.
//   d <= 3: enumerate the stencil of offsets satisfying the predicate (21 in
//           2D, 117 in 3D including self) and probe the cell hash table
//           (P:L489-493), one thread per cell, the warp's lanes being 32
//           consecutive cells so that their probes coalesce.
//   d >= 4: "enumerating all possible neighboring cells can be inefficient in
//           practice for higher dimensions"; the
//           paper inserts the cells into a k-d tree and runs range queries.
//           Here: a bounding-volume tree over the cells in Morton order
//           (leaves of 32 cells, implicit complete binary tree of integer
//           boxes, built bottom-up in one kernel), queried by one warp per
//           cell with the same exact gap test on boxes; lanes test the 32
//           cells of a leaf at once.
#include <algorithm>

#include <cstdlib>

#include "internal.h"

namespace db {

// Offsets delta != 0 with sum_k gap_k^2 <= eps^2, ordered by ascending squared
// gap so that every CSR row lists the nearest cells first (the early exits of
// MarkCore, BCP and ClusterBorder then fire sooner); ties lexicographic.
std::vector<int8_t> stencil_offsets(const Geo& g) {
  const int d = g.d, R = (int)g.R;
  std::vector<std::pair<unsigned __int128, std::vector<int8_t>>> all;
  std::vector<int> off(d, -R);
  while (true) {
    bool zero = true;
    unsigned __int128 acc = 0;
    for (int k = 0; k < d; ++k) {
      int a = off[k] < 0 ? -off[k] : off[k];
      if (a) {
        zero = false;
        unsigned __int128 gap = (unsigned __int128)(a - 1) * g.s + 1;
        acc += gap * gap;
      }
    }
    if (!zero && acc <= g.eps2) all.push_back({acc, std::vector<int8_t>(off.begin(), off.end())});
    int k = d - 1;
    while (k >= 0 && off[k] == R) { off[k] = -R; --k; }
    if (k < 0) break;
    ++off[k];
  }
  std::stable_sort(all.begin(), all.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<int8_t> out;
  for (auto& e : all) out.insert(out.end(), e.second.begin(), e.second.end());
  return out;
}

// ------------------------------------------------------------------ stencil
// Offsets live in shared memory as {delta_0..2, packed key (or directory)
// delta}. Two mappings:
//  * thread per cell (many cells): the 32 lanes of a warp are 32 consecutive
//    cells in key order (mostly one column, consecutive last-axis coordinates)
//    probing the same offset, so their keys are consecutive and the probes of
//    one warp instruction coalesce (locality-preserving slot hash, or the
//    dense directory);
//  * warp per cell (few cells, e.g. seed-spreader data): lanes over offsets,
//    so a handful of cells still fill the machine.
// DENSE: a directory over the lattice padded by R cells on every side (cell
// id or ~0), indexed like the key (axis 0 major), chosen when the padded
// lattice has at most DENSE_PER_POINT cells per point: one load per probe and
// no range checks (out-of-range neighbours land in the padding).
// The count pass also accumulates ub[g] = sum of the neighbours' sizes, the
// MarkCore upper bound (core.cu), saturating at 2^32-1.
constexpr int MAX_SMEM_OFFS = 2048;
constexpr int64_t DENSE_PER_POINT = 8;
constexpr uint32_t WARP_PER_CELL_BELOW = 1u << 15;

struct __align__(16) StencilOff {
  int8_t d[8];      // per-axis lattice offset
  long long delta;  // packed-key (or padded directory) offset
};

struct Lattice {
  uint64_t stride[3];
};

template <int DIM, bool DENSE>
__device__ __forceinline__ uint32_t probe(const StencilOff& o, const uint32_t* cc, uint64_t base,
                                          const Geo& g, const Slot* __restrict__ T, uint64_t mask,
                                          const uint32_t* __restrict__ dir) {
  if constexpr (DENSE) {
    return __ldg(dir + (base + (uint64_t)o.delta));
  } else {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < (DIM ? DIM : 8); ++k) {
      if (DIM || k < g.d) {
        const int64_t q = (int64_t)cc[k] + o.d[k];
        ok &= (q >= 0) & (q <= (int64_t)g.maxc[k]);
      }
    }
    if (!ok) return 0xffffffffu;
    return hash_lookup(T, mask, base + (uint64_t)o.delta);
  }
}

template <int DIM, bool DENSE, bool WARP>
__global__ void __launch_bounds__(256) nbr_stencil_kernel(
    int fill, const uint64_t* __restrict__ cell_key, uint32_t ncells, Geo g,
    const StencilOff* __restrict__ offs, int noffs, const Slot* __restrict__ T, uint64_t mask,
    const uint32_t* __restrict__ dir, Lattice lat, const uint32_t* __restrict__ cell_start,
    uint32_t* __restrict__ cnt, uint32_t* __restrict__ ub, const uint64_t* __restrict__ off,
    uint32_t* __restrict__ nbr, int n0, int n01, uint32_t* __restrict__ ccount) {
  __shared__ StencilOff s_offs[MAX_SMEM_OFFS];
  const bool in_smem = noffs <= MAX_SMEM_OFFS;
  if (in_smem)
    for (int i = threadIdx.x; i < noffs; i += blockDim.x) s_offs[i] = offs[i];
  __syncthreads();
  const StencilOff* O = in_smem ? s_offs : offs;
  const int lane = threadIdx.x & 31;
  const uint32_t stride = WARP ? (gridDim.x * blockDim.x) >> 5 : gridDim.x * blockDim.x;
  uint32_t cell = WARP ? (blockIdx.x * blockDim.x + threadIdx.x) >> 5 : blockIdx.x * blockDim.x + threadIdx.x;
  for (; cell < ncells; cell += stride) {
    const uint64_t key = cell_key[cell];
    uint32_t cc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) cc[k] = (k < (DIM ? DIM : g.d)) ? cell_coord(key, g, k) : 0;
    uint64_t base = key;
    if constexpr (DENSE) {
      base = 0;
#pragma unroll
      for (int k = 0; k < DIM; ++k) base += (uint64_t)(cc[k] + g.R) * lat.stride[k];
    }
    uint64_t wpos = fill ? off[cell] : 0;
    uint32_t total = 0, c0 = 0, c1 = 0;  // (offsets are class-sorted: [0, n0) class 0, [n0, n01) class 1)
    uint64_t sum = 0;
    if constexpr (WARP) {
      const uint32_t lt = lanemask_lt();
      for (int t0 = 0; t0 < noffs; t0 += 32) {
        const int t = t0 + lane;
        uint32_t id = 0xffffffffu;
        if (t < noffs) id = probe<DIM, DENSE>(O[t], cc, base, g, T, mask, dir);
        const bool found = id != 0xffffffffu;
        const uint32_t b = __ballot_sync(DB_FULL, found);
        if (fill) {
          if (found) nbr[wpos + __popc(b & lt)] = id;
        } else if (found) {
          sum += cell_start[id + 1] - cell_start[id];
        }
        c0 += __popc(__ballot_sync(DB_FULL, found && t < n0));
        c1 += __popc(__ballot_sync(DB_FULL, found && t >= n0 && t < n01));
        wpos += __popc(b);
        total += __popc(b);
      }
      if (!fill) {
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(DB_FULL, sum, o);
        if (lane == 0) {
          cnt[cell] = total;
          ub[cell] = (uint32_t)min(sum, (uint64_t)0xffffffffu);
          if (ccount) { ccount[cell] = c0; ccount[ncells + cell] = c1; }
        }
      }
    } else {
      for (int t = 0; t < noffs; ++t) {
        const uint32_t id = probe<DIM, DENSE>(O[t], cc, base, g, T, mask, dir);
        if (id == 0xffffffffu) continue;
        if (fill) nbr[wpos++] = id;
        else sum += cell_start[id + 1] - cell_start[id];
        ++total;
        c0 += t < n0;
        c1 += t >= n0 && t < n01;
      }
      if (!fill) {
        cnt[cell] = total;
        ub[cell] = (uint32_t)min(sum, (uint64_t)0xffffffffu);
        if (ccount) { ccount[cell] = c0; ccount[ncells + cell] = c1; }
      }
    }
  }
}

__global__ void dense_fill_kernel(const uint64_t* __restrict__ cell_key, uint32_t ncells, Geo g,
                                  Lattice lat, uint32_t* __restrict__ dir) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncells) return;
  const uint64_t key = cell_key[i];
  uint64_t lin = 0;
  for (int k = 0; k < g.d; ++k) lin += (uint64_t)(cell_coord(key, g, k) + g.R) * lat.stride[k];
  dir[lin] = i;
}

// Size of the neighbour CSR for the allocations: the exact count (a host read,
// i.e. a synchronisation) only when the structural bound would be large;
// otherwise the bound, and the exact count stays on the device (c.nbr_total_d,
// read with the call's final counters).
constexpr uint64_t NBR_BOUND_MAX = 1ull << 25;  // entries (128 MB of u32, 256 MB of pairs)
static uint64_t nbr_total_bound(Ctx& c, const uint64_t* total_d, uint64_t bound) {
  c.nbr_total_d = total_d;
  if (bound <= NBR_BOUND_MAX) return bound;
  return c.read(total_d);
}

void neighbors_stencil(Ctx& c, const Geo& g, const uint64_t* cell_key, const uint32_t* cell_start,
                       uint32_t ncells, int64_t n, uint64_t** nbr_off, uint32_t** nbr,
                       uint32_t** ub_out, uint64_t* total, bool* dense_out, const uint32_t** ccls) {
  std::vector<int8_t> offs0 = stencil_offsets(g);
  const int noffs = (int)(offs0.size() / g.d);
  // rows by class of lattice L1 distance (1, 2, >= 3; gap order inside a
  // class) so that ClusterCore's waves read only their segment
  std::vector<int8_t> offs;
  offs.reserve(offs0.size());
  int ncls[3] = {0, 0, 0};
  for (int cl = 0; cl < 3; ++cl)
    for (int t = 0; t < noffs; ++t) {
      int l1 = 0;
      for (int k = 0; k < g.d; ++k) l1 += std::abs((int)offs0[(size_t)t * g.d + k]);
      const int c = l1 <= 1 ? 0 : (l1 == 2 ? 1 : 2);
      if (c != cl) continue;
      offs.insert(offs.end(), offs0.begin() + (size_t)t * g.d, offs0.begin() + (size_t)(t + 1) * g.d);
      ++ncls[cl];
    }
  const int n0 = ncls[0], n01 = ncls[0] + ncls[1];
  // dense directory when the padded lattice is small relative to n (d <= 3 only)
  Lattice lat{{0, 0, 0}};
  bool dense = false;
  if (g.d <= 3) {
    unsigned __int128 vol = 1;
    for (int k = g.d - 1; k >= 0; --k) {
      lat.stride[k] = (uint64_t)vol;
      vol *= (unsigned __int128)g.maxc[k] + 1 + 2 * (unsigned __int128)g.R;
    }
    dense = vol <= (unsigned __int128)(DENSE_PER_POINT * n + (1 << 20));
    if (dense) {
      const uint64_t volume = (uint64_t)vol;
      uint32_t* dir = c.alloc<uint32_t>(volume);
      DB_CUDA(cudaMemsetAsync(dir, 0xff, sizeof(uint32_t) * volume, c.st));
      dense_fill_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(cell_key, ncells, g, lat, dir);
      c.launched();
      c.dense_dir = dir;
      c.dense_lat[0] = lat.stride[0]; c.dense_lat[1] = lat.stride[1]; c.dense_lat[2] = lat.stride[2];
    }
  }
  Slot* T = nullptr;
  uint64_t mask = 0;
  if (!dense) mask = build_hash(c, cell_key, ncells, &T);
  *dense_out = dense;
  std::vector<StencilOff> so((size_t)noffs + 1);
  for (int t = 0; t < noffs; ++t) {
    int64_t dl = 0;
    StencilOff& o = so[t];
    for (int k = 0; k < 8; ++k) o.d[k] = 0;
    for (int k = 0; k < g.d; ++k) {
      const int8_t v = offs[(size_t)t * g.d + k];
      o.d[k] = v;
      dl += (int64_t)v * (dense ? (int64_t)lat.stride[k] : (int64_t)(1ull << g.shift[k]));
    }
    o.delta = dl;
  }
  StencilOff* doffs = c.alloc<StencilOff>(so.size());
  c.upload(doffs, so.data(), so.size());
  uint32_t* cnt = c.alloc<uint32_t>(ncells);
  uint32_t* ub = c.alloc<uint32_t>(ncells);
  uint64_t* off = c.alloc<uint64_t>((size_t)ncells + 1);
  uint32_t* ccount = c.alloc<uint32_t>(2 * (size_t)ncells);
  const bool warp = ncells < WARP_PER_CELL_BELOW;
  const unsigned grid = warp ? grid_for((int64_t)ncells * 32, 256, 1 << 30) : grid_for(ncells, 256, 1 << 30);
  auto launch = [&](int fill, uint32_t* list) {
    auto go = [&](auto Dc, auto Dn, auto Wp) {
      constexpr int DIM = decltype(Dc)::value;
      constexpr bool DN = decltype(Dn)::value, WP = decltype(Wp)::value;
      nbr_stencil_kernel<DIM, DN, WP><<<grid, 256, 0, c.st>>>(fill, cell_key, ncells, g, doffs, noffs, T,
                                                              mask, c.dense_dir, lat, cell_start, cnt, ub,
                                                              off, list, n0, n01, ccount);
    };
    using F = std::false_type;
    using Tt = std::true_type;
    auto by_mode = [&](auto Dc) {
      if (dense) { if (warp) go(Dc, Tt(), Tt()); else go(Dc, Tt(), F()); }
      else { if (warp) go(Dc, F(), Tt()); else go(Dc, F(), F()); }
    };
    if (g.d == 1) by_mode(std::integral_constant<int, 1>());
    else if (g.d == 2) by_mode(std::integral_constant<int, 2>());
    else if (g.d == 3) by_mode(std::integral_constant<int, 3>());
    else {  // forced stencil, d >= 4: hash only, runtime d
      if (warp) go(std::integral_constant<int, 0>(), F(), Tt());
      else go(std::integral_constant<int, 0>(), F(), F());
    }
    c.launched();
  };
  launch(0, nullptr);
  exclusive_scan_u32_u64(c, cnt, off, ncells);
  *total = nbr_total_bound(c, off + ncells, (uint64_t)ncells * (uint64_t)noffs);
  uint32_t* list = c.alloc<uint32_t>(*total + 1);
  launch(1, list);
  *nbr_off = off;
  *nbr = list;
  *ub_out = ub;
  *ccls = ccount;
}

// ------------------------------------------------------------ all-pairs cells
// d >= 4 with few cells (the seed-spreader configs: 1.6K-4.7K cells): testing
// every pair of cells with the exact gap predicate is cheaper than any tree
// (4.7K^2 = 2.2e7 tests against ~10^2 tree-node visits x 32 lanes per query
// with a per-warp stack). Warp per query cell, lanes over all cells, lattice
// coordinates pre-decoded (cc[8] per cell), the squared gap per axis from a
// shared table indexed by min(|delta|, R+1) (entry R+1 exceeds eps^2 on its
// own). Cells are bucketed by their axis-0 and axis-1 coordinates first
// (counting sort; axis 0 only when the 2D buckets would outnumber the cells
// four times), so a query scans 2R+1 runs of `order`: the axis-1 window
// c1 - R .. c1 + R of each axis-0 bucket c0 - R .. c0 + R. Rows come out in three classes
// of lattice L1 distance (1, 2, >= 3), nearest class first; the count pass
// records the class sizes so that the fill pass places every entry in one
// sweep.
constexpr uint32_t BRUTE_MAX_CELLS = 131072;
constexpr int GT_MAX = 64;

__global__ void decode_cells_kernel(const uint64_t* __restrict__ cell_key, uint32_t ncells, Geo g,
                                    uint32_t* __restrict__ cc) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncells) return;
  const uint64_t key = cell_key[i];
  uint4 a = make_uint4(0, 0, 0, 0), b = make_uint4(0, 0, 0, 0);
  uint32_t v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = k < g.d ? cell_coord(key, g, k) : 0u;
  a = make_uint4(v[0], v[1], v[2], v[3]);
  b = make_uint4(v[4], v[5], v[6], v[7]);
  reinterpret_cast<uint4*>(cc)[2 * i] = a;
  reinterpret_cast<uint4*>(cc)[2 * i + 1] = b;
}

__global__ void iota_kernel(uint32_t* __restrict__ v, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

// bucket of a cell: (axis-0, axis-1[, axis-2]) coordinates, (c0 * B1 + c1) * B2 + c2
// (B1 = 1: axis 0 only; B2 = 1: two axes)
__device__ __forceinline__ uint32_t cell_bucket(const uint32_t* __restrict__ cc, uint32_t i, uint32_t B1,
                                                uint32_t B2) {
  const uint32_t* c = cc + 8 * (size_t)i;
  return B1 > 1 ? (c[0] * B1 + c[1]) * B2 + (B2 > 1 ? c[2] : 0u) : c[0];
}

__global__ void bucket_count_kernel(const uint32_t* __restrict__ cc, uint32_t ncells, uint32_t B1, uint32_t B2,
                                    uint32_t* __restrict__ bcnt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ncells) atomicAdd(bcnt + cell_bucket(cc, i, B1, B2), 1u);
}

// (ccs: the cells' decoded coordinates in bucket order, so that a query
// streams its candidates' coordinates without the order[] indirection)
__global__ void bucket_fill_kernel(const uint32_t* __restrict__ cc, uint32_t ncells, uint32_t B1, uint32_t B2,
                                   const uint32_t* __restrict__ bstart, uint32_t* __restrict__ bcur,
                                   uint32_t* __restrict__ order, uint32_t* __restrict__ ccs,
                                   const uint32_t* __restrict__ cell_start, uint32_t* __restrict__ bsize,
                                   uint32_t* __restrict__ bpos) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncells) return;
  const uint32_t b = cell_bucket(cc, i, B1, B2);
  const uint32_t t = bstart[b] + atomicAdd(bcur + b, 1u);
  order[t] = i;
  bpos[i] = t;
  bsize[t] = cell_start[i + 1] - cell_start[i];
  reinterpret_cast<uint4*>(ccs)[2 * t] = reinterpret_cast<const uint4*>(cc)[2 * i];
  reinterpret_cast<uint4*>(ccs)[2 * t + 1] = reinterpret_cast<const uint4*>(cc)[2 * i + 1];
}

// PACK: 32-bit table entries gap^2 | |delta| << 27 (host: d (eps^2 + 1) <
// 2^27, d gmax < 32), so one add per axis accumulates both the squared gap
// and the lattice L1 distance that sets the class
template <int DD, bool PACK>
__global__ void __launch_bounds__(256) nbr_brute_kernel(int fill, const uint32_t* __restrict__ cc,
                                                        const uint32_t* __restrict__ ccs,
                                                        const uint32_t* __restrict__ order,
                                                        const uint32_t* __restrict__ bsize,
                                                        const uint32_t* __restrict__ bpos,
                                                        const uint32_t* __restrict__ bstart, uint32_t maxb,
                                                        uint32_t B1, uint32_t B2, uint32_t ncells, Geo g,
                                                        const uint64_t* __restrict__ gtab_g, int gmax,
                                                        const uint32_t* __restrict__ cell_start,
                                                        uint32_t* __restrict__ ccount /*[3][ncells]*/,
                                                        uint32_t* __restrict__ cnt, uint32_t* __restrict__ ub,
                                                        const uint64_t* __restrict__ off,
                                                        uint32_t* __restrict__ nbr, uint32_t* __restrict__ ownc) {
  // fill: 0 = count (cnt, ccount, ub), 1 = write class-sorted rows at off,
  // 2 = one symmetric pass: only candidates after q in bucket order are
  // tested, and a pair found adds (other cell | class << 30) to BOTH rows of
  // candidate capacity at off: q's own entries forward from the row start
  // (the warp's running count, ownc[q]), the mirror entries backward from
  // the row end through the counter cnt[] of the found cell (mirror entries
  // only; nbr_add_kernel then adds the own ones)
  // (nbr_compact_kernel then class-sorts the rows into the final CSR and
  // counts the classes and ub)
  __shared__ unsigned long long gt[GT_MAX + 1];
  __shared__ uint32_t gtp[GT_MAX + 1];
  for (int i = threadIdx.x; i <= gmax; i += blockDim.x) {
    gt[i] = gtab_g[i];
    if (PACK) gtp[i] = (uint32_t)gtab_g[i] | ((uint32_t)i << 27);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint4* C = reinterpret_cast<const uint4*>(cc);
  for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < ncells; q += nwarps) {
    uint32_t cq[8];
    {
      const uint4 a = C[2 * q], b = C[2 * q + 1];
      cq[0] = a.x; cq[1] = a.y; cq[2] = a.z; cq[3] = a.w; cq[4] = b.x; cq[5] = b.y; cq[6] = b.z; cq[7] = b.w;
    }
    uint64_t pos[3] = {0, 0, 0};
    if (fill == 2) {
      pos[0] = off[q];
    } else if (fill) {
      pos[0] = off[q];
      pos[1] = pos[0] + ccount[q];
      pos[2] = pos[1] + ccount[ncells + q];
    }
    uint32_t n3[3] = {0, 0, 0};  // fill == 1: warp totals; else per lane, reduced at the end
    uint32_t sum = 0;            // per lane: < n < 2^32
    const uint32_t c0 = maxb ? cq[0] : 0u;  // maxb = 0: a single bucket
    const uint32_t blo = c0 > g.R ? c0 - g.R : 0u, bhi = min(maxb, c0 + g.R);
    // B1 > 1: buckets by (axis 0, axis 1); for each axis-0 bucket the axis-1
    // window c1 - R .. c1 + R is one contiguous run of `order`. B2 > 1:
    // buckets by (axis 0, axis 1, axis 2); a run per (axis-0, axis-1) bucket
    // over the axis-2 window.
    const uint32_t y0 = B1 > 1 ? (cq[1] > g.R ? cq[1] - g.R : 0u) : 0u;
    const uint32_t y1 = B1 > 1 ? min(B1 - 1, cq[1] + g.R) : 0u;
    const uint32_t z0 = B2 > 1 ? (cq[2] > g.R ? cq[2] - g.R : 0u) : 0u;
    const uint32_t z1 = B2 > 1 ? min(B2 - 1, cq[2] + g.R) : 0u;
    const uint32_t tq = fill == 2 ? bpos[q] : 0u;
    // fill == 2: a lane's mirror entry (q into the found cell h's row) is
    // written one step after its counter atomic is issued, so the atomic's
    // round trip overlaps the next step's tests
    uint64_t pend_at = 0;      // last slot of the found cell's row (off[h + 1] - 1)
    uint32_t pend_slot = 0, pend_val = 0, own = 0;
    bool pend = false;
    for (uint32_t b0 = blo; b0 <= bhi; ++b0) {
    for (uint32_t b1 = y0; b1 <= (B2 > 1 ? y1 : y0); ++b1) {
    const uint32_t r0 = B2 > 1 ? (b0 * B1 + b1) * B2 + z0 : b0 * B1 + y0;
    const uint32_t r1 = B2 > 1 ? (b0 * B1 + b1) * B2 + z1 : b0 * B1 + y1;
    const uint32_t t1 = bstart[r1 + 1];
    const uint32_t ts = fill == 2 ? max(bstart[r0], tq + 1) : bstart[r0];
    for (uint32_t t0 = ts; t0 < t1; t0 += 32) {
      const uint32_t t = t0 + lane;
      int cls = -1;
      if (t < t1) {
        const uint4* CS = reinterpret_cast<const uint4*>(ccs);
        uint32_t ch[8];
        const uint4 a = CS[2 * t];
        ch[0] = a.x; ch[1] = a.y; ch[2] = a.z; ch[3] = a.w;
        if (DD > 4) {
          const uint4 b = CS[2 * t + 1];
          ch[4] = b.x; ch[5] = b.y; ch[6] = b.z; ch[7] = b.w;
        }
        uint32_t l1;
        bool in;
        if constexpr (PACK) {
          uint32_t acc = 0;
#pragma unroll
          for (int k = 0; k < DD; ++k) acc += gtp[min(__usad(ch[k], cq[k], 0u), (uint32_t)gmax)];
          l1 = acc >> 27;
          in = (acc & 0x7ffffffu) <= (uint32_t)g.eps2;
        } else {
          uint64_t acc = 0;
          l1 = 0;
#pragma unroll
          for (int k = 0; k < DD; ++k) {
            const uint32_t dl = min(__usad(ch[k], cq[k], 0u), (uint32_t)gmax);
            acc += gt[dl];
            l1 += dl;
          }
          in = acc <= g.eps2;
        }
        if (in && l1 > 0) cls = l1 <= 1 ? 0 : (l1 == 2 ? 1 : 2);  // (l1 = 0: the query itself)
      }
      if (fill == 2) {
        const uint32_t b = __ballot_sync(DB_FULL, cls >= 0);
        if (b) {
          if (cls >= 0) {
            const uint32_t h = order[t];
            nbr[pos[0] + own + __popc(b & lt)] = h | ((uint32_t)cls << 30);
            if (pend) nbr[pend_at - pend_slot] = pend_val;
            pend_slot = atomicAdd(cnt + h, 1u);
            pend_at = off[h + 1] - 1;
            pend_val = q | ((uint32_t)cls << 30);
            pend = true;
          }
          own += __popc(b);
        }
        continue;
      }
      if (fill == 1) {
        const uint32_t h = cls >= 0 ? order[t] : 0u;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const uint32_t b = __ballot_sync(DB_FULL, cls == c);
          if (cls == c) nbr[pos[c] + __popc(b & lt)] = h;
          pos[c] += __popc(b);
        }
      } else {
        n3[0] += cls == 0;
        n3[1] += cls == 1;
        n3[2] += cls == 2;
        if (cls >= 0) sum += bsize[t];
      }
    }
    }
    }
    if (pend) nbr[pend_at - pend_slot] = pend_val;
    if (fill == 2 && lane == 0) ownc[q] = own;  // (cnt[] holds the mirror entries only, their slots)
    if (fill == 0) {
      uint64_t sum64 = sum;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        sum64 += __shfl_xor_sync(DB_FULL, sum64, o);
        n3[0] += __shfl_xor_sync(DB_FULL, n3[0], o);
        n3[1] += __shfl_xor_sync(DB_FULL, n3[1], o);
        n3[2] += __shfl_xor_sync(DB_FULL, n3[2], o);
      }
      const uint64_t sum = sum64;
      if (lane == 0) {
        cnt[q] = n3[0] + n3[1] + n3[2];
        ccount[q] = n3[0];
        ccount[ncells + q] = n3[1];
        ub[q] = (uint32_t)min(sum, (uint64_t)0xffffffffu);
      }
    }
  }
}

__global__ void nbr_add_kernel(uint32_t* __restrict__ cnt, const uint32_t* __restrict__ ownc, uint32_t ncells) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ncells) cnt[i] += ownc[i];
}

__global__ void cell_size_kernel(const uint32_t* __restrict__ cell_start, uint32_t ncells,
                                 uint32_t* __restrict__ bsize) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < ncells) bsize[i] = cell_start[i + 1] - cell_start[i];
}

// candidate capacity of each cell's row: the length of its bucket runs (what
// nbr_brute_kernel scans), no distance tests
__global__ void nbr_cap_kernel(const uint32_t* __restrict__ cc, const uint32_t* __restrict__ bstart, uint32_t maxb,
                               uint32_t B1, uint32_t B2, uint32_t ncells, uint32_t R, uint32_t* __restrict__ cap) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ncells) return;
  const uint32_t c0 = maxb ? cc[8 * q] : 0u, c1 = cc[8 * q + 1], c2 = cc[8 * q + 2];
  const uint32_t blo = c0 > R ? c0 - R : 0u, bhi = min(maxb, c0 + R);
  const uint32_t y0 = B1 > 1 ? (c1 > R ? c1 - R : 0u) : 0u, y1 = B1 > 1 ? min(B1 - 1, c1 + R) : 0u;
  const uint32_t z0 = B2 > 1 ? (c2 > R ? c2 - R : 0u) : 0u, z1 = B2 > 1 ? min(B2 - 1, c2 + R) : 0u;
  uint32_t sum = 0;
  for (uint32_t b0 = blo; b0 <= bhi; ++b0)
    for (uint32_t b1 = y0; b1 <= (B2 > 1 ? y1 : y0); ++b1) {
      const uint32_t r0 = B2 > 1 ? (b0 * B1 + b1) * B2 + z0 : b0 * B1 + y0;
      const uint32_t r1 = B2 > 1 ? (b0 * B1 + b1) * B2 + z1 : b0 * B1 + y1;
      sum += bstart[r1 + 1] - bstart[r0];
    }
  cap[q] = sum;
}

// one warp per cell: the tagged row (candidate order) -> the final row,
// class-sorted, order kept inside a class (the rows fill == 1 writes)
__global__ void __launch_bounds__(256) nbr_compact_kernel(const uint32_t* __restrict__ tagged,
                                                          const uint64_t* __restrict__ toff,
                                                          const uint32_t* __restrict__ cnt,
                                                          const uint32_t* __restrict__ ownc,
                                                          const uint32_t* __restrict__ cell_start,
                                                          uint32_t* __restrict__ ccount, uint32_t* __restrict__ ub,
                                                          const uint64_t* __restrict__ off, uint32_t ncells,
                                                          uint32_t* __restrict__ nbr) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < ncells; q += nwarps) {
    // the row: own entries [0, own), mirror entries at its end
    const uint32_t* src = tagged + toff[q];
    const uint32_t len = cnt[q], own = ownc[q], skip = (uint32_t)(toff[q + 1] - toff[q]) - len;
    auto at = [&](uint32_t t) { return src[t < own ? t : t + skip]; };
    // class counts and ub (the sum of the neighbours' sizes)
    uint32_t n0 = 0, n1 = 0;
    uint64_t sum = 0;
    for (uint32_t t = lane; t < len; t += 32) {
      const uint32_t v = at(t), h = v & 0x3fffffffu, cls = v >> 30;
      n0 += cls == 0;
      n1 += cls == 1;
      sum += cell_start[h + 1] - cell_start[h];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      n0 += __shfl_xor_sync(DB_FULL, n0, o);
      n1 += __shfl_xor_sync(DB_FULL, n1, o);
      sum += __shfl_xor_sync(DB_FULL, sum, o);
    }
    if (lane == 0) {
      ccount[q] = n0;
      ccount[ncells + q] = n1;
      ub[q] = (uint32_t)min(sum, (uint64_t)0xffffffffu);
    }
    uint64_t pos[3];
    pos[0] = off[q];
    pos[1] = pos[0] + n0;
    pos[2] = pos[1] + n1;
    for (uint32_t t0 = 0; t0 < len; t0 += 32) {
      const uint32_t t = t0 + lane;
      const uint32_t v = t < len ? at(t) : 0xffffffffu;
      const uint32_t cls = v >> 30;
#pragma unroll
      for (uint32_t k = 0; k < 3; ++k) {
        const uint32_t b = __ballot_sync(DB_FULL, cls == k);
        if (cls == k) nbr[pos[k] + __popc(b & lt)] = v & 0x3fffffffu;
        pos[k] += __popc(b);
      }
    }
  }
}

constexpr uint64_t NBR_ONEPASS_MAX = 1ull << 29;  // tagged-row entries (2 GB)

static bool neighbors_brute(Ctx& c, const Geo& g, const uint64_t* cell_key, const uint32_t* cell_start,
                            uint32_t ncells, uint64_t** nbr_off, uint32_t** nbr, uint32_t** ub_out,
                            uint64_t* total, const uint32_t** ccls) {
  // squared gap per |delta| (u = |delta| clamped to R+1; entry R+1 > eps^2)
  const int gmax = (int)g.R + 1;
  if (gmax > GT_MAX || g.d < 4) return false;
  std::vector<unsigned long long> gt((size_t)gmax + 1);
  gt[0] = 0;
  for (int i = 1; i <= (int)g.R; ++i) {
    const unsigned long long gap = (unsigned long long)(i - 1) * g.s + 1;
    gt[i] = gap * gap;
  }
  gt[gmax] = g.eps2 + 1;
  unsigned long long* dgt = c.alloc<unsigned long long>(gt.size());
  c.upload(dgt, gt.data(), gt.size());
  uint32_t* cc = c.alloc<uint32_t>((size_t)ncells * 8);
  decode_cells_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(cell_key, ncells, g, cc);
  c.launched();
  // axis-0 buckets (one bucket if the axis is too long to bucket cheaply)
  uint32_t maxb = (uint64_t)g.maxc[0] < 4ull * ncells + 1024 ? g.maxc[0] : 0u;
  // two bucketed axes when their buckets fit the same budget
  const uint32_t B1 = maxb && g.d >= 2 &&
                              ((uint64_t)g.maxc[0] + 1) * ((uint64_t)g.maxc[1] + 1) < 4ull * ncells + 1024
                          ? g.maxc[1] + 1
                          : 1u;
  // a third bucketed axis when the lattice is crowded (many cells, clustered:
  // SS-varden 7D has 72K cells and ~1,150 neighbours per cell) and the 3D
  // bucket grid stays within 32 buckets per cell
  const uint64_t v3 = ((uint64_t)g.maxc[0] + 1) * ((uint64_t)g.maxc[1] + 1) * ((uint64_t)g.maxc[2] + 1);
  const uint32_t B2 = B1 > 1 && g.d >= 3 && ncells >= 16384 && v3 <= 32ull * ncells + (1u << 20)
                          ? g.maxc[2] + 1
                          : 1u;
  const uint64_t nbk = ((uint64_t)maxb + 1) * B1 * B2;  // buckets 0 .. nbk - 1
  uint32_t* bcnt = c.alloc<uint32_t>((size_t)nbk + 1);
  uint32_t* bstart = c.alloc<uint32_t>((size_t)nbk + 1);
  uint32_t* order = c.alloc<uint32_t>(ncells);
  uint32_t* ccs = cc;  // (one bucket: the cells in their own order)
  uint32_t* bsize = c.alloc<uint32_t>(ncells);  // points per cell, bucket order
  uint32_t* bpos = c.alloc<uint32_t>(ncells);   // each cell's position in bucket order
  c.zero(bcnt, sizeof(uint32_t) * ((size_t)nbk + 1));
  if (maxb) {
    bucket_count_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(cc, ncells, B1, B2, bcnt);
    c.launched();
    exclusive_scan_u32_u32(c, bcnt, bstart, (int64_t)nbk);
    c.zero(bcnt, sizeof(uint32_t) * ((size_t)nbk + 1));
    ccs = c.alloc<uint32_t>((size_t)ncells * 8);
    bucket_fill_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(cc, ncells, B1, B2, bstart, bcnt, order,
                                                                         ccs, cell_start, bsize, bpos);
    c.launched();
  } else {
    // one bucket: every cell (cc[0] is then clamped by maxb = 0 -> buckets 0..0)
    const uint32_t h2[2] = {0u, ncells};
    c.upload(bstart, h2, 2);
    iota_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(order, ncells);
    c.launched();
    cell_size_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(cell_start, ncells, bsize);
    c.launched();
  }
  uint32_t* ccount = c.alloc<uint32_t>(2 * (size_t)ncells);
  uint32_t* cnt = c.alloc<uint32_t>(ncells);
  uint32_t* ub = c.alloc<uint32_t>(ncells);
  uint64_t* off = c.alloc<uint64_t>((size_t)ncells + 1);
  const unsigned grid = grid_for((int64_t)ncells * 32, 256, c.sms * 16);
  const bool pack = (uint64_t)g.d * (g.eps2 + 1) < (1ull << 27) && (uint64_t)g.d * gmax < 32;
  uint32_t* ownc = nullptr;  // (one pass: own entries per row)
  auto launch = [&](int fill, uint32_t* list, const uint64_t* lo) {
    auto go = [&](auto kern) {
      kern<<<grid, 256, 0, c.st>>>(fill, cc, ccs, order, bsize, bpos, bstart, maxb, B1, B2, ncells, g,
                                   (const uint64_t*)dgt, gmax, cell_start, ccount, cnt, ub, lo, list, ownc);
    };
    if (g.d <= 4) {
      if (pack) go(nbr_brute_kernel<4, true>);
      else go(nbr_brute_kernel<4, false>);
    } else {
      if (pack) go(nbr_brute_kernel<8, true>);
      else go(nbr_brute_kernel<8, false>);
    }
    c.launched();
  };
  // one test pass when the candidate rows fit: rows of candidate capacity
  // (bucket runs) take the tagged neighbours and the counts; a compaction
  // pass class-sorts them into the CSR (two passes of tests otherwise: count,
  // then fill at the scanned offsets)
  bool onepass = false;
  if (maxb && ncells < (1u << 30) && !(c.flags & DBSCAN_F_NBR_TWO_PASS)) {
    uint32_t* cap = c.alloc<uint32_t>(ncells);
    uint64_t* toff = c.alloc<uint64_t>((size_t)ncells + 1);
    nbr_cap_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(cc, bstart, maxb, B1, B2, ncells, g.R, cap);
    c.launched();
    exclusive_scan_u32_u64(c, cap, toff, ncells);
    const uint64_t tcap = c.read(toff + ncells);
    if (tcap <= NBR_ONEPASS_MAX) {
      uint32_t* tagged = c.alloc<uint32_t>(tcap + 1);
      ownc = c.alloc<uint32_t>(ncells);
      c.zero(cnt, sizeof(uint32_t) * ncells);  // the rows' fill counters
      launch(2, tagged, toff);
      nbr_add_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(cnt, ownc, ncells);
      c.launched();
      exclusive_scan_u32_u64(c, cnt, off, ncells);
      *total = nbr_total_bound(c, off + ncells, tcap);
      uint32_t* list = c.alloc<uint32_t>(*total + 1);
      nbr_compact_kernel<<<grid, 256, 0, c.st>>>(tagged, toff, cnt, ownc, cell_start, ccount, ub, off, ncells,
                                                 list);
      c.launched();
      *nbr = list;
      onepass = true;
    }
  }
  if (!onepass) {
    launch(0, nullptr, off);
    exclusive_scan_u32_u64(c, cnt, off, ncells);
    *total = nbr_total_bound(c, off + ncells, (uint64_t)ncells * (uint64_t)ncells);
    uint32_t* list = c.alloc<uint32_t>(*total + 1);
    launch(1, list, off);
    *nbr = list;
  }
  *nbr_off = off;
  *ub_out = ub;
  *ccls = ccount;  // rows are class-sorted: waves read only their class's segment
  return true;
}

// ------------------------------------------------------------------ cell tree
constexpr int LEAF = 32;

struct Box {
  uint32_t lo[8];
  uint32_t hi[8];
};

// Morton code: interleave the bits of the lattice coordinates, most
// significant bit first, axis 0 first within a bit level; total width = bits.
__global__ void morton_kernel(const uint64_t* __restrict__ cell_key, uint32_t ncells, Geo g,
                              uint64_t* __restrict__ code, uint32_t* __restrict__ id) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncells) return;
  uint64_t key = cell_key[i];
  uint32_t cc[8];
  uint32_t maxw = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    cc[k] = k < g.d ? cell_coord(key, g, k) : 0;
    if (k < g.d) maxw = max(maxw, g.width[k]);
  }
  uint64_t m = 0;
  for (int b = (int)maxw - 1; b >= 0; --b)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < g.d && (uint32_t)b < g.width[k]) m = (m << 1) | ((cc[k] >> b) & 1u);
  code[i] = m;
  id[i] = i;
}

__device__ __forceinline__ uint64_t box_gap2(const uint32_t* q, const uint32_t* lo,
                                             const uint32_t* hi, const Geo& g) {
  uint64_t acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (k < g.d) {
      uint32_t dlt = q[k] < lo[k] ? lo[k] - q[k] : (q[k] > hi[k] ? q[k] - hi[k] : 0u);
      acc += gap_term(dlt, g);
    }
  }
  return acc;
}

// Leaves (thread per leaf slot of the padded power-of-two layer), then
// climb: the second child to arrive at a node builds its box.
__global__ void tree_build_kernel(const uint64_t* __restrict__ cell_key, const uint32_t* __restrict__ mcell,
                                  uint32_t ncells, Geo g, uint32_t P2, Box* nodes, uint32_t* flags) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P2) return;
  Box b;
#pragma unroll
  for (int k = 0; k < 8; ++k) { b.lo[k] = 0xffffffffu; b.hi[k] = 0; }
  const uint32_t s0 = i * LEAF, s1 = min(s0 + LEAF, ncells);
  for (uint32_t t = s0; t < s1; ++t) {
    uint64_t key = cell_key[mcell[t]];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < g.d) {
        uint32_t v = cell_coord(key, g, k);
        b.lo[k] = min(b.lo[k], v);
        b.hi[k] = max(b.hi[k], v);
      }
  }
  uint32_t node = P2 - 1 + i;
  nodes[node] = b;
  while (node > 0) {
    __threadfence();
    uint32_t parent = (node - 1) >> 1;
    if (atomicAdd(flags + parent, 1u) == 0) return;
    __threadfence();
    const volatile Box* l = nodes + 2 * parent + 1;
    const volatile Box* r = nodes + 2 * parent + 2;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      b.lo[k] = min(l->lo[k], r->lo[k]);
      b.hi[k] = max(l->hi[k], r->hi[k]);
    }
    nodes[parent] = b;
    node = parent;
  }
}

__global__ void __launch_bounds__(128) tree_query_kernel(
    int fill, const uint64_t* __restrict__ cell_key, const uint32_t* __restrict__ mcell,
    uint32_t ncells, Geo g, uint32_t P2, const Box* __restrict__ nodes,
    const uint32_t* __restrict__ cell_start, uint32_t* __restrict__ cnt, uint32_t* __restrict__ ub,
    const uint64_t* __restrict__ off, uint32_t* __restrict__ nbr) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t lt = lanemask_lt();
  for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < ncells; q += nwarps) {
    uint32_t cq[8];
    const uint64_t key = cell_key[q];
#pragma unroll
    for (int k = 0; k < 8; ++k) cq[k] = k < g.d ? cell_coord(key, g, k) : 0;
    uint64_t wpos = fill ? off[q] : 0;
    uint32_t total = 0;
    uint64_t sum = 0;
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
      const uint32_t node = stack[--sp];
      if (node >= P2 - 1) {
        const uint32_t t = (node - (P2 - 1)) * LEAF + lane;
        bool found = false;
        uint32_t h = 0;
        if (t < ncells) {
          h = mcell[t];
          if (h != q) {
            uint64_t hk = cell_key[h];
            uint64_t acc = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (k < g.d) {
                uint32_t a = cell_coord(hk, g, k);
                acc += gap_term(a > cq[k] ? a - cq[k] : cq[k] - a, g);
              }
            found = acc <= g.eps2;
          }
        }
        uint32_t b = __ballot_sync(DB_FULL, found);
        if (fill && found) nbr[wpos + __popc(b & lt)] = h;
        if (!fill && found) sum += cell_start[h + 1] - cell_start[h];
        wpos += __popc(b);
        total += __popc(b);
      } else {
        // children in reverse so the left child is visited first
        for (int ch = 2; ch >= 1; --ch) {
          const uint32_t cidx = 2 * node + ch;
          const Box& bx = nodes[cidx];
          if (box_gap2(cq, bx.lo, bx.hi, g) <= g.eps2) stack[sp++] = cidx;
        }
      }
    }
    if (!fill) {
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(DB_FULL, sum, o);
      if (lane == 0) {
        cnt[q] = total;
        ub[q] = (uint32_t)min(sum, (uint64_t)0xffffffffu);
      }
    }
  }
}

// Order each CSR row by ascending lattice gap to its cell (nearest first), a
// block per row: bitonic sort of (scaled squared gap << 32 | id) in shared
// memory. Rows longer than ROW_SORT_MAX stay in tree order (order only
// affects how soon early exits fire, never the result).
constexpr int ROW_SORT_MAX = 2048;

__global__ void __launch_bounds__(256) sort_rows_kernel(const uint64_t* __restrict__ cell_key,
                                                        uint32_t ncells, Geo g,
                                                        const uint64_t* __restrict__ off,
                                                        uint32_t* __restrict__ nbr) {
  __shared__ unsigned long long sk[ROW_SORT_MAX];
  for (uint32_t q = blockIdx.x; q < ncells; q += gridDim.x) {
    const uint64_t b = off[q], e = off[q + 1];
    const int len = (int)(e - b);
    if (len < 2 || len > ROW_SORT_MAX) continue;
    int P = 1;
    while (P < len) P <<= 1;
    const uint64_t kq = cell_key[q];
    const float inv = 1.0f / (float)g.eps2;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      unsigned long long v = ~0ull;
      if (i < len) {
        const uint32_t h = nbr[b + i];
        const uint64_t kh = cell_key[h];
        uint64_t acc = 0;
        for (int k = 0; k < g.d; ++k) {
          const uint32_t x = cell_coord(kq, g, k), y = cell_coord(kh, g, k);
          acc += gap_term(x > y ? x - y : y - x, g);
        }
        const uint32_t rank = (uint32_t)fminf((float)acc * inv * 2147483647.0f, 4294967295.0f);
        v = ((unsigned long long)rank << 32) | h;
      }
      sk[i] = v;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const unsigned long long a = sk[i], c2 = sk[ixj];
            const bool up = (i & k) == 0;
            if ((a > c2) == up) { sk[i] = c2; sk[ixj] = a; }
          }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < len; i += blockDim.x) nbr[b + i] = (uint32_t)sk[i];
    __syncthreads();
  }
}

void neighbors_tree(Ctx& c, const Geo& g, const uint64_t* cell_key, const uint32_t* cell_start,
                    uint32_t ncells, uint64_t** nbr_off, uint32_t** nbr, uint32_t** ub_out,
                    uint64_t* total, bool allow_brute, const uint32_t** ccls) {
  *ccls = nullptr;
  if (allow_brute && ncells <= BRUTE_MAX_CELLS &&
      neighbors_brute(c, g, cell_key, cell_start, ncells, nbr_off, nbr, ub_out, total, ccls))
    return;
  uint64_t* code0 = c.alloc<uint64_t>(ncells);
  uint64_t* code1 = c.alloc<uint64_t>(ncells);
  uint32_t* id0 = c.alloc<uint32_t>(ncells);
  uint32_t* id1 = c.alloc<uint32_t>(ncells);
  morton_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(cell_key, ncells, g, code0, id0);
  c.launched();
  uint64_t* ksorted;
  uint32_t* mcell;
  radix_sort_u64(c, code0, id0, code1, id1, ncells, (int)g.bits, &ksorted, &mcell);
  const uint32_t L = (ncells + LEAF - 1) / LEAF;
  uint32_t P2 = 1;
  while (P2 < L) P2 <<= 1;
  Box* nodes = c.alloc<Box>(2 * (size_t)P2 - 1);
  uint32_t* flags = c.alloc<uint32_t>(P2);
  c.zero(flags, sizeof(uint32_t) * P2);
  tree_build_kernel<<<grid_for(P2, 128, 1 << 30), 128, 0, c.st>>>(cell_key, mcell, ncells, g, P2,
                                                                   nodes, flags);
  c.launched();
  uint32_t* cnt = c.alloc<uint32_t>(ncells);
  uint32_t* ub = c.alloc<uint32_t>(ncells);
  uint64_t* off = c.alloc<uint64_t>((size_t)ncells + 1);
  const unsigned grid = grid_for((int64_t)ncells * 32, 128, c.sms * 32);
  tree_query_kernel<<<grid, 128, 0, c.st>>>(0, cell_key, mcell, ncells, g, P2, nodes, cell_start, cnt,
                                            ub, nullptr, nullptr);
  c.launched();
  exclusive_scan_u32_u64(c, cnt, off, ncells);
  *total = c.read(off + ncells);
  uint32_t* list = c.alloc<uint32_t>(*total + 1);
  tree_query_kernel<<<grid, 128, 0, c.st>>>(1, cell_key, mcell, ncells, g, P2, nodes, cell_start,
                                            nullptr, nullptr, off, list);
  c.launched();
  sort_rows_kernel<<<grid_for(ncells, 1, c.sms * 8), 256, 0, c.st>>>(cell_key, ncells, g, off, list);
  c.launched();
  *nbr_off = off;
  *nbr = list;
  *ub_out = ub;
}

}  // namespace db
