// group.cu — grouping points by cell with a hash table and one counting pass
// (SURVEY §8(a) rows a2-a4 in one; the paper's semisort, PAPER.md P:L475-483,
// next-row f3).
//
// The paper groups (cellID, pointID) pairs with a semisort and keeps the
// non-empty cells in a hash table. When the data has few cells
// (the seed-spreader configs: 10^2..10^4 cells for 10^6..10^7 points) an LSD
// radix sort spends 3-7 passes over 12-24 bytes per point to order keys that
// take only a few thousand values. Here instead:
//   A. count: every point computes its packed cell key; the lanes of a warp
//      holding one key (__match_any_sync) add their number to that key's slot
//      with one atomic (find-or-insert, linear probing);
//   B. the non-empty slots are compacted and ranked by key, so cell ids follow
//      key order exactly as after the radix sort (the sparse path's rank
//      directory relies on it); cell_start = exclusive scan of the counts in
//      rank order;
//   C. scatter: every point looks its key up again, the warp's lanes of one
//      cell take consecutive positions from the cell's cursor (one atomic per
//      warp and cell) and write the padded point, its input index and its
//      cell id there. The leader also records the smallest input index of its
//      run (atomicMin), which gives each cell's minimum index for a9.
// Order inside a cell is the atomics' order (not stable); nothing downstream
// needs input order inside a cell (labels take the minimum explicitly).
// A table holds at most 2^20 slots (16 MB, L2-resident); a probe longer than
// MAX_PROBE means too many cells for it (uniform data, c5): the pass stops and
// the caller falls back to the radix sort (grid.cu / radix.cu).
#include <algorithm>

#include "internal.h"

namespace db {

constexpr int GR_THREADS = 256;
constexpr int MAX_PROBE = 128;
constexpr uint32_t RANK_SMALL = 8192;  // <= this many cells: O(m^2) rank kernel, else radix

struct __align__(16) GSlot {
  unsigned long long key;
  uint32_t cnt;
  uint32_t id;
};

__device__ __forceinline__ uint64_t gslot(uint64_t key, uint64_t mask) { return mix64(key) & mask; }

// floor(off / s) for the cell coordinate (s = the cell side): a 32-bit
// multiply-high and a shift when every offset is below 2^31 (m32 = ceil(2^(32+r)
// / s), r = ceil(log2 s) - 1: the product's error off (m32 s - 2^(32+r)) stays
// below 2^(32+r), so the quotient is exact), else a 64-bit multiply-high by
// ceil(2^64 / s); s = 1: the offset itself.
struct CDiv {
  uint64_t m64;
  uint32_t m32, r32;
};
__device__ __forceinline__ uint32_t cdiv(uint32_t off, const CDiv& v) {
  if (v.m32) return __umulhi(off, v.m32) >> v.r32;
  return v.m64 ? (uint32_t)__umul64hi((uint64_t)off, v.m64) : off;
}
static CDiv make_cdiv(const Geo& g) {
  CDiv v{0, 0, 0};
  if (g.s <= 1) return v;
  uint64_t span = 0;  // largest offset x - lo: below (maxc + 1) s
  for (int k = 0; k < g.d; ++k) span = std::max<uint64_t>(span, ((uint64_t)g.maxc[k] + 1) * g.s);
  if (span <= (1ull << 31)) {
    const int r = 63 - __builtin_clzll((unsigned long long)g.s - 1);  // ceil(log2 s) - 1
    v.m32 = (uint32_t)((((unsigned __int128)1 << (32 + r)) + g.s - 1) / g.s);
    v.r32 = (uint32_t)r;
  } else {
    v.m64 = (uint64_t)((((unsigned __int128)1 << 64) + g.s - 1) / g.s);
  }
  return v;
}

template <int DD>
__device__ __forceinline__ uint64_t point_key(const int32_t* __restrict__ pts, uint32_t i, const Geo& g,
                                              const CDiv& dv, int32_t* x) {
  uint64_t key = 0;
#pragma unroll
  for (int k = 0; k < DD; ++k) {
    x[k] = __ldg(pts + (uint64_t)i * DD + k);
    const uint32_t off = (uint32_t)x[k] - (uint32_t)g.lo[k];
    const uint32_t ck = cdiv(off, dv);
    key |= (uint64_t)ck << g.shift[k];
  }
  return key;
}

__global__ void group_init_kernel(GSlot* T, uint64_t cap) {
  const uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (h < cap) reinterpret_cast<uint4*>(T)[h] = make_uint4(0xffffffffu, 0xffffffffu, 0u, 0u);
}

// find-or-insert a key; returns the slot, or ~0 when the probe runs too long
// (too many cells for the table: *overflow is set)
__device__ __forceinline__ uint64_t gslot_insert(GSlot* T, uint64_t mask, uint64_t key, uint32_t* overflow) {
  uint64_t h = gslot(key, mask);
  for (int probe = 0; probe < MAX_PROBE; ++probe) {
    const unsigned long long prev = atomicCAS(&T[h].key, (unsigned long long)EMPTY_KEY, (unsigned long long)key);
    if (prev == EMPTY_KEY || prev == key) return h;
    h = (h + 1) & mask;
  }
  atomicExch(overflow, 1u);
  return ~0ull;
}

// A: count points per key. A warp walks a contiguous chunk of the input, 32
// points per step (coalesced). Clustered data keeps one key for long runs:
// while the whole warp holds the key of the current run, lane 0 only adds to
// a register; the count is flushed with one atomic when the key changes.
// Steps with several keys go through __match_any_sync, one atomic per key.
constexpr uint32_t GR_CHUNK = 256;  // points per warp chunk (several chunks per warp: balance)

template <int DD>
__global__ void __launch_bounds__(GR_THREADS) group_count_kernel(const int32_t* __restrict__ pts, uint32_t n,
                                                                 Geo g, CDiv dv, GSlot* T,
                                                                 uint64_t mask, uint32_t* overflow) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t nchunks = (n + GR_CHUNK - 1) / GR_CHUNK;
  uint64_t run_key = ~0ull, run_slot = ~0ull;  // lane 0's current run
  uint32_t run_cnt = 0;
  auto flush = [&]() {
    if (run_cnt && run_slot != ~0ull) atomicAdd(&T[run_slot].cnt, run_cnt);
    run_cnt = 0;
  };
  for (uint32_t ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch < nchunks; ch += nwarps) {
    uint32_t ov = 0;
    if (lane == 0) ov = *(volatile uint32_t*)overflow;
    if (__shfl_sync(DB_FULL, ov, 0)) return;  // warp-uniform
    const uint32_t c0 = ch * GR_CHUNK, c1 = min(n, c0 + GR_CHUNK);
    for (uint32_t i0 = c0; i0 < c1; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool valid = i < c1;
      int32_t x[DD];
      const uint64_t key = valid ? point_key<DD>(pts, i, g, dv, x) : ~0ull;
      const uint64_t k0 = __shfl_sync(DB_FULL, key, 0);
      const uint32_t vmask = __ballot_sync(DB_FULL, valid);
      if (__all_sync(DB_FULL, !valid || key == k0)) {
        if (lane == 0) {
          if (k0 != run_key) {
            flush();
            run_key = k0;
            run_slot = gslot_insert(T, mask, k0, overflow);
          }
          run_cnt += __popc(vmask);
        }
        continue;
      }
      const uint32_t peers = __match_any_sync(DB_FULL, key);
      if (valid && (peers & lanemask_lt()) == 0) {
        const uint64_t h = gslot_insert(T, mask, key, overflow);
        if (h != ~0ull) atomicAdd(&T[h].cnt, (uint32_t)__popc(peers));
      }
    }
  }
  if (lane == 0) flush();
}

// B1: compact the non-empty slots (slot index list; one atomic per block).
__global__ void __launch_bounds__(GR_THREADS) group_compact_kernel(const GSlot* __restrict__ T, uint64_t cap,
                                                                   uint32_t* __restrict__ list,
                                                                   uint32_t* __restrict__ nlist) {
  __shared__ uint32_t s_base;
  __shared__ uint32_t s_scan[33];
  const uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const bool full = h < cap && T[h].key != EMPTY_KEY;
  uint32_t tot;
  const uint32_t ex = block_exclusive_scan<uint32_t>(full ? 1u : 0u, s_scan, &tot);
  if (threadIdx.x == 0) s_base = tot ? atomicAdd(nlist, tot) : 0;
  __syncthreads();
  if (full) list[s_base + ex] = (uint32_t)h;
}

// B2 (m <= RANK_SMALL): rank of each key among the m distinct keys, by
// counting smaller keys (keys are distinct), tiles of keys in shared memory.
__global__ void __launch_bounds__(GR_THREADS) group_rank_kernel(const GSlot* __restrict__ T,
                                                                const uint32_t* __restrict__ list,
                                                                uint32_t m, uint32_t* __restrict__ rank_slot) {
  __shared__ unsigned long long sk[GR_THREADS];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long mine = t < m ? T[list[t]].key : ~0ull;
  uint32_t r = 0;
  for (uint32_t b = 0; b < m; b += GR_THREADS) {
    sk[threadIdx.x] = b + threadIdx.x < m ? T[list[b + threadIdx.x]].key : ~0ull;
    __syncthreads();
    const uint32_t lim = min((uint32_t)GR_THREADS, m - b);
    for (uint32_t q = 0; q < lim; ++q) r += sk[q] < mine;
    __syncthreads();
  }
  if (t < m) rank_slot[r] = list[t];
}

// B2 (large m): gather the keys for the radix sort of (key, slot).
__global__ void group_keys_kernel(const GSlot* __restrict__ T, const uint32_t* __restrict__ list, uint32_t m,
                                  uint64_t* __restrict__ keys) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) keys[t] = T[list[t]].key;
}

// B3: cells in rank order: counts for the scan, cell_key, slot id = rank.
__global__ void group_cells_kernel(GSlot* T, const uint32_t* __restrict__ rank_slot, uint32_t m,
                                   uint32_t* __restrict__ cnt, uint64_t* __restrict__ cell_key,
                                   uint32_t* __restrict__ cellmin) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  GSlot& s = T[rank_slot[r]];
  cnt[r] = s.cnt;
  cell_key[r] = s.key;
  s.id = r;
  cellmin[r] = 0xffffffffu;
}

// C: scatter points to their cells (padded rows), see the file comment. A
// warp walks a contiguous chunk of the input (as in the count pass): while
// the whole warp stays in the cell of the previous step, its id is reused
// without a table probe and its run minimum is already recorded.
template <int DD, int D>
__global__ void __launch_bounds__(GR_THREADS) group_scatter_kernel(
    const int32_t* __restrict__ pts, uint32_t n, Geo g, CDiv dv, const GSlot* __restrict__ T,
    uint64_t mask, uint32_t* __restrict__ cursor, uint32_t* __restrict__ cellmin, int32_t* __restrict__ Ps,
    uint32_t* __restrict__ idx, uint32_t* __restrict__ cell_of, uint32_t* __restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t nchunks = (n + GR_CHUNK - 1) / GR_CHUNK;
  for (uint32_t ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch < nchunks; ch += nwarps) {
    const uint32_t c0 = ch * GR_CHUNK, c1 = min(n, c0 + GR_CHUNK);
    uint64_t run_key = ~0ull;
    uint32_t run_id = 0xffffffffu;
    for (uint32_t i0 = c0; i0 < c1; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool valid = i < c1;
      int32_t x[DD];
      const uint64_t key = valid ? point_key<DD>(pts, i, g, dv, x) : ~0ull;
      const uint64_t k0 = __shfl_sync(DB_FULL, key, 0);
      const bool uniform = __all_sync(DB_FULL, !valid || key == k0);
      uint32_t id = 0xffffffffu;
      bool new_run = true;
      if (uniform && k0 == run_key) {
        id = run_id;  // same cell as the previous step
        new_run = false;
      } else if (valid) {
        uint64_t h = gslot(key, mask);
        while (true) {
          const uint4 s = __ldg(reinterpret_cast<const uint4*>(T + h));
          if ((((uint64_t)s.y << 32) | s.x) == key) { id = s.w; break; }
          h = (h + 1) & mask;  // present: inserted by the count pass
        }
      }
      if (uniform) {
        run_key = k0;
        run_id = __shfl_sync(DB_FULL, id, 0);
        id = run_id;
      } else {
        run_key = ~0ull;
      }
      const uint32_t peers = uniform ? __ballot_sync(DB_FULL, valid) : __match_any_sync(DB_FULL, id);
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (valid && lane == leader) {
        base = atomicAdd(cursor + id, (uint32_t)__popc(peers));
        // lanes hold increasing i: the leader's is the minimum of its run
        if (new_run) atomicMin(cellmin + id, i);
      }
      base = __shfl_sync(DB_FULL, base, leader);
      if (!valid) continue;
      const uint32_t pos = base + __popc(peers & lanemask_lt());
      int32_t y[D];
#pragma unroll
      for (int k = 0; k < D; ++k) y[k] = k < DD ? x[k] : 0;
      if constexpr (D == 2) {
        reinterpret_cast<int2*>(Ps)[pos] = make_int2(y[0], y[1]);
      } else if constexpr (D == 4) {
        reinterpret_cast<int4*>(Ps)[pos] = make_int4(y[0], y[1], y[2], y[3]);
      } else {
        reinterpret_cast<int4*>(Ps)[2 * pos] = make_int4(y[0], y[1], y[2], y[3]);
        reinterpret_cast<int4*>(Ps)[2 * pos + 1] = make_int4(y[4], y[5], y[6], y[7]);
      }
      idx[pos] = i;
      cell_of[pos] = id;
      if (inv) inv[i] = pos;  // (coalesced: lanes hold consecutive i)
    }
  }
}

template <typename F>
static void by_dim_g(int d, F&& f) {
  using std::integral_constant;
  switch (d) {
    case 1: f(integral_constant<int, 1>(), integral_constant<int, 2>()); break;
    case 2: f(integral_constant<int, 2>(), integral_constant<int, 2>()); break;
    case 3: f(integral_constant<int, 3>(), integral_constant<int, 4>()); break;
    case 4: f(integral_constant<int, 4>(), integral_constant<int, 4>()); break;
    case 5: f(integral_constant<int, 5>(), integral_constant<int, 8>()); break;
    case 6: f(integral_constant<int, 6>(), integral_constant<int, 8>()); break;
    case 7: f(integral_constant<int, 7>(), integral_constant<int, 8>()); break;
    default: f(integral_constant<int, 8>(), integral_constant<int, 8>()); break;
  }
}

bool group_by_hash(Ctx& c, const int32_t* pts, int64_t n, const Geo& g, int sparse_mode, int32_t* Ps,
                   uint32_t* idx, uint32_t* cell_of, uint32_t* cell_start, uint64_t* cell_key,
                   uint32_t** cellmin_out, uint32_t* ncells_out, bool* ordered) {
  uint64_t cap = 1024;
  while (cap < 2ull * (uint64_t)n && cap < (1ull << 20)) cap <<= 1;
  const CDiv dv = make_cdiv(g);
  GSlot* T = c.alloc<GSlot>(cap);
  uint32_t* ctr = c.alloc<uint32_t>(2);  // [0] overflow, [1] distinct keys
  group_init_kernel<<<(unsigned)((cap + 255) / 256), 256, 0, c.st>>>(T, cap);
  c.launched();
  c.zero(ctr, 2 * sizeof(uint32_t));
  const unsigned grid = grid_for(n, GR_THREADS, c.sms * 8);
  by_dim_g(g.d, [&](auto Dd, auto) {
    constexpr int DD = decltype(Dd)::value;
    group_count_kernel<DD><<<grid, GR_THREADS, 0, c.st>>>(pts, (uint32_t)n, g, dv, T, cap - 1, ctr);
  });
  c.launched();
  uint32_t* list = c.alloc<uint32_t>(cap);
  group_compact_kernel<<<(unsigned)((cap + GR_THREADS - 1) / GR_THREADS), GR_THREADS, 0, c.st>>>(T, cap, list,
                                                                                               ctr + 1);
  c.launched();
  uint32_t h2[2];
  const uint32_t* h2_h = c.fetch(ctr, 2);
  c.sync();
  h2[0] = h2_h[0];
  h2[1] = h2_h[1];
  if (h2[0]) return false;  // too many cells for the table: radix path
  const uint32_t m = h2[1];
  // Cell ids in key order are needed by the sparse path's rank directory
  // (sparse_mode: 0 never, 1 if the lattice is sparse, 2 forced) and keep
  // thread-per-cell hash probes coalesced when there are many cells; the
  // CSR path over few cells takes any order (the table's).
  const bool order = (sparse_mode == 2) || (sparse_mode == 1 && (uint64_t)n <= SPARSE_MEAN_PER_CELL * m) ||
                     m > 32768;
  uint32_t* rank_slot = list;
  *ordered = order;
  if (!order) {
    // compaction order
  } else if (m <= RANK_SMALL) {
    rank_slot = c.alloc<uint32_t>(m);
    group_rank_kernel<<<grid_for(m, GR_THREADS, 1 << 30), GR_THREADS, 0, c.st>>>(T, list, m, rank_slot);
    c.launched();
  } else {
    uint64_t* k0 = c.alloc<uint64_t>(m);
    uint64_t* k1 = c.alloc<uint64_t>(m);
    uint32_t* v1 = c.alloc<uint32_t>(m);
    group_keys_kernel<<<grid_for(m, 256, 1 << 30), 256, 0, c.st>>>(T, list, m, k0);
    c.launched();
    uint64_t* ko;
    radix_sort_u64(c, k0, list, k1, v1, m, (int)g.bits, &ko, &rank_slot);
  }
  uint32_t* cnt = c.alloc<uint32_t>(m);
  uint32_t* cellmin = c.alloc<uint32_t>(m);
  group_cells_kernel<<<grid_for(m, 256, 1 << 30), 256, 0, c.st>>>(T, rank_slot, m, cnt, cell_key, cellmin);
  c.launched();
  exclusive_scan_u32_u32(c, cnt, cell_start, m);
  uint32_t* cursor = c.alloc<uint32_t>(m);
  DB_CUDA(cudaMemcpyAsync(cursor, cell_start, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, c.st));
  by_dim_g(g.d, [&](auto Dd, auto Dp) {
    constexpr int DD = decltype(Dd)::value, D = decltype(Dp)::value;
    group_scatter_kernel<DD, D><<<grid, GR_THREADS, 0, c.st>>>(pts, (uint32_t)n, g, dv, T, cap - 1, cursor,
                                                               cellmin, Ps, idx, cell_of, c.inv);
  });
  c.launched();
  *cellmin_out = cellmin;
  *ncells_out = m;
  return true;
}


// ===========================================================================
// Lattice counting sort (d <= 3, sparse lattices such as BASELINE configs[4]):
// when the padded lattice has at most LAT_PER_POINT cells per point, count
// the points of every lattice cell directly (packed 8-bit counters, L2
// resident: 43 MB for c5), derive the rank directory, cell_start and cell_key
// from the counts in linear order (= key order), and scatter each point to
// cell_start[rank] + its slot. Two reads of the points and one scattered
// write replace the key array, four radix passes and the gather. The largest
// cell size falls out of the counts, so Alg 2's global bound (reading 13)
// can declare every point non-core before any point is moved.
// A cell with more than 255 points overflows its counter: the pass reports it
// and the caller falls back to the radix sort.
// ===========================================================================
constexpr int LAT_THREADS = 256;

template <int DD>
__device__ __forceinline__ uint64_t point_lin(const int32_t* __restrict__ pts, uint32_t i, const Geo& g,
                                              const CDiv& dv, const uint64_t* stride, int32_t* x) {
  uint64_t lin = 0;
#pragma unroll
  for (int k = 0; k < DD; ++k) {
    x[k] = __ldg(pts + (uint64_t)i * DD + k);
    const uint32_t off = (uint32_t)x[k] - (uint32_t)g.lo[k];
    const uint32_t ck = cdiv(off, dv);
    lin += (uint64_t)(ck + g.R) * stride[k];
  }
  return lin;
}

struct LatArgs {
  Geo g;
  CDiv dv;             // floor(offset / s)
  uint64_t stride[3];
  uint64_t dims[3];    // padded lattice extent per axis
  uint64_t words;      // 32-cell words
  uint64_t smagic[3];  // ceil(2^64 / stride) (stride 1: 0 -> handled as identity below)
  int small;           // padded lattice volume < 2^32: 32-bit coordinates by multiply-high
};

// pass 1: slot of every point in its lattice cell (8-bit packed counters)
template <int DD>
__global__ void __launch_bounds__(LAT_THREADS) lat_count_kernel(const int32_t* __restrict__ pts, uint32_t n,
                                                                LatArgs L, uint32_t* __restrict__ cnt8,
                                                                uint8_t* __restrict__ slot, uint32_t* overflow) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t x[DD];
  const uint64_t lin = point_lin<DD>(pts, i, L.g, L.dv, L.stride, x);
  const uint32_t sh = ((uint32_t)lin & 3u) * 8u;
  const uint32_t old = (atomicAdd(cnt8 + (lin >> 2), 1u << sh) >> sh) & 255u;
  if (old == 255u) *overflow = 1u;  // the add carried into the next counter
  slot[i] = (uint8_t)old;
}

// pass 2a: per 32-cell word, occupancy bits and point count
__global__ void __launch_bounds__(LAT_THREADS) lat_words_kernel(const uint32_t* __restrict__ cnt8, LatArgs L,
                                                                uint32_t* __restrict__ bm,
                                                                uint32_t* __restrict__ wcells,
                                                                uint32_t* __restrict__ wpts, uint32_t* mx) {
  const uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t m = 0;
  if (w < L.words) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(cnt8) + 2 * w);
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(cnt8) + 2 * w + 1);
    const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t bits = 0, sum = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t c = (v[q] >> (8 * k)) & 255u;
        bits |= (uint32_t)(c != 0) << (4 * q + k);
        sum += c;
        m = max(m, c);
      }
    bm[w] = bits;
    wcells[w] = __popc(bits);
    wpts[w] = sum;
  }
  // largest cell: one atomic per block (same-address atomics serialise)
  __shared__ uint32_t s_m;
  if (threadIdx.x == 0) s_m = 0;
  __syncthreads();
  m = __reduce_max_sync(DB_FULL, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(&s_m, m);
  __syncthreads();
  if (threadIdx.x == 0 && s_m) atomicMax(mx, s_m);
}

// pass 2b, a thread per 4 counters (one u32 of cnt8; 8 threads per 32-cell
// word): the cells of its counters in linear order — cell_start, cell_key,
// and cell_of for their points — at the rank and position given by the
// word's prefixes plus an 8-lane exclusive scan; lane 0 of a word writes its
// directory entry {bits w, bits w+1, cells before w, 0}. (A thread per word
// looping over its cells ran at ~17 active lanes.)
__device__ __forceinline__ uint64_t lat_key(uint64_t lin, const LatArgs& L) {
  uint64_t key = 0;
  if (L.small) {
    uint32_t rem = (uint32_t)lin;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (ax < L.g.d) {
        const uint32_t ca = L.smagic[ax] ? (uint32_t)__umul64hi((uint64_t)rem, L.smagic[ax]) : rem;
        rem -= ca * (uint32_t)L.stride[ax];
        key |= (uint64_t)(ca - L.g.R) << L.g.shift[ax];
      }
    }
  } else {
    uint64_t rem = lin;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (ax < L.g.d) {
        const uint64_t ca = rem / L.stride[ax];
        rem -= ca * L.stride[ax];
        key |= (ca - L.g.R) << L.g.shift[ax];
      }
    }
  }
  return key;
}

__global__ void __launch_bounds__(LAT_THREADS) lat_cells4_kernel(const uint32_t* __restrict__ cnt8, LatArgs L,
                                                                 const uint32_t* __restrict__ bm,
                                                                 const uint32_t* __restrict__ cpre,
                                                                 const uint32_t* __restrict__ ppre,
                                                                 uint32_t* __restrict__ cell_start,
                                                                 uint64_t* __restrict__ cell_key,
                                                                 uint4* __restrict__ dir,
                                                                 uint32_t* __restrict__ cell_of) {
  // the warp's (<= 128) cells, compacted: {offset in the warp's 128 lattice
  // cells | points << 8, rank, first position}
  __shared__ uint3 s_cell[LAT_THREADS / 32][128];
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t w = t >> 3;
  const uint32_t q = (uint32_t)t & 7u;
  const bool valid = w < L.words;
  const uint32_t v = valid ? __ldg(cnt8 + t) : 0u;
  const uint32_t bw = valid ? __ldg(bm + w) : 0u;
  const uint32_t nib = (bw >> (4 * q)) & 15u;
  const uint32_t cx = __popc(nib);
  const uint32_t px = (v & 255u) + ((v >> 8) & 255u) + ((v >> 16) & 255u) + (v >> 24);
  // exclusive scans over the 8 lanes of the word (ranks, positions) and over
  // the warp (compacted slot)
  uint32_t ci = cx, pi = px, mi = cx;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t m2 = __shfl_up_sync(DB_FULL, mi, d);
    if (lane >= (uint32_t)d) mi += m2;
    if (d < 8) {
      const uint32_t c2 = __shfl_up_sync(DB_FULL, ci, d, 8), p2 = __shfl_up_sync(DB_FULL, pi, d, 8);
      if (q >= (uint32_t)d) { ci += c2; pi += p2; }
    }
  }
  const uint32_t M = __shfl_sync(DB_FULL, mi, 31);
  uint3* sc = s_cell[threadIdx.x >> 5];
  if (valid) {
    if (q == 0) dir[w] = make_uint4(bw, w + 1 < L.words ? __ldg(bm + w + 1) : 0u, __ldg(cpre + w), 0u);
    if (nib) {
      uint32_t m = mi - cx, r = __ldg(cpre + w) + ci - cx, p = __ldg(ppre + w) + pi - px;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t c = (v >> (8 * k)) & 255u;
        if (c) {
          sc[m] = make_uint3((lane * 4 + k) | (c << 8), r, p);
          ++m;
          ++r;
          p += c;
        }
      }
    }
  }
  __syncwarp();
  const uint64_t lin0 = 4 * (t - lane);
  for (uint32_t m = lane; m < M; m += 32) {
    const uint3 e = sc[m];
    const uint32_t c = e.x >> 8;
    cell_start[e.y] = e.z;
    cell_key[e.y] = lat_key(lin0 + (e.x & 255u), L);
    for (uint32_t s = 0; s < c; ++s) cell_of[e.z + s] = e.y;
  }
}

// pass 3: the permutation, in two steps so that no write lands far from the
// others of its time. The lattice words are cut into buckets of 2^ws
// consecutive words; a bucket's points take the contiguous positions
// ppre[b 2^ws] .. ppre[(b+1) 2^ws) (key order = linear order), about
// BK_TARGET of them.
//  3a: a block takes BK_ITEMS consecutive points per thread, ranks them by
//      bucket in shared memory, reserves room in each bucket's range with one
//      atomic per (block, bucket) and writes the records {lin - bucket start
//      | slot << 24, x, y, z} and the input index there (runs of ~BK_ITEMS x
//      BK_THREADS / buckets records). No gather: the bucket is lin >> (5+ws).
//  3b: a thread per staged record (read coalesced) finds its cell rank on
//      the directory and its position cell_start[rank] + slot, and writes the
//      point, its input index and the cell id there. A block's records belong
//      to one or two buckets, so its directory words, cell starts and output
//      positions lie in one small window (L1 / L2 merge the writes).
constexpr int BK_THREADS = 512;
constexpr int BK_ITEMS = 8;            // 3a: 4096 points per block
constexpr int BK_MAXB = 4096;          // buckets held by a 3a block's shared histogram
constexpr uint32_t BK_TARGET = 16384;  // points per bucket aimed at
constexpr int BK_MAXWS = 19;           // lin - bucket start < 2^24
constexpr int64_t LAT_MAX_N = 1 << 25;  // (the documented limit of the lattice sort)

constexpr int BK_N = BK_THREADS * BK_ITEMS;  // points per 3a block

// 3a. Shared memory (dynamic): the block's points (bulk copy) and, reusing the
// space once they are in registers, its records ordered by bucket — so the
// write-out is coalesced: consecutive threads write consecutive positions of
// one bucket's run, whole sectors at a time — then hist / gbase [nbk].
template <int DD>
__global__ void __launch_bounds__(BK_THREADS, 2) lat_stage_kernel(const int32_t* __restrict__ pts, uint32_t n,
                                                                  LatArgs L, const uint8_t* __restrict__ slot,
                                                                  const uint32_t* __restrict__ ppre, int ws,
                                                                  uint32_t nbk, uint32_t* __restrict__ bcur,
                                                                  uint4* __restrict__ rec,
                                                                  uint32_t* __restrict__ reci) {
  extern __shared__ __align__(16) uint8_t st_raw[];
  int32_t* s_pts = reinterpret_cast<int32_t*>(st_raw);             // [BK_N * DD], then:
  uint4* srec = reinterpret_cast<uint4*>(st_raw);                  // [BK_N] records by bucket
  uint32_t* sidx = reinterpret_cast<uint32_t*>(st_raw + BK_N * 16); // [BK_N] input index
  uint32_t* spos = sidx + BK_N;                                    // [BK_N] staging position
  uint32_t* hist = spos + BK_N;                                    // [nbk] count, then local base
  uint32_t* gbase = hist + nbk;                                    // [nbk] staging base
  __shared__ uint64_t bar;
  __shared__ uint32_t s_scan[33];
  const uint32_t i0 = blockIdx.x * BK_N;
  // a full chunk at a 16-byte aligned address comes in with one bulk copy
  const bool bulk = i0 + BK_N <= n && (((uintptr_t)(pts + (uint64_t)i0 * DD)) & 15) == 0;
  if (bulk && threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    bulk_load(s_pts, pts + (uint64_t)i0 * DD, BK_N * DD * 4, &bar);
  }
  for (uint32_t b = threadIdx.x; b < nbk; b += BK_THREADS) hist[b] = 0;
  __syncthreads();
  if (bulk) mbar_wait(&bar, 0);
  uint32_t lr[BK_ITEMS], key[BK_ITEMS], bk[BK_ITEMS];
  int32_t x[BK_ITEMS][3];
#pragma unroll
  for (int t = 0; t < BK_ITEMS; ++t) {
    const uint32_t i = i0 + t * BK_THREADS + threadIdx.x;
    bk[t] = 0xffffffffu;
    if (i < n) {
      int32_t xx[DD];
      const int32_t* src = bulk ? s_pts + (uint64_t)(t * BK_THREADS + threadIdx.x) * DD : pts + (uint64_t)i * DD;
      uint64_t lin = 0;
#pragma unroll
      for (int k = 0; k < DD; ++k) {
        xx[k] = src[k];
        const uint32_t off = (uint32_t)xx[k] - (uint32_t)L.g.lo[k];
        const uint32_t ck = cdiv(off, L.dv);
        lin += (uint64_t)(ck + L.g.R) * L.stride[k];
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) x[t][k] = k < DD ? xx[k] : 0;
      bk[t] = (uint32_t)(lin >> (5 + ws));
      key[t] = (uint32_t)(lin - ((uint64_t)bk[t] << (5 + ws))) | ((uint32_t)__ldg(slot + i) << 24);
    }
  }
#pragma unroll
  for (int t = 0; t < BK_ITEMS; ++t)
    if (bk[t] != 0xffffffffu) lr[t] = atomicAdd(hist + bk[t], 1u);
  __syncthreads();  // (the points are in registers from here on)
  // reserve each touched bucket's run (one atomic per block and bucket)
  for (uint32_t b = threadIdx.x; b < nbk; b += BK_THREADS)
    if (hist[b]) gbase[b] = __ldg(ppre + ((uint64_t)b << ws)) + atomicAdd(bcur + b, hist[b]);
  // local bases: exclusive scan of the counts, a run of buckets per thread
  const uint32_t per = (nbk + BK_THREADS - 1) / BK_THREADS, b0 = threadIdx.x * per;
  uint32_t sum = 0;
  for (uint32_t q = 0; q < per; ++q)
    if (b0 + q < nbk) sum += hist[b0 + q];
  uint32_t tot;
  uint32_t ex = block_exclusive_scan<uint32_t>(sum, s_scan, &tot);  // (synchronises: all reads done)
  for (uint32_t q = 0; q < per; ++q)
    if (b0 + q < nbk) {
      const uint32_t v = hist[b0 + q];
      hist[b0 + q] = ex;
      ex += v;
    }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < BK_ITEMS; ++t) {
    if (bk[t] == 0xffffffffu) continue;
    const uint32_t j = hist[bk[t]] + lr[t];
    srec[j] = make_uint4(key[t], (uint32_t)x[t][0], (uint32_t)x[t][1], (uint32_t)x[t][2]);
    sidx[j] = i0 + t * BK_THREADS + threadIdx.x;
    spos[j] = gbase[bk[t]] + lr[t];
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < tot; j += BK_THREADS) {
    const uint32_t o = spos[j];
    rec[o] = srec[j];
    reci[o] = sidx[j];
  }
}

constexpr int PL_THREADS = 512;

// 3b's block -> bucket table: chunk c (records c PL_THREADS ..) starts in the
// bucket b with base(b) <= c PL_THREADS < base(b + 1); a thread per bucket.
__global__ void lat_chunks_kernel(const uint32_t* __restrict__ ppre, int ws, uint64_t words, uint32_t nbk,
                                  uint32_t nchunks, uint32_t* __restrict__ chunk_bucket) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbk) return;
  const uint32_t lo = ppre[min((uint64_t)b << ws, words)];
  const uint32_t hi = b + 1 < nbk ? ppre[min((uint64_t)(b + 1) << ws, words)] : 0xffffffffu;
  for (uint32_t c = (lo + PL_THREADS - 1) / PL_THREADS; c < nchunks && (uint64_t)c * PL_THREADS < hi; ++c)
    chunk_bucket[c] = b;
}

template <int D>
__global__ void __launch_bounds__(PL_THREADS) lat_place_kernel(uint32_t n, const uint4* __restrict__ rec,
                                                               const uint32_t* __restrict__ reci,
                                                               const uint4* __restrict__ dir,
                                                               const uint32_t* __restrict__ cell_start,
                                                               const uint32_t* __restrict__ ppre, int ws,
                                                               uint64_t words, uint32_t nbk,
                                                               const uint32_t* __restrict__ chunk_bucket,
                                                               int32_t* __restrict__ Ps, uint32_t* __restrict__ idx,
                                                               uint32_t* __restrict__ cell_of) {
  const uint32_t t0 = blockIdx.x * PL_THREADS;
  auto base_of = [&](uint32_t b) { return __ldg(ppre + min((uint64_t)b << ws, words)); };
  const uint32_t s_b0 = __ldg(chunk_bucket + blockIdx.x);  // bucket of t0
  const uint32_t t = t0 + threadIdx.x;
  if (t >= n) return;
  const uint4 r = __ldg(rec + t);
  const uint32_t i = __ldg(reci + t);
  uint32_t b = s_b0;
  while (b + 1 < nbk && base_of(b + 1) <= t) ++b;
  const uint64_t lin = ((uint64_t)b << (5 + ws)) + (r.x & 0xffffffu);
  const uint4 e = __ldg(dir + (lin >> 5));
  const uint32_t rank = e.z + __popc(e.x & ((1u << ((uint32_t)lin & 31u)) - 1u));
  const uint32_t pos = __ldg(cell_start + rank) + (r.x >> 24);
  if constexpr (D == 2) reinterpret_cast<int2*>(Ps)[pos] = make_int2((int32_t)r.y, (int32_t)r.z);
  else reinterpret_cast<int4*>(Ps)[pos] = make_int4((int32_t)r.y, (int32_t)r.z, (int32_t)r.w, 0);
  idx[pos] = i;
}

bool lattice_applicable(const Geo& g, int64_t n) {
  if (g.d > 3 || n == 0 || n > LAT_MAX_N) return false;
  unsigned __int128 vol = 1;
  for (int k = 0; k < g.d; ++k) vol *= (unsigned __int128)g.maxc[k] + 1 + 2 * (unsigned __int128)g.R;
  return vol <= (unsigned __int128)LAT_PER_POINT * (unsigned __int128)n + (1u << 20);
}

int lattice_group(Ctx& c, const int32_t* pts, int64_t n, const Geo& g, uint64_t min_pts_bound_cells,
                  int64_t min_pts, int32_t* Ps, uint32_t* idx, uint32_t* cell_of, uint32_t* cell_start,
                  uint64_t* cell_key, const uint4** dir_out, uint32_t* ncells_out) {
  LatArgs L{};
  L.g = g;
  L.dv = make_cdiv(g);
  unsigned __int128 vol = 1;
  for (int k = g.d - 1; k >= 0; --k) {
    L.stride[k] = (uint64_t)vol;
    L.dims[k] = (uint64_t)g.maxc[k] + 1 + 2 * (uint64_t)g.R;
    vol *= L.dims[k];
  }
  L.words = ((uint64_t)vol + 31) / 32 + 1;
  L.small = vol + 64 < ((unsigned __int128)1 << 32);
  for (int k = 0; k < g.d; ++k)
    L.smagic[k] = L.stride[k] > 1 ? (uint64_t)((((unsigned __int128)1 << 64) + L.stride[k] - 1) / L.stride[k])
                                  : 0;
  uint32_t* cnt8 = c.alloc<uint32_t>(8 * L.words);
  uint8_t* slot = c.alloc<uint8_t>(n);
  uint32_t* flags = c.alloc<uint32_t>(2);  // [0] overflow, [1] largest cell
  c.zero(cnt8, sizeof(uint32_t) * 8 * L.words);
  c.zero(flags, 2 * sizeof(uint32_t));
  const unsigned pgrid = grid_for(n, LAT_THREADS, 1 << 30);
  auto by_d = [&](auto f) {
    if (g.d == 1) f(std::integral_constant<int, 1>(), std::integral_constant<int, 2>());
    else if (g.d == 2) f(std::integral_constant<int, 2>(), std::integral_constant<int, 2>());
    else f(std::integral_constant<int, 3>(), std::integral_constant<int, 4>());
  };
  by_d([&](auto Dd, auto) {
    constexpr int DD = decltype(Dd)::value;
    lat_count_kernel<DD><<<pgrid, LAT_THREADS, 0, c.st>>>(pts, (uint32_t)n, L, cnt8, slot, flags);
  });
  c.launched();
  uint32_t* bm = c.alloc<uint32_t>(L.words);
  uint32_t* wcells = c.alloc<uint32_t>(L.words);
  uint32_t* wpts = c.alloc<uint32_t>(L.words);
  const unsigned wgrid = grid_for((int64_t)L.words, LAT_THREADS, 1 << 30);
  lat_words_kernel<<<wgrid, LAT_THREADS, 0, c.st>>>(cnt8, L, bm, wcells, wpts, flags + 1);
  c.launched();
  uint32_t h[2];
  const uint32_t* h_h = c.fetch(flags, 2);
  c.sync();
  h[0] = h_h[0];
  h[1] = h_h[1];
  if (h[0]) return LAT_FALLBACK;
  // Alg 2's count is at most (stencil cells) x (largest cell): below minPts,
  // no point is core and nothing needs to be grouped (reading 13)
  if ((uint64_t)h[1] * min_pts_bound_cells < (uint64_t)min_pts) return LAT_ALL_NOISE;
  uint32_t* cpre = c.alloc<uint32_t>(L.words + 1);
  uint32_t* ppre = c.alloc<uint32_t>(L.words + 1);
  exclusive_scan_u32_u32(c, wcells, cpre, (int64_t)L.words);
  exclusive_scan_u32_u32(c, wpts, ppre, (int64_t)L.words);
  uint4* dir = c.alloc<uint4>(L.words);
  lat_cells4_kernel<<<grid_for((int64_t)L.words * 8, LAT_THREADS, 1 << 30), LAT_THREADS, 0, c.st>>>(
      cnt8, L, bm, cpre, ppre, cell_start, cell_key, dir, cell_of);
  c.launched();
  const uint32_t ncells = c.read(cpre + L.words);
  DB_CUDA(cudaMemcpyAsync(cell_start + ncells, ppre + L.words, sizeof(uint32_t), cudaMemcpyDeviceToDevice, c.st));
  // pass 3: stage by bucket of lattice words, then place
  int ws = 0;
  const double ppw = (double)n / (double)L.words;  // points per word
  while (ws < BK_MAXWS && (((L.words + (1ull << ws) - 1) >> ws) > (uint64_t)BK_MAXB ||
                           ppw * (double)(1ull << ws) < (double)BK_TARGET / 2))
    ++ws;
  const uint32_t nbk = (uint32_t)((L.words + (1ull << ws) - 1) >> ws);
  if (nbk > (uint32_t)BK_MAXB) throw Error(-4, "lattice sort: too many buckets");
  uint32_t* bcur = c.alloc<uint32_t>(nbk);
  uint4* rec = c.alloc<uint4>((size_t)n);
  uint32_t* reci = c.alloc<uint32_t>((size_t)n);
  c.zero(bcur, sizeof(uint32_t) * nbk);
  const unsigned nchunks = (unsigned)((n + PL_THREADS - 1) / PL_THREADS);
  uint32_t* chunk_bucket = c.alloc<uint32_t>(nchunks);
  const unsigned sgrid = (unsigned)((n + BK_THREADS * BK_ITEMS - 1) / (BK_THREADS * BK_ITEMS));
  by_d([&](auto Dd, auto Dp) {
    constexpr int DD = decltype(Dd)::value, D = decltype(Dp)::value;
    const int ssm = BK_N * 24 + 2 * 4 * (int)nbk;
    DB_CUDA(cudaFuncSetAttribute(lat_stage_kernel<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
    lat_stage_kernel<DD><<<sgrid, BK_THREADS, ssm, c.st>>>(pts, (uint32_t)n, L, slot, ppre, ws, nbk, bcur, rec, reci);
    c.launched();
    lat_chunks_kernel<<<(nbk + 255) / 256, 256, 0, c.st>>>(ppre, ws, L.words, nbk, nchunks, chunk_bucket);
    c.launched();
    lat_place_kernel<D><<<nchunks, PL_THREADS, 0, c.st>>>((uint32_t)n, rec, reci, dir, cell_start, ppre, ws,
                                                          L.words, nbk, chunk_bucket, Ps, idx, cell_of);
    c.launched();
  });
  *dir_out = dir;
  *ncells_out = ncells;
  return LAT_OK;
}

}  // namespace db
