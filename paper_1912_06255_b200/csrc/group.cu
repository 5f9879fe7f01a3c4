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

template <int DD>
__device__ __forceinline__ uint64_t point_key(const int32_t* __restrict__ pts, uint32_t i, const Geo& g,
                                              uint64_t magic, int32_t* x) {
  uint64_t key = 0;
#pragma unroll
  for (int k = 0; k < DD; ++k) {
    x[k] = __ldg(pts + (uint64_t)i * DD + k);
    const uint32_t off = (uint32_t)x[k] - (uint32_t)g.lo[k];
    const uint32_t ck = magic ? (uint32_t)__umul64hi((uint64_t)off, magic) : off;
    key |= (uint64_t)ck << g.shift[k];
  }
  return key;
}

__global__ void group_init_kernel(GSlot* T, uint64_t cap) {
  const uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (h < cap) reinterpret_cast<uint4*>(T)[h] = make_uint4(0xffffffffu, 0xffffffffu, 0u, 0u);
}

// A: count points per key. Every thread runs the same number of iterations so
// the warp-wide match is always full.
template <int DD>
__global__ void __launch_bounds__(GR_THREADS) group_count_kernel(const int32_t* __restrict__ pts, uint32_t n,
                                                                 Geo g, uint64_t magic, GSlot* T,
                                                                 uint64_t mask, uint32_t* overflow) {
  const int lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t iters = (n + stride - 1) / stride;
  for (uint32_t it = 0; it < iters; ++it) {
    if ((it & 7) == 0) {
      uint32_t ov = 0;
      if (lane == 0) ov = *(volatile uint32_t*)overflow;
      if (__shfl_sync(DB_FULL, ov, 0)) return;  // warp-uniform
    }
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + it * stride;
    const bool valid = i < n;
    int32_t x[DD];
    const uint64_t key = valid ? point_key<DD>(pts, i, g, magic, x) : ~0ull;
    const uint32_t peers = __match_any_sync(DB_FULL, key);
    if (!valid || (peers & lanemask_lt()) != 0) continue;  // one leader per distinct key
    uint64_t h = gslot(key, mask);
    int probe = 0;
    while (true) {
      const unsigned long long prev = atomicCAS(&T[h].key, (unsigned long long)EMPTY_KEY,
                                                (unsigned long long)key);
      if (prev == EMPTY_KEY || prev == key) {
        atomicAdd(&T[h].cnt, (uint32_t)__popc(peers));
        break;
      }
      if (++probe == MAX_PROBE) { atomicExch(overflow, 1u); break; }
      h = (h + 1) & mask;
    }
  }
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

// C: scatter points to their cells (padded rows), see the file comment.
template <int DD, int D>
__global__ void __launch_bounds__(GR_THREADS) group_scatter_kernel(
    const int32_t* __restrict__ pts, uint32_t n, Geo g, uint64_t magic, const GSlot* __restrict__ T,
    uint64_t mask, uint32_t* __restrict__ cursor, uint32_t* __restrict__ cellmin, int32_t* __restrict__ Ps,
    uint32_t* __restrict__ idx, uint32_t* __restrict__ cell_of) {
  const int lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t iters = (n + stride - 1) / stride;
  for (uint32_t it = 0; it < iters; ++it) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + it * stride;
    const bool valid = i < n;
    int32_t x[DD];
    uint32_t id = 0xffffffffu;
    if (valid) {
      const uint64_t key = point_key<DD>(pts, i, g, magic, x);
      uint64_t h = gslot(key, mask);
      while (true) {
        const uint4 s = __ldg(reinterpret_cast<const uint4*>(T + h));
        if ((((uint64_t)s.y << 32) | s.x) == key) { id = s.w; break; }
        h = (h + 1) & mask;  // present: inserted by the count pass
      }
    }
    const uint32_t peers = __match_any_sync(DB_FULL, id);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (valid && lane == leader) {
      base = atomicAdd(cursor + id, (uint32_t)__popc(peers));
      atomicMin(cellmin + id, i);  // lanes hold increasing i: the leader's is the run's minimum
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

bool group_by_hash(Ctx& c, const int32_t* pts, int64_t n, const Geo& g, int32_t* Ps, uint32_t* idx,
                   uint32_t* cell_of, uint32_t* cell_start, uint64_t* cell_key, uint32_t** cellmin_out,
                   uint32_t* ncells_out) {
  uint64_t cap = 1024;
  while (cap < 2ull * (uint64_t)n && cap < (1ull << 20)) cap <<= 1;
  const uint64_t magic = g.s > 1 ? (uint64_t)((((unsigned __int128)1 << 64) + g.s - 1) / g.s) : 0;
  GSlot* T = c.alloc<GSlot>(cap);
  uint32_t* ctr = c.alloc<uint32_t>(2);  // [0] overflow, [1] distinct keys
  group_init_kernel<<<(unsigned)((cap + 255) / 256), 256, 0, c.st>>>(T, cap);
  c.launched();
  c.zero(ctr, 2 * sizeof(uint32_t));
  const unsigned grid = grid_for(n, GR_THREADS, c.sms * 8);
  by_dim_g(g.d, [&](auto Dd, auto) {
    constexpr int DD = decltype(Dd)::value;
    group_count_kernel<DD><<<grid, GR_THREADS, 0, c.st>>>(pts, (uint32_t)n, g, magic, T, cap - 1, ctr);
  });
  c.launched();
  uint32_t* list = c.alloc<uint32_t>(cap);
  group_compact_kernel<<<(unsigned)((cap + GR_THREADS - 1) / GR_THREADS), GR_THREADS, 0, c.st>>>(T, cap, list,
                                                                                               ctr + 1);
  c.launched();
  uint32_t h2[2];
  DB_CUDA(cudaMemcpyAsync(h2, ctr, sizeof(h2), cudaMemcpyDeviceToHost, c.st));
  DB_CUDA(cudaStreamSynchronize(c.st));
  if (h2[0]) return false;  // too many cells for the table: radix path
  const uint32_t m = h2[1];
  uint32_t* rank_slot = c.alloc<uint32_t>(m);
  if (m <= RANK_SMALL) {
    group_rank_kernel<<<grid_for(m, GR_THREADS, 1 << 30), GR_THREADS, 0, c.st>>>(T, list, m, rank_slot);
    c.launched();
  } else {
    uint64_t* k0 = c.alloc<uint64_t>(m);
    uint64_t* k1 = c.alloc<uint64_t>(m);
    uint32_t* v1 = c.alloc<uint32_t>(m);
    group_keys_kernel<<<grid_for(m, 256, 1 << 30), 256, 0, c.st>>>(T, list, m, k0);
    c.launched();
    uint64_t* ko;
    uint32_t* vo;
    radix_sort_u64(c, k0, list, k1, v1, m, (int)g.bits, &ko, &vo);
    DB_CUDA(cudaMemcpyAsync(rank_slot, vo, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, c.st));
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
    group_scatter_kernel<DD, D><<<grid, GR_THREADS, 0, c.st>>>(pts, (uint32_t)n, g, magic, T, cap - 1, cursor,
                                                               cellmin, Ps, idx, cell_of);
  });
  c.launched();
  *cellmin_out = cellmin;
  *ncells_out = m;
  return true;
}

}  // namespace db
