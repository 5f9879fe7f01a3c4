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
                                                                 Geo g, uint64_t magic, GSlot* T,
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
      const uint64_t key = valid ? point_key<DD>(pts, i, g, magic, x) : ~0ull;
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
    const int32_t* __restrict__ pts, uint32_t n, Geo g, uint64_t magic, const GSlot* __restrict__ T,
    uint64_t mask, uint32_t* __restrict__ cursor, uint32_t* __restrict__ cellmin, int32_t* __restrict__ Ps,
    uint32_t* __restrict__ idx, uint32_t* __restrict__ cell_of) {
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
      const uint64_t key = valid ? point_key<DD>(pts, i, g, magic, x) : ~0ull;
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
    group_scatter_kernel<DD, D><<<grid, GR_THREADS, 0, c.st>>>(pts, (uint32_t)n, g, magic, T, cap - 1, cursor,
                                                               cellmin, Ps, idx, cell_of);
  });
  c.launched();
  *cellmin_out = cellmin;
  *ncells_out = m;
  return true;
}


// ===========================================================================
// Lattice counting sort (d <= 3, sparse lattices such as BASELINE configs[4]):
// when the padded lattice has at most LAT_PER_POINT cells per point, the
// points are counted per lattice cell, in BUCKETS of LB_CELLS consecutive
// lattice cells (linear order = key order), so that every count lives in
// shared memory:
//  1. hist:  per point its bucket (lin >> LB_WB); per-block shared histogram,
//            one global atomic per (block, bucket);
//  2. scan of the bucket counts: bucket b's points take the contiguous
//            positions bbase[b] .. bbase[b+1] of the output;
//  3. stage: a block takes BK_N points (one TMA bulk copy), ranks them by
//            bucket in shared memory, reserves a run in each bucket's range
//            with one atomic per (block, bucket) and writes the records
//            {lin - bucket start, x, y, z} and input indices there coalesced;
//  4. sort:  a CTA per bucket counts its records per cell with 8-bit packed
//            shared-memory counters (the atomic's old value is the point's
//            slot in its cell), derives, per 32-cell directory word, the
//            occupancy bits and the point and cell prefixes (one block scan),
//            takes the bucket's first cell id from a decoupled look-back over
//            the buckets, writes the directory words (the sparse path's rank
//            directory), cell_start and cell_key of its cells, then places
//            every record at bbase[b] + (points of the cells before) + slot,
//            with its input index and cell id (cell_of) — writes confined to
//            the bucket's contiguous output range.
// The largest cell size falls out of the counts (Alg 2's global bound,
// reading 13). A cell with more than 255 points overflows its counter: the
// pass reports it and the caller falls back to the radix sort.
// ===========================================================================
constexpr int LAT_THREADS = 256;

template <int DD>
__device__ __forceinline__ uint64_t point_lin(const int32_t* __restrict__ pts, uint32_t i, const Geo& g,
                                              uint64_t magic, const uint64_t* stride, int32_t* x) {
  uint64_t lin = 0;
#pragma unroll
  for (int k = 0; k < DD; ++k) {
    x[k] = __ldg(pts + (uint64_t)i * DD + k);
    const uint32_t off = (uint32_t)x[k] - (uint32_t)g.lo[k];
    const uint32_t ck = magic ? (uint32_t)__umul64hi((uint64_t)off, magic) : off;
    lin += (uint64_t)(ck + g.R) * stride[k];
  }
  return lin;
}

struct LatArgs {
  Geo g;
  uint64_t magic;
  uint64_t stride[3];
  uint64_t dims[3];    // padded lattice extent per axis
  uint64_t words;      // 32-cell words
  uint64_t smagic[3];  // ceil(2^64 / stride) (stride 1: 0 -> handled as identity below)
  int small;           // padded lattice volume < 2^32: 32-bit coordinates by multiply-high
};

constexpr int LB_WB = 16;                    // lattice cells per sort bucket: 2^16
constexpr uint32_t LB_CELLS = 1u << LB_WB;
constexpr int LB_GROUPS = LB_CELLS / 32;     // directory words per bucket
constexpr int LB_THREADS = 512;
constexpr int LB_GPT = LB_GROUPS / LB_THREADS;
constexpr int BK_THREADS = 512;
constexpr int BK_ITEMS = 8;                  // stage: 4096 points per block
constexpr int BK_N = BK_THREADS * BK_ITEMS;
constexpr int BK_MAXB = 8448;                // buckets (lattice <= 8 n + 2^20 cells, n <= 2^25)
constexpr int64_t LAT_MAX_N = 1 << 25;       // (the documented limit of the lattice sort)

// 1. bucket histogram: HIST_ITEMS points per thread, shared counts, one global
// atomic per (block, touched bucket)
constexpr int HIST_ITEMS = 16;

template <int DD>
__global__ void __launch_bounds__(LAT_THREADS) lat_hist_kernel(const int32_t* __restrict__ pts, uint32_t n, LatArgs L,
                                                               uint32_t nbk, uint32_t* __restrict__ bcnt) {
  extern __shared__ uint32_t hist[];
  for (uint32_t b = threadIdx.x; b < nbk; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const uint32_t i0 = blockIdx.x * (LAT_THREADS * HIST_ITEMS);
#pragma unroll 4
  for (int t = 0; t < HIST_ITEMS; ++t) {
    const uint32_t i = i0 + t * LAT_THREADS + threadIdx.x;
    if (i < n) {
      int32_t x[DD];
      const uint64_t lin = point_lin<DD>(pts, i, L.g, L.magic, L.stride, x);
      atomicAdd(hist + (uint32_t)(lin >> LB_WB), 1u);
    }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nbk; b += blockDim.x)
    if (hist[b]) atomicAdd(bcnt + b, hist[b]);
}

// 3. stage by bucket. Shared memory (dynamic): the block's points (bulk copy)
// and, reusing the space once they are in registers, its records ordered by
// bucket — so the write-out is coalesced: consecutive threads write
// consecutive positions of one bucket's run, whole sectors at a time — then
// hist / gbase [nbk].
template <int DD>
__global__ void __launch_bounds__(BK_THREADS, 2) lat_stage_kernel(const int32_t* __restrict__ pts, uint32_t n,
                                                               LatArgs L, const uint32_t* __restrict__ bbase,
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
        const uint32_t ck = L.magic ? (uint32_t)__umul64hi((uint64_t)off, L.magic) : off;
        lin += (uint64_t)(ck + L.g.R) * L.stride[k];
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) x[t][k] = k < DD ? xx[k] : 0;
      bk[t] = (uint32_t)(lin >> LB_WB);
      key[t] = (uint32_t)lin & (LB_CELLS - 1u);
    }
  }
#pragma unroll
  for (int t = 0; t < BK_ITEMS; ++t)
    if (bk[t] != 0xffffffffu) lr[t] = atomicAdd(hist + bk[t], 1u);
  __syncthreads();  // (the points are in registers from here on)
  // reserve each touched bucket's run (one atomic per block and bucket)
  for (uint32_t b = threadIdx.x; b < nbk; b += BK_THREADS)
    if (hist[b]) gbase[b] = __ldg(bbase + b) + atomicAdd(bcur + b, hist[b]);
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

// packed key of lattice cell `lin` (padded linear index)
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

// byte-sum of the counters of cells [w*4, w*4 + k) of a packed counter word
__device__ __forceinline__ uint32_t bytes_below(uint32_t v, uint32_t k) {
  return __dp4a(k >= 4 ? v : (v & ((1u << (8 * k)) - 1u)), 0x01010101u, 0u);
}

// 4. a CTA per bucket (see the section comment). flags: [0] counter overflow,
// [1] largest cell, [2] number of cells (written by the last bucket).
template <int D>
__global__ void __launch_bounds__(LB_THREADS, 2) lat_sort_kernel(
    const uint4* __restrict__ rec, const uint32_t* __restrict__ reci, uint8_t* __restrict__ slot,
    const uint32_t* __restrict__ bbase, uint32_t nbk, LatArgs L, uint64_t* __restrict__ lbst,
    int32_t* __restrict__ Ps, uint32_t* __restrict__ idx, uint32_t* __restrict__ cell_of,
    uint32_t* __restrict__ cell_start, uint64_t* __restrict__ cell_key, uint4* __restrict__ dir,
    uint32_t* __restrict__ flags) {
  extern __shared__ __align__(16) uint32_t lb_sm[];
  uint32_t* cnt = lb_sm;                  // [LB_CELLS / 4] 8-bit counters, packed
  uint32_t* gpts = cnt + LB_CELLS / 4;    // [LB_GROUPS] points of the bucket before the word
  uint32_t* gcel = gpts + LB_GROUPS;      // [LB_GROUPS] cells of the bucket before the word
  uint32_t* gbit = gcel + LB_GROUPS;      // [LB_GROUPS] occupancy bits of the word
  __shared__ unsigned long long s_scan[33];
  __shared__ unsigned long long s_cbase;
  const uint32_t b = blockIdx.x;
  const uint32_t r0 = __ldg(bbase + b), r1 = __ldg(bbase + b + 1);
  for (uint32_t i = threadIdx.x; i < LB_CELLS / 4; i += LB_THREADS) cnt[i] = 0;
  __syncthreads();
  // counts; the old counter value is the record's slot in its cell
  bool ovf = false;
  for (uint32_t t = r0 + threadIdx.x; t < r1; t += LB_THREADS) {
    const uint32_t rl = __ldg(&rec[t].x);
    const uint32_t sh = (rl & 3u) * 8u;
    const uint32_t s = (atomicAdd(cnt + (rl >> 2), 1u << sh) >> sh) & 255u;
    ovf |= s == 255u;
    slot[t] = (uint8_t)s;
  }
  // a counter passed 255 and carried into its neighbour: the caller falls
  // back to the radix sort; this bucket publishes no cell and writes nothing
  const bool bad = __syncthreads_or(ovf);
  if (bad && threadIdx.x == 0) atomicExch(flags, 1u);
  // per directory word (32 cells = 8 counter words): bits, points, largest cell
  uint32_t gb[LB_GPT], gp[LB_GPT];
  uint32_t sp = 0, sc = 0, mx = 0;
#pragma unroll
  for (int q = 0; q < LB_GPT; ++q) {
    const uint32_t g = threadIdx.x * LB_GPT + q;
    uint32_t bits = 0, pts = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t v = cnt[g * 8 + w];
      pts += __dp4a(v, 0x01010101u, 0u);
      const uint32_t nz = __vcmpne4(v, 0u);  // 0xff per non-empty cell
      bits |= ((nz & 1u) | ((nz >> 7) & 2u) | ((nz >> 14) & 4u) | ((nz >> 21) & 8u)) << (4 * w);
      const uint32_t m2 = __vmaxu4(v, v >> 16);
      mx = max(mx, max(m2 & 255u, (m2 >> 8) & 255u));
    }
    gb[q] = bits;
    gp[q] = pts;
    sp += pts;
    sc += __popc(bits);
  }
  unsigned long long tot;
  unsigned long long ex = block_exclusive_scan<unsigned long long>(
      (unsigned long long)sp | ((unsigned long long)sc << 32), s_scan, &tot);
  if (bad) tot = 0;
#pragma unroll
  for (int q = 0; q < LB_GPT; ++q) {
    const uint32_t g = threadIdx.x * LB_GPT + q;
    gpts[g] = (uint32_t)ex;
    gcel[g] = (uint32_t)(ex >> 32);
    gbit[g] = gb[q];
    ex += (unsigned long long)gp[q] | ((unsigned long long)__popc(gb[q]) << 32);
  }
  // the bucket's first cell id: look-back over the buckets (warp 0)
  if (threadIdx.x < 32) {
    const uint64_t cb = lb_exclusive_warp(lbst, b, 1, tot >> 32);
    if (threadIdx.x == 0) {
      s_cbase = cb;
      if (b + 1 == nbk) {
        flags[2] = (uint32_t)(cb + (tot >> 32));
        cell_start[cb + (tot >> 32)] = r1;  // = n
      }
    }
  }
  mx = __reduce_max_sync(DB_FULL, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(flags + 1, mx);
  __syncthreads();
  if (bad) return;
  const uint32_t cbase = (uint32_t)s_cbase;
  // directory words, cell_start, cell_key: a thread per word
#pragma unroll
  for (int q = 0; q < LB_GPT; ++q) {
    const uint32_t g = threadIdx.x * LB_GPT + q;
    const uint64_t w = (uint64_t)b * LB_GROUPS + g;
    if (w >= L.words) continue;
    const uint32_t bits = gbit[g];
    // {bits of word w, bits of word w + 1, cells before w, 0}; the next word
    // of the bucket's last word belongs to the next bucket, which writes that
    // field (disjoint bytes: no ordering needed between the two buckets)
    if (g + 1 < (uint32_t)LB_GROUPS) {
      dir[w] = make_uint4(bits, gbit[g + 1], cbase + gcel[g], 0u);
    } else {
      uint32_t* e = reinterpret_cast<uint32_t*>(dir + w);
      e[0] = bits;
      if (b + 1 == nbk) e[1] = 0u;
      e[2] = cbase + gcel[g];
      e[3] = 0u;
    }
    if (g == 0 && w > 0) reinterpret_cast<uint32_t*>(dir + w - 1)[1] = bits;
    uint32_t r = cbase + gcel[g], p = r0 + gpts[g];
    for (uint32_t bb = bits; bb; bb &= bb - 1) {
      const int k = __ffs(bb) - 1;
      cell_start[r] = p;
      cell_key[r] = lat_key(w * 32 + (uint64_t)k, L);
      p += (cnt[g * 8 + (k >> 2)] >> (8 * (k & 3))) & 255u;
      ++r;
    }
  }
  // place: bbase[b] + points of the cells before + slot
  for (uint32_t t = r0 + threadIdx.x; t < r1; t += LB_THREADS) {
    const uint4 v = __ldg(rec + t);
    const uint32_t rl = v.x, g = rl >> 5, k = rl & 31u;
    uint32_t pre = gpts[g];
    const uint32_t cw = rl >> 2;
    for (uint32_t w = g * 8; w < cw; ++w) pre += __dp4a(cnt[w], 0x01010101u, 0u);
    pre += bytes_below(cnt[cw], rl & 3u);
    const uint32_t pos = r0 + pre + __ldg(slot + t);
    const uint32_t rank = cbase + gcel[g] + __popc(gbit[g] & ((1u << k) - 1u));
    if constexpr (D == 2) reinterpret_cast<int2*>(Ps)[pos] = make_int2((int32_t)v.y, (int32_t)v.z);
    else reinterpret_cast<int4*>(Ps)[pos] = make_int4((int32_t)v.y, (int32_t)v.z, (int32_t)v.w, 0);
    idx[pos] = __ldg(reci + t);
    cell_of[pos] = rank;
  }
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
  L.magic = g.s > 1 ? (uint64_t)((((unsigned __int128)1 << 64) + g.s - 1) / g.s) : 0;
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
  // buckets of LB_CELLS lattice cells cover the directory's words
  const uint32_t nbk = (uint32_t)((L.words * 32 + LB_CELLS - 1) / LB_CELLS);
  if (nbk > (uint32_t)BK_MAXB) throw Error(-4, "lattice sort: too many buckets");
  auto by_d = [&](auto f) {
    if (g.d == 1) f(std::integral_constant<int, 1>(), std::integral_constant<int, 2>());
    else if (g.d == 2) f(std::integral_constant<int, 2>(), std::integral_constant<int, 2>());
    else f(std::integral_constant<int, 3>(), std::integral_constant<int, 4>());
  };
  uint32_t* bcnt = c.alloc<uint32_t>(nbk);
  uint32_t* bbase = c.alloc<uint32_t>(nbk + 1);
  uint32_t* bcur = c.alloc<uint32_t>(nbk);
  uint64_t* lbst = c.alloc<uint64_t>(nbk);
  uint32_t* flags = c.alloc<uint32_t>(4);  // [0] overflow, [1] largest cell, [2] cells
  c.zero(bcnt, sizeof(uint32_t) * nbk);
  c.zero(bcur, sizeof(uint32_t) * nbk);
  c.zero(lbst, sizeof(uint64_t) * nbk);
  c.zero(flags, 4 * sizeof(uint32_t));
  uint4* rec = c.alloc<uint4>((size_t)n);
  uint32_t* reci = c.alloc<uint32_t>((size_t)n);
  uint8_t* slot = c.alloc<uint8_t>((size_t)n);
  uint4* dir = c.alloc<uint4>(L.words);
  by_d([&](auto Dd, auto Dp) {
    constexpr int DD = decltype(Dd)::value, D = decltype(Dp)::value;
    const unsigned hgrid = (unsigned)((n + LAT_THREADS * HIST_ITEMS - 1) / (LAT_THREADS * HIST_ITEMS));
    const int hsm = 4 * (int)nbk;
    DB_CUDA(cudaFuncSetAttribute(lat_hist_kernel<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm));
    lat_hist_kernel<DD><<<hgrid, LAT_THREADS, hsm, c.st>>>(pts, (uint32_t)n, L, nbk, bcnt);
    c.launched();
    exclusive_scan_u32_u32(c, bcnt, bbase, nbk);
    const unsigned sgrid = (unsigned)((n + BK_N - 1) / BK_N);
    const int ssm = BK_N * 24 + 2 * 4 * (int)nbk;
    DB_CUDA(cudaFuncSetAttribute(lat_stage_kernel<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
    lat_stage_kernel<DD><<<sgrid, BK_THREADS, ssm, c.st>>>(pts, (uint32_t)n, L, bbase, nbk, bcur, rec, reci);
    c.launched();
    const int lsm = (int)(LB_CELLS + 3 * 4 * LB_GROUPS);
    DB_CUDA(cudaFuncSetAttribute(lat_sort_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, lsm));
    lat_sort_kernel<D><<<nbk, LB_THREADS, lsm, c.st>>>(rec, reci, slot, bbase, nbk, L, lbst, Ps, idx, cell_of,
                                                       cell_start, cell_key, dir, flags);
    c.launched();
  });
  const uint32_t* h = c.fetch(flags, 4);
  c.sync();
  if (h[0]) return LAT_FALLBACK;
  // Alg 2's count is at most (stencil cells) x (largest cell): below minPts,
  // no point is core (reading 13)
  if ((uint64_t)h[1] * min_pts_bound_cells < (uint64_t)min_pts) return LAT_ALL_NOISE;
  *dir_out = dir;
  *ncells_out = h[2];
  return LAT_OK;
}

}  // namespace db
