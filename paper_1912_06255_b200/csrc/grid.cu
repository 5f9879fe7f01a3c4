// grid.cu — Grid construction, SURVEY §8(a) rows a1-a4.
//
// PAPER.md §4.1 "Grid Computation": points go to cells of side
// eps/sqrt(d); the paper groups (cellID, pointID) pairs with a semisort
// and stores non-empty cells in a hash table keyed by the cell
// (P:L486-489). Here (B200 design): integer side s, packed
// cell key, an LSD radix sort of (key, index) with one onesweep scatter pass per
// 8-bit digit (block ranking by warp match + decoupled look-back), one
// segmentation pass that also gathers the points into a padded sorted array,
// and an open-addressing hash table of the unique cell keys.
#include <algorithm>

#include "internal.h"

namespace db {

// histogram of 64-bit keys for the generic sort
__global__ void __launch_bounds__(256) hist_u64_kernel(const uint64_t* __restrict__ keys, uint32_t n,
                                                       int passes, uint32_t* hist) {
  __shared__ uint32_t sh[8 * 256];
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t iters = (n + stride - 1) / stride;
  for (uint32_t it = 0; it < iters; ++it) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + it * stride;
    bool valid = i < n;
    uint64_t key = valid ? keys[i] : 0;
    for (int p = 0; p < passes; ++p) {
      uint32_t dg = valid ? (uint32_t)(key >> (8 * p)) & 255u : 256u;
      uint32_t peers = __match_any_sync(DB_FULL, dg);
      if (valid && (peers & lanemask_lt()) == 0) atomicAdd(sh + p * 256 + dg, __popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, sh[i]);
}

void radix_sort_u64(Ctx& c, uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                    int64_t n, int bits, uint64_t** out_keys, uint32_t** out_vals) {
  const int passes = (bits + 7) / 8;
  uint32_t* hist = c.alloc<uint32_t>(8 * 256);
  c.zero(hist, sizeof(uint32_t) * 8 * 256);
  if (passes > 0) {
    hist_u64_kernel<<<grid_for(n, 256, c.sms * 8), 256, 0, c.st>>>(keys, (uint32_t)n, passes, hist);
    c.launched();
  }
  radix_sort_pairs_u64(c, keys, vals, keys_alt, vals_alt, (uint32_t)n, passes, hist,
                            out_keys, out_vals);
}

// --------------------------------------------- a3: segmentation + point gather
constexpr int SG_THREADS = 256;
constexpr int SG_ITEMS = 8;
constexpr int SG_TILE = SG_THREADS * SG_ITEMS;

// head[j] = key[j] != key[j-1]; cell id = inclusive count of heads - 1 (one
// single-pass chained scan over tiles). Writes cell_of, cell_start, cell_key
// and gathers Ps[j] = pts[idx[j]] padded to D int32 (padding = 0).
template <typename K, int D>
__global__ void __launch_bounds__(SG_THREADS, 2) segment_kernel(
    const K* __restrict__ keys, const uint32_t* __restrict__ idx, const int32_t* __restrict__ pts,
    int d, uint32_t n, int32_t* __restrict__ Ps, uint32_t* __restrict__ cell_of,
    uint32_t* __restrict__ cell_start, uint64_t* __restrict__ cell_key, uint64_t* status,
    uint32_t* tile_ctr, uint32_t* ncells) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_scan[33];
  __shared__ uint32_t s_pref;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t j0 = tile * SG_TILE + threadIdx.x * SG_ITEMS;
  K prev = 0;
  if (j0 > 0 && j0 < n) prev = keys[j0 - 1];
  K kk[SG_ITEMS];
  uint32_t heads = 0, cnt = 0;
#pragma unroll
  for (int i = 0; i < SG_ITEMS; ++i) {
    uint32_t j = j0 + i;
    kk[i] = j < n ? keys[j] : 0;
    bool h = j < n && (j == 0 || kk[i] != prev);
    heads |= (uint32_t)h << i;
    cnt += h;
    prev = kk[i];
  }
  uint32_t tot;
  uint32_t ex = block_exclusive_scan(cnt, s_scan, &tot);
  if (threadIdx.x == 0) s_pref = (uint32_t)lb_exclusive(status, tile, 1, tot);
  __syncthreads();
  uint32_t c = s_pref + ex;  // heads before this thread's first item
#pragma unroll
  for (int i = 0; i < SG_ITEMS; ++i) {
    uint32_t j = j0 + i;
    if (j >= n) break;
    if ((heads >> i) & 1u) {
      cell_start[c] = j;
      cell_key[c] = (uint64_t)kk[i];
      ++c;
    }
    cell_of[j] = c - 1;
    uint32_t src = idx[j];
    int32_t x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = k < d ? pts[(int64_t)src * d + k] : 0;
    if constexpr (D == 2) {
      reinterpret_cast<int2*>(Ps)[j] = make_int2(x[0], x[1]);
    } else if constexpr (D == 4) {
      reinterpret_cast<int4*>(Ps)[j] = make_int4(x[0], x[1], x[2], x[3]);
    } else {
      reinterpret_cast<int4*>(Ps)[2 * j] = make_int4(x[0], x[1], x[2], x[3]);
      reinterpret_cast<int4*>(Ps)[2 * j + 1] = make_int4(x[4], x[5], x[6], x[7]);
    }
    if (j == n - 1) {
      cell_start[c] = n;
      *ncells = c;
    }
  }
}

uint32_t segment_and_gather(Ctx& c, const void* sorted_keys, bool key64, const uint32_t* sorted_idx,
                            const int32_t* pts, int64_t n, const Geo& g, int32_t* Ps,
                            uint32_t* cell_of, uint32_t* cell_start, uint64_t* cell_key) {
  const uint32_t tiles = (uint32_t)((n + SG_TILE - 1) / SG_TILE);
  uint64_t* status = c.alloc<uint64_t>(tiles);
  uint32_t* ctr = c.alloc<uint32_t>(2);
  c.zero(status, sizeof(uint64_t) * tiles);
  c.zero(ctr, sizeof(uint32_t) * 2);
  auto go = [&](auto Dc) {
    constexpr int D = decltype(Dc)::value;
    if (key64)
      segment_kernel<uint64_t, D><<<tiles, SG_THREADS, 0, c.st>>>(
          (const uint64_t*)sorted_keys, sorted_idx, pts, g.d, (uint32_t)n, Ps, cell_of, cell_start,
          cell_key, status, ctr, ctr + 1);
    else
      segment_kernel<uint32_t, D><<<tiles, SG_THREADS, 0, c.st>>>(
          (const uint32_t*)sorted_keys, sorted_idx, pts, g.d, (uint32_t)n, Ps, cell_of, cell_start,
          cell_key, status, ctr, ctr + 1);
  };
  if (g.D == 2) go(std::integral_constant<int, 2>());
  else if (g.D == 4) go(std::integral_constant<int, 4>());
  else go(std::integral_constant<int, 8>());
  c.launched();
  return c.read(ctr + 1);
}

// -------------------------------------------------------------- a4: hash table
__global__ void hash_insert_kernel(const uint64_t* __restrict__ cell_key, uint32_t ncells, Slot* T,
                                   uint64_t mask) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncells) return;
  uint64_t key = cell_key[i];
  uint64_t h = slot_of(key, mask);
  while (true) {
    unsigned long long prev = atomicCAS(&T[h].key, (unsigned long long)EMPTY_KEY,
                                        (unsigned long long)key);
    if (prev == EMPTY_KEY) { T[h].val = i; return; }
    h = (h + 1) & mask;  // keys are unique after segmentation: never equal
  }
}

uint64_t build_hash(Ctx& c, const uint64_t* cell_key, uint32_t ncells, Slot** table) {
  uint64_t cap = 1024;
  while (cap < 2ull * ncells) cap <<= 1;
  Slot* T = c.alloc<Slot>(cap);
  DB_CUDA(cudaMemsetAsync(T, 0xff, sizeof(Slot) * cap, c.st));
  hash_insert_kernel<<<grid_for(ncells, 256, 1 << 30), 256, 0, c.st>>>(cell_key, ncells, T, cap - 1);
  c.launched();
  *table = T;
  return cap - 1;
}

}  // namespace db
