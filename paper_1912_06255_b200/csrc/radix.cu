// radix.cu — LSD radix sort of (key, u32 value) pairs, SURVEY §8(a) row a2.
//
// PAPER.md groups points by cell with a semisort and uses a
// parallel integer sort for the quadtree; BASELINE
// north_star asks for a radix sort of the cell keys. Onesweep structure:
// every digit histogram is built once up front (fused into the keys kernel,
// grid.cu), then one scatter pass per 8-bit digit. A pass over a tile of
// THREADS*ITEMS keys:
//   1. claim the tile id from an atomic counter (tiles start in id order, so
//      the look-back below never waits on a tile that has not started);
//   2. load keys and values, warp-striped (item i of lane l = i*32 + l);
//   3. rank each key within its warp in item order with __match_any_sync
//      (stable), counting per warp and digit in 16-bit shared counters;
//   4. per digit: exclusive offsets across warps and the tile count, published
//      at once as this tile's aggregate (decoupled look-back, Merrill & Garland);
//   5. block scan of the digit counts (tile-local offsets), then a windowed
//      look-back (4 predecessors per step) for the global offset of each digit;
//   6. reorder the tile in shared memory by (digit, rank) and write it out in
//      digit runs, so stores coalesce.
// Stable, so the cells' points keep increasing input index (used by a9).
#include <algorithm>

#include "internal.h"

namespace db {

__device__ __forceinline__ uint64_t lb_window_exclusive(uint64_t* status, int64_t tile, int64_t stride) {
  uint64_t excl = 0;
  int64_t t = tile - 1;
  while (t >= 0) {
    uint64_t s[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) s[q] = (t - q >= 0) ? lb_read(status + (t - q) * stride) : LB_INC;
    int used = 0;
    bool done = false;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (done || used < q) break;
      const uint64_t v = s[q];
      if ((v & ~LB_VAL) == 0) break;  // not published yet: re-read from here
      excl += v & LB_VAL;
      ++used;
      if (v & LB_INC) done = true;
    }
    if (done) break;
    t -= used;
  }
  return excl;
}

template <typename K, int THREADS, int ITEMS>
struct RadixCfg {
  static constexpr int WARPS = THREADS / 32;
  static constexpr int TILE = THREADS * ITEMS;
  static constexpr size_t SMEM = (size_t)TILE * (sizeof(K) + 4) + (size_t)WARPS * 256 * 2 + 256 * 4 * 2;
};

template <typename K, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) radix_pass_kernel(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, uint32_t n, int shift, const uint32_t* __restrict__ bucket_base,
    uint64_t* status, uint32_t* tile_ctr) {
  using C = RadixCfg<K, THREADS, ITEMS>;
  constexpr int WARPS = C::WARPS, TILE = C::TILE;
  static_assert(THREADS >= 256, "one thread per digit");
  static_assert(32 * ITEMS <= 65535, "16-bit warp counters");
  extern __shared__ __align__(16) uint8_t smem_raw[];
  K* skey = reinterpret_cast<K*>(smem_raw);
  uint32_t* sval = reinterpret_cast<uint32_t*>(skey + TILE);
  uint16_t* whist = reinterpret_cast<uint16_t*>(sval + TILE);            // [WARPS][256]
  uint32_t* tloc = reinterpret_cast<uint32_t*>(whist + WARPS * 256);     // tile-local digit offset
  int32_t* gofs = reinterpret_cast<int32_t*>(tloc + 256);               // global - local offset
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_scan[33];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = tid; i < WARPS * 128; i += THREADS) reinterpret_cast<uint32_t*>(whist)[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t wbase = tile * TILE + w * (32 * ITEMS);

  K key[ITEMS];
  uint32_t val[ITEMS];
  uint16_t rank[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t pos = wbase + i * 32 + lane;
    key[i] = pos < n ? kin[pos] : K(0);
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t pos = wbase + i * 32 + lane;
    val[i] = pos < n ? vin[pos] : 0u;
  }
  uint16_t* wh = whist + w * 256;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const bool valid = wbase + i * 32 + lane < n;
    const uint32_t dg = valid ? (uint32_t)(key[i] >> shift) & 255u : 256u;
    const uint32_t peers = __match_any_sync(DB_FULL, dg);
    const uint32_t before = __popc(peers & lt);
    const uint32_t cnt = valid ? wh[dg] : 0u;
    __syncwarp();
    if (valid && before == 0) wh[dg] = (uint16_t)(cnt + __popc(peers));
    __syncwarp();
    rank[i] = (uint16_t)(cnt + before);
  }
  __syncthreads();
  // digit tid: exclusive offsets across warps; publish the tile aggregate early
  uint32_t run = 0;
  if (tid < 256) {
#pragma unroll
    for (int ww = 0; ww < WARPS; ++ww) {
      const uint32_t c = whist[ww * 256 + tid];
      whist[ww * 256 + tid] = (uint16_t)run;
      run += c;
    }
    lb_publish(status + (size_t)tile * 256 + tid, (tile == 0 ? LB_INC : LB_AGG) | run);
  }
  uint32_t tot;
  const uint32_t local = block_exclusive_scan(tid < 256 ? run : 0u, s_scan, &tot);
  if (tid < 256) {
    const uint64_t excl = tile == 0 ? 0 : lb_window_exclusive(status + tid, tile, 256);
    if (tile != 0) lb_publish(status + (size_t)tile * 256 + tid, LB_INC | (excl + run));
    tloc[tid] = local;
    gofs[tid] = (int32_t)(bucket_base[tid] + (uint32_t)excl) - (int32_t)local;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (wbase + i * 32 + lane < n) {
      const uint32_t dg = (uint32_t)(key[i] >> shift) & 255u;
      const uint32_t lp = tloc[dg] + whist[w * 256 + dg] + rank[i];
      skey[lp] = key[i];
      sval[lp] = val[i];
    }
  }
  __syncthreads();
  const uint32_t tstart = tile * TILE;
  const uint32_t cnt = min((uint32_t)TILE, n - tstart);
  for (uint32_t j = tid; j < cnt; j += THREADS) {
    const K k = skey[j];
    const uint32_t dg = (uint32_t)(k >> shift) & 255u;
    const uint32_t o = (uint32_t)(gofs[dg] + (int32_t)j);
    kout[o] = k;
    vout[o] = sval[j];
  }
}

// bucket_base[p][b] = exclusive prefix of hist[p][*] (one block per pass)
__global__ void bucket_base_kernel(const uint32_t* hist, uint32_t* base) {
  __shared__ uint32_t sm[33];
  uint32_t tot;
  const uint32_t v = hist[blockIdx.x * 256 + threadIdx.x];
  base[blockIdx.x * 256 + threadIdx.x] = block_exclusive_scan(v, sm, &tot);
}

template <typename K, int THREADS, int ITEMS>
static void sort_passes(Ctx& c, K* k0, uint32_t* v0, K* k1, uint32_t* v1, uint32_t n, int passes,
                        const uint32_t* hist, K** ko, uint32_t** vo) {
  using Cfg = RadixCfg<K, THREADS, ITEMS>;
  if (passes == 0 || n == 0) { *ko = k0; *vo = v0; return; }
  uint32_t* base = c.alloc<uint32_t>((size_t)passes * 256);
  bucket_base_kernel<<<passes, 256, 0, c.st>>>(hist, base);
  c.launched();
  const uint32_t tiles = (n + Cfg::TILE - 1) / Cfg::TILE;
  uint64_t* status = c.alloc<uint64_t>((size_t)passes * tiles * 256);
  uint32_t* ctr = c.alloc<uint32_t>(passes);
  c.zero(status, sizeof(uint64_t) * (size_t)passes * tiles * 256);
  c.zero(ctr, sizeof(uint32_t) * passes);
  DB_CUDA(cudaFuncSetAttribute(radix_pass_kernel<K, THREADS, ITEMS>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
  K* ka = k0; uint32_t* va = v0; K* kb = k1; uint32_t* vb = v1;
  for (int p = 0; p < passes; ++p) {
    radix_pass_kernel<K, THREADS, ITEMS><<<tiles, THREADS, Cfg::SMEM, c.st>>>(
        ka, va, kb, vb, n, 8 * p, base + 256 * p, status + (size_t)p * tiles * 256, ctr + p);
    c.launched();
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  *ko = ka; *vo = va;
}

void radix_sort_pairs_u32(Ctx& c, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint32_t n,
                          int passes, const uint32_t* hist, uint32_t** ko, uint32_t** vo) {
  sort_passes<uint32_t, 512, 12>(c, k0, v0, k1, v1, n, passes, hist, ko, vo);
}

void radix_sort_pairs_u64(Ctx& c, uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, uint32_t n,
                          int passes, const uint32_t* hist, uint64_t** ko, uint32_t** vo) {
  sort_passes<uint64_t, 512, 8>(c, k0, v0, k1, v1, n, passes, hist, ko, vo);
}

}  // namespace db
