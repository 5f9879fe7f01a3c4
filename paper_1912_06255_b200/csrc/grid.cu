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

// ------------------------------------------------------------------ a1: bbox
__global__ void bbox_init_kernel(int32_t* lohi) {
  int t = threadIdx.x;
  if (t < 8) lohi[t] = INT32_MAX;
  else if (t < 16) lohi[t] = INT32_MIN;
}

// Per-axis min/max over the row-major int32 array, read as a flat stream of
// n*d elements (element e belongs to axis e mod d).
__global__ void __launch_bounds__(256) bbox_kernel(const int32_t* __restrict__ pts, int64_t n_el,
                                                   int d, int32_t* lohi) {
  int32_t mn[8], mx[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { mn[k] = INT32_MAX; mx[k] = INT32_MIN; }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool aligned = (reinterpret_cast<uintptr_t>(pts) & 15) == 0;
  const int64_t nvec = aligned ? n_el / 4 : 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += stride) {
    int4 q = __ldg(reinterpret_cast<const int4*>(pts) + v);
    int a = (int)((4 * v) % d);
    int32_t e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k == a) { mn[k] = min(mn[k], e[j]); mx[k] = max(mx[k], e[j]); }
      a = (a + 1 == d) ? 0 : a + 1;
    }
  }
  for (int64_t e = 4 * nvec + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_el; e += stride) {
    int a = (int)(e % d);
    int32_t x = pts[e];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k == a) { mn[k] = min(mn[k], x); mx[k] = max(mx[k], x); }
  }
  __shared__ int32_t smn[8][8], smx[8][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn[k] = min(mn[k], __shfl_xor_sync(DB_FULL, mn[k], o));
      mx[k] = max(mx[k], __shfl_xor_sync(DB_FULL, mx[k], o));
    }
    if (lane == 0) { smn[w][k] = mn[k]; smx[w][k] = mx[k]; }
  }
  __syncthreads();
  if (threadIdx.x < 8 && threadIdx.x < d) {
    int k = threadIdx.x;
    int32_t a = INT32_MAX, b = INT32_MIN;
    for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) { a = min(a, smn[ww][k]); b = max(b, smx[ww][k]); }
    atomicMin(lohi + k, a);
    atomicMax(lohi + 8 + k, b);
  }
}

void bbox(Ctx& c, const int32_t* pts, int64_t n, int d, int32_t* lohi) {
  bbox_init_kernel<<<1, 32, 0, c.st>>>(lohi);
  c.launched();
  int64_t nel = n * d;
  bbox_kernel<<<grid_for(nel / 4 + 1, 256, c.sms * 8), 256, 0, c.st>>>(pts, nel, d, lohi);
  c.launched();
}

// ------------------------------------------------------- a1: keys + histogram
// key = sum_k ((x_k - lo_k) div s) << shift_k; idx = input row. Also builds the
// 256-bin histogram of every 8-bit digit the sort will use (onesweep's single
// upfront histogram), aggregated per warp with match_any before the shared
// atomics to survive skewed digits.
template <typename K>
__global__ void __launch_bounds__(256) keys_kernel(const int32_t* __restrict__ pts, uint32_t n,
                                                   Geo g, int passes, K* __restrict__ keys,
                                                   uint32_t* __restrict__ idx,
                                                   uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[8 * 256];
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t start = blockIdx.x * blockDim.x + threadIdx.x;
  // every thread runs the same number of iterations so the warp-level match is full
  const uint32_t iters = (n + stride - 1) / stride;
  for (uint32_t it = 0; it < iters; ++it) {
    uint32_t i = start + it * stride;
    bool valid = i < n;
    K key = 0;
    if (valid) {
      const int32_t* p = pts + (int64_t)i * g.d;
      for (int k = 0; k < g.d; ++k) {
        uint32_t off = (uint32_t)((int64_t)p[k] - (int64_t)g.lo[k]);  // < 2^32
        uint32_t ck = off / g.s;
        key |= (K)ck << g.shift[k];
      }
      keys[i] = key;
      idx[i] = i;
    }
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

// bucket_base[p][b] = exclusive prefix of hist[p][*] (one block per pass)
__global__ void bucket_base_kernel(const uint32_t* hist, uint32_t* base) {
  __shared__ uint32_t sm[33];
  uint32_t tot;
  uint32_t v = hist[blockIdx.x * 256 + threadIdx.x];
  base[blockIdx.x * 256 + threadIdx.x] = block_exclusive_scan(v, sm, &tot);
}

// -------------------------------------------------- a2: onesweep scatter pass
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

template <typename K>
constexpr size_t rs_smem() {
  return (size_t)RS_TILE * (sizeof(K) + 4) + (size_t)RS_WARPS * 256 * 4 + 256 * 4 * 2;
}

// One stable LSD pass on digit (key >> shift) & 255. Tiles are claimed in
// launch order through an atomic counter so the look-back never waits on a
// tile that has not started. Within a tile, items are warp-striped
// (item i of lane l = i*32 + l), ranked per warp in item order with
// __match_any_sync (stable), combined across warps per digit, offset across
// tiles by decoupled look-back, locally reordered through shared memory and
// written out in digit runs.
template <typename K>
__global__ void __launch_bounds__(RS_THREADS) radix_pass_kernel(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, uint32_t n, int shift, const uint32_t* __restrict__ bucket_base,
    uint64_t* status, uint32_t* tile_ctr) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  K* skey = reinterpret_cast<K*>(smem_raw);
  uint32_t* sval = reinterpret_cast<uint32_t*>(skey + RS_TILE);
  uint32_t* whist = sval + RS_TILE;            // [RS_WARPS][256]
  uint32_t* tloc = whist + RS_WARPS * 256;     // tile-local exclusive offset per digit
  int32_t* gofs = reinterpret_cast<int32_t*>(tloc + 256);  // global - local offset per digit
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_scan[33];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int i = tid; i < RS_WARPS * 256; i += RS_THREADS) whist[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t wbase = tile * RS_TILE + w * (32 * RS_ITEMS);

  K key[RS_ITEMS];
  uint32_t val[RS_ITEMS];
  uint32_t rank[RS_ITEMS];
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i) {
    uint32_t pos = wbase + i * 32 + lane;
    if (pos < n) { key[i] = kin[pos]; val[i] = vin[pos]; }
    else { key[i] = 0; val[i] = 0; }
  }
  uint32_t* wh = whist + w * 256;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i) {
    uint32_t pos = wbase + i * 32 + lane;
    bool valid = pos < n;
    uint32_t dg = valid ? (uint32_t)(key[i] >> shift) & 255u : 256u;
    uint32_t peers = __match_any_sync(DB_FULL, dg);
    uint32_t before = __popc(peers & lt);
    uint32_t cnt = valid ? wh[dg] : 0u;
    __syncwarp();
    if (valid && before == 0) wh[dg] = cnt + __popc(peers);
    __syncwarp();
    rank[i] = cnt + before;
  }
  __syncthreads();
  // digit tid: exclusive offsets across warps, tile count
  uint32_t run = 0;
#pragma unroll
  for (int ww = 0; ww < RS_WARPS; ++ww) {
    uint32_t c = whist[ww * 256 + tid];
    whist[ww * 256 + tid] = run;
    run += c;
  }
  uint32_t tot;
  uint32_t local = block_exclusive_scan(run, s_scan, &tot);
  uint64_t excl = lb_exclusive(status + tid, tile, 256, run);
  tloc[tid] = local;
  gofs[tid] = (int32_t)(bucket_base[tid] + (uint32_t)excl) - (int32_t)local;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RS_ITEMS; ++i) {
    uint32_t pos = wbase + i * 32 + lane;
    if (pos < n) {
      uint32_t dg = (uint32_t)(key[i] >> shift) & 255u;
      uint32_t lp = tloc[dg] + whist[w * 256 + dg] + rank[i];
      skey[lp] = key[i];
      sval[lp] = val[i];
    }
  }
  __syncthreads();
  const uint32_t tstart = tile * RS_TILE;
  const uint32_t cnt = min((uint32_t)RS_TILE, n - tstart);
  for (uint32_t j = tid; j < cnt; j += RS_THREADS) {
    K k = skey[j];
    uint32_t dg = (uint32_t)(k >> shift) & 255u;
    uint32_t o = (uint32_t)(gofs[dg] + (int32_t)j);
    kout[o] = k;
    vout[o] = sval[j];
  }
}

template <typename K>
static void radix_sort_impl(Ctx& c, K* k0, uint32_t* v0, K* k1, uint32_t* v1, uint32_t n,
                            int passes, const uint32_t* hist, K** ko, uint32_t** vo) {
  if (passes == 0) { *ko = k0; *vo = v0; return; }
  uint32_t* base = c.alloc<uint32_t>((size_t)passes * 256);
  bucket_base_kernel<<<passes, 256, 0, c.st>>>(hist, base);
  c.launched();
  const uint32_t tiles = (n + RS_TILE - 1) / RS_TILE;
  uint64_t* status = c.alloc<uint64_t>((size_t)passes * tiles * 256);
  uint32_t* ctr = c.alloc<uint32_t>(passes);
  c.zero(status, sizeof(uint64_t) * (size_t)passes * tiles * 256);
  c.zero(ctr, sizeof(uint32_t) * passes);
  const size_t smem = rs_smem<K>();
  DB_CUDA(cudaFuncSetAttribute(radix_pass_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  K* ka = k0; uint32_t* va = v0; K* kb = k1; uint32_t* vb = v1;
  for (int p = 0; p < passes; ++p) {
    radix_pass_kernel<K><<<tiles, RS_THREADS, smem, c.st>>>(
        ka, va, kb, vb, n, 8 * p, base + 256 * p, status + (size_t)p * tiles * 256, ctr + p);
    c.launched();
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  *ko = ka; *vo = va;
}

void cell_keys_and_sort(Ctx& c, const int32_t* pts, int64_t n, const Geo& g, bool key64,
                        void** sorted_keys, uint32_t** sorted_idx, int* passes_out) {
  const int passes = (int)((g.bits + 7) / 8);
  *passes_out = passes;
  uint32_t* hist = c.alloc<uint32_t>(8 * 256);
  c.zero(hist, sizeof(uint32_t) * 8 * 256);
  uint32_t* v0 = c.alloc<uint32_t>(n);
  uint32_t* v1 = c.alloc<uint32_t>(n);
  const unsigned grid = grid_for(n, 256, c.sms * 8);
  if (key64) {
    uint64_t* k0 = c.alloc<uint64_t>(n);
    uint64_t* k1 = c.alloc<uint64_t>(n);
    keys_kernel<uint64_t><<<grid, 256, 0, c.st>>>(pts, (uint32_t)n, g, passes, k0, v0, hist);
    c.launched();
    uint64_t* ko; uint32_t* vo;
    radix_sort_impl<uint64_t>(c, k0, v0, k1, v1, (uint32_t)n, passes, hist, &ko, &vo);
    *sorted_keys = ko; *sorted_idx = vo;
  } else {
    uint32_t* k0 = c.alloc<uint32_t>(n);
    uint32_t* k1 = c.alloc<uint32_t>(n);
    keys_kernel<uint32_t><<<grid, 256, 0, c.st>>>(pts, (uint32_t)n, g, passes, k0, v0, hist);
    c.launched();
    uint32_t* ko; uint32_t* vo;
    radix_sort_impl<uint32_t>(c, k0, v0, k1, v1, (uint32_t)n, passes, hist, &ko, &vo);
    *sorted_keys = ko; *sorted_idx = vo;
  }
}

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
  radix_sort_impl<uint64_t>(c, keys, vals, keys_alt, vals_alt, (uint32_t)n, passes, hist,
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
__global__ void __launch_bounds__(SG_THREADS) segment_kernel(
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
