// scan.cu — device-wide exclusive prefix sum (Table 1 "prefix sum",
// P:L303-310), as one single-pass chained scan with decoupled look-back:
// each 2048-item tile reduces, publishes its aggregate, looks back for its
// exclusive prefix and writes its outputs — 1 read + 1 write per item.
#include "internal.h"

namespace db {

constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 16;  // consecutive items per thread: 4 x 16-byte loads
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

// mask (optional): items with mask[i] >= 0 count as 0 (their in[i] is not read)
// Thread t of a tile owns items [16t, 16t + 16): vector loads and stores
// straight from registers (a warp's 4 loads / 8 stores of 16 B cover whole
// sectors), the tile total is published as the aggregate before the look-back.
// zero_if (optional, device): when *zero_if == 0 every input is known to be 0
// (e.g. no border point at all): the outputs are written as zeros without
// reading the input or looking back — the caller need not read the flag on
// the host first.
template <typename TOut>
__global__ void __launch_bounds__(SC_THREADS) scan_kernel(const uint32_t* __restrict__ in,
                                                          const int32_t* __restrict__ mask,
                                                          TOut* __restrict__ out, int64_t n,
                                                          uint64_t* status, uint32_t* tile_ctr,
                                                          const unsigned long long* zero_if) {
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_scan[33];
  __shared__ uint64_t s_pref;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t j0 = tile * SC_TILE + (int64_t)threadIdx.x * SC_ITEMS;
  if (zero_if && *zero_if == 0) {
    // the tile's outputs as 16-byte stores, consecutive threads on
    // consecutive 16 bytes (each warp store covers 512 contiguous bytes)
    const int64_t t0 = tile * SC_TILE;
    constexpr int PER16 = 16 / sizeof(TOut);
    if (t0 + SC_TILE <= n && (reinterpret_cast<uintptr_t>(out + t0) & 15) == 0) {
      uint4* o4 = reinterpret_cast<uint4*>(out + t0);
#pragma unroll
      for (int q = 0; q < SC_TILE / PER16 / SC_THREADS; ++q) o4[q * SC_THREADS + threadIdx.x] = make_uint4(0, 0, 0, 0);
    } else {
      for (int64_t j = t0 + threadIdx.x; j < min(n, t0 + SC_TILE); j += SC_THREADS) out[j] = 0;
    }
    if (t0 + SC_TILE >= n && threadIdx.x == 0) out[n] = 0;
    return;
  }
  uint32_t v[SC_ITEMS];
  const bool full = j0 + SC_ITEMS <= n && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
                    (!mask || (reinterpret_cast<uintptr_t>(mask) & 15) == 0);
  if (full) {
#pragma unroll
    for (int q = 0; q < SC_ITEMS / 4; ++q) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(in + j0) + q);
      v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
      if (mask) {
        const int4 m = __ldg(reinterpret_cast<const int4*>(mask + j0) + q);
        if (m.x >= 0) v[4 * q] = 0;
        if (m.y >= 0) v[4 * q + 1] = 0;
        if (m.z >= 0) v[4 * q + 2] = 0;
        if (m.w >= 0) v[4 * q + 3] = 0;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) {
      const int64_t j = j0 + i;
      v[i] = (j < n && !(mask && mask[j] >= 0)) ? in[j] : 0u;
    }
  }
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) sum += v[i];
  uint64_t tot;
  const uint64_t ex = block_exclusive_scan<uint64_t>(sum, s_scan, &tot);
  if (threadIdx.x < 32) {
    const uint64_t pref = lb_exclusive_warp(status, tile, 1, tot);
    if (threadIdx.x == 0) s_pref = pref;
  }
  __syncthreads();
  uint64_t run = s_pref + ex;
  TOut o[SC_ITEMS];
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) { o[i] = (TOut)run; run += v[i]; }
  constexpr int PER16 = 16 / sizeof(TOut);  // outputs per 16-byte store
  const int64_t t0 = tile * SC_TILE;
  const bool tfull = t0 + SC_TILE <= n && (reinterpret_cast<uintptr_t>(out + t0) & 15) == 0;
  if (tfull) {
    // through shared memory, a warp's store instruction then covers 512
    // contiguous bytes (straight from registers, lanes were 64-128 B apart)
    __shared__ uint4 s_out[SC_THREADS / 32][32 * SC_ITEMS / PER16];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < SC_ITEMS / PER16; ++q) {
      uint4 x;
      if constexpr (PER16 == 4) {
        x = make_uint4((uint32_t)o[4 * q], (uint32_t)o[4 * q + 1], (uint32_t)o[4 * q + 2], (uint32_t)o[4 * q + 3]);
      } else {
        const uint64_t a = (uint64_t)o[2 * q], b = (uint64_t)o[2 * q + 1];
        x = make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32));
      }
      s_out[w][lane * (SC_ITEMS / PER16) + q] = x;
    }
    __syncwarp();
    uint4* o4 = reinterpret_cast<uint4*>(out + t0) + (int64_t)w * (32 * SC_ITEMS / PER16);
#pragma unroll
    for (int q = 0; q < SC_ITEMS / PER16; ++q) o4[q * 32 + lane] = s_out[w][q * 32 + lane];
  } else {
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i)
      if (j0 + i < n) out[j0 + i] = o[i];
  }
  if (j0 < n && j0 + SC_ITEMS >= n) out[n] = (TOut)run;  // total (the thread holding item n-1)
}

template <typename TOut>
static void scan_impl(Ctx& c, const uint32_t* in, TOut* out, int64_t n, const int32_t* mask = nullptr,
                      const unsigned long long* zero_if = nullptr) {
  if (n == 0) {
    c.zero(out, sizeof(TOut));
    return;
  }
  const int64_t tiles = (n + SC_TILE - 1) / SC_TILE;
  uint64_t* status = c.alloc<uint64_t>(tiles + 1);  // [tiles]: the tile counter
  uint32_t* ctr = reinterpret_cast<uint32_t*>(status + tiles);
  c.zero(status, sizeof(uint64_t) * (tiles + 1));
  scan_kernel<TOut><<<(unsigned)tiles, SC_THREADS, 0, c.st>>>(in, mask, out, n, status, ctr, zero_if);
  c.launched();
}

void exclusive_scan_u32_u64(Ctx& c, const uint32_t* in, uint64_t* out, int64_t n) {
  scan_impl<uint64_t>(c, in, out, n);
}
void exclusive_scan_u32_i64(Ctx& c, const uint32_t* in, int64_t* out, int64_t n,
                            const unsigned long long* zero_if) {
  scan_impl<int64_t>(c, in, out, n, nullptr, zero_if);
}
void exclusive_scan_u32_i64_masked(Ctx& c, const uint32_t* in, const int32_t* mask, int64_t* out, int64_t n,
                                   const unsigned long long* zero_if) {
  scan_impl<int64_t>(c, in, out, n, mask, zero_if);
}

}  // namespace db

namespace db {
void exclusive_scan_u32_u32(Ctx& c, const uint32_t* in, uint32_t* out, int64_t n) {
  scan_impl<uint32_t>(c, in, out, n);
}
}  // namespace db
