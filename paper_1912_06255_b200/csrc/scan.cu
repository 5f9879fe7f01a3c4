// scan.cu — device-wide exclusive prefix sum (Table 1 "prefix sum",
// P:L303-310), as one single-pass chained scan with decoupled look-back:
// each 2048-item tile reduces, publishes its aggregate, looks back for its
// exclusive prefix and writes its outputs — 1 read + 1 write per item.
#include "internal.h"

namespace db {

constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 8;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

// mask (optional): items with mask[i] >= 0 count as 0 (their in[i] is not read)
template <typename TOut>
__global__ void __launch_bounds__(SC_THREADS) scan_kernel(const uint32_t* __restrict__ in,
                                                          const int32_t* __restrict__ mask,
                                                          TOut* __restrict__ out, int64_t n,
                                                          uint64_t* status, uint32_t* tile_ctr) {
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_scan[33];
  __shared__ uint64_t s_pref;
  __shared__ uint32_t s_in[SC_TILE];
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * SC_TILE;
  // coalesced load through shared memory, then blocked per-thread sums
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    int64_t j = base + i * SC_THREADS + threadIdx.x;
    s_in[i * SC_THREADS + threadIdx.x] = (j < n && !(mask && mask[j] >= 0)) ? in[j] : 0u;
  }
  __syncthreads();
  uint32_t v[SC_ITEMS];
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) { v[i] = s_in[threadIdx.x * SC_ITEMS + i]; sum += v[i]; }
  uint64_t tot;
  uint64_t ex = block_exclusive_scan<uint64_t>(sum, s_scan, &tot);
  if (threadIdx.x == 0) s_pref = lb_exclusive(status, tile, 1, tot);
  __syncthreads();
  uint64_t run = s_pref + ex;
  // write back through shared memory for coalescing (two halves for 64-bit outputs)
  TOut* s_out = reinterpret_cast<TOut*>(s_in);  // reuse: SC_TILE*4 bytes
  constexpr int PER = (int)(sizeof(uint32_t) * SC_TILE / sizeof(TOut));  // outputs per round
  TOut o[SC_ITEMS];
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) { o[i] = (TOut)run; run += v[i]; }
  __syncthreads();
  for (int r = 0; r < SC_TILE / PER; ++r) {
    const int lo = r * PER;
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) {
      int li = threadIdx.x * SC_ITEMS + i;
      if (li >= lo && li < lo + PER) s_out[li - lo] = o[i];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < PER; t += SC_THREADS) {
      int64_t j = base + lo + t;
      if (j < n) out[j] = s_out[t];
    }
    __syncthreads();
  }
  if ((n - 1) / SC_TILE == tile && threadIdx.x == SC_THREADS - 1) out[n] = (TOut)run;  // total
}

template <typename TOut>
static void scan_impl(Ctx& c, const uint32_t* in, TOut* out, int64_t n, const int32_t* mask = nullptr) {
  if (n == 0) {
    c.zero(out, sizeof(TOut));
    return;
  }
  const int64_t tiles = (n + SC_TILE - 1) / SC_TILE;
  uint64_t* status = c.alloc<uint64_t>(tiles);
  uint32_t* ctr = c.alloc<uint32_t>(1);
  c.zero(status, sizeof(uint64_t) * tiles);
  c.zero(ctr, sizeof(uint32_t));
  scan_kernel<TOut><<<(unsigned)tiles, SC_THREADS, 0, c.st>>>(in, mask, out, n, status, ctr);
  c.launched();
}

void exclusive_scan_u32_u64(Ctx& c, const uint32_t* in, uint64_t* out, int64_t n) {
  scan_impl<uint64_t>(c, in, out, n);
}
void exclusive_scan_u32_i64(Ctx& c, const uint32_t* in, int64_t* out, int64_t n) {
  scan_impl<int64_t>(c, in, out, n);
}
void exclusive_scan_u32_i64_masked(Ctx& c, const uint32_t* in, const int32_t* mask, int64_t* out, int64_t n) {
  scan_impl<int64_t>(c, in, out, n, mask);
}

}  // namespace db

namespace db {
void exclusive_scan_u32_u32(Ctx& c, const uint32_t* in, uint32_t* out, int64_t n) {
  scan_impl<uint32_t>(c, in, out, n);
}
}  // namespace db
