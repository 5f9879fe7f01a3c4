// keys.cu — grid construction front end: bounding box,
// cell keys and the digit histograms of the radix sort.
//
// points go to cells of side eps/sqrt(d)
// (integer side s here, reading 5) keyed by their cell; the cell
// coordinate is c_k = (x_k - lo_k) div s with lo the per-axis minimum
// (half-open boxes, reading 6), packed with axis 0 most significant.
// Both kernels are streaming passes over the int32 input with the dimension a
// compile-time constant (no per-element modulo); the division by s is an
// exact 64-bit multiply-high by M = ceil(2^64 / s): for x < 2^32 and
// 2 <= s < 2^32, floor(x * M / 2^64) = floor(x / s) because the error
// x (M - 2^64/s) / 2^64 < 2^-32 <= 1/s.
#include "internal.h"

namespace db {

__global__ void bbox_init_kernel(int32_t* lohi) {
  const int t = threadIdx.x;
  if (t < 8) lohi[t] = INT32_MAX;
  else if (t < 16) lohi[t] = INT32_MIN;
  else if (t == 16) lohi[t] = 0;  // sampled cell collisions
}

// Thread per row (grid-stride); a warp reads 32 consecutive rows = 128*DD
// contiguous bytes per step.
template <int DD>
__global__ void __launch_bounds__(256) bbox_kernel(const int32_t* __restrict__ pts, int64_t n,
                                                   int32_t* lohi) {
  int32_t mn[DD], mx[DD];
#pragma unroll
  for (int k = 0; k < DD; ++k) { mn[k] = INT32_MAX; mx[k] = INT32_MIN; }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
#pragma unroll
    for (int k = 0; k < DD; ++k) {
      const int32_t x = __ldg(pts + i * DD + k);
      mn[k] = min(mn[k], x);
      mx[k] = max(mx[k], x);
    }
  }
  __shared__ int32_t smn[8][DD], smx[8][DD];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < DD; ++k) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn[k] = min(mn[k], __shfl_xor_sync(DB_FULL, mn[k], o));
      mx[k] = max(mx[k], __shfl_xor_sync(DB_FULL, mx[k], o));
    }
    if (lane == 0) { smn[w][k] = mn[k]; smx[w][k] = mx[k]; }
  }
  __syncthreads();
  if (threadIdx.x < DD) {
    const int k = threadIdx.x;
    int32_t a = INT32_MAX, b = INT32_MIN;
    for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) { a = min(a, smn[ww][k]); b = max(b, smx[ww][k]); }
    atomicMin(lohi + k, a);
    atomicMax(lohi + 8 + k, b);
  }
}

template <typename F>
static void by_dim(int d, F&& f) {
  switch (d) {
    case 1: f(std::integral_constant<int, 1>()); break;
    case 2: f(std::integral_constant<int, 2>()); break;
    case 3: f(std::integral_constant<int, 3>()); break;
    case 4: f(std::integral_constant<int, 4>()); break;
    case 5: f(std::integral_constant<int, 5>()); break;
    case 6: f(std::integral_constant<int, 6>()); break;
    case 7: f(std::integral_constant<int, 7>()); break;
    default: f(std::integral_constant<int, 8>()); break;
  }
}

// Sampled cell collisions, an estimate of how many distinct cells there are
// (it decides between the hash counting sort and the radix sort, DESIGN.md
// §a2): S = min(n, 4096) evenly spaced points, cell coordinates taken from a
// fixed origin (INT32_MIN; no bounding box needed, so this runs beside it),
// hashed to a non-zero 32-bit fingerprint and inserted into a shared-memory
// set; out = number of inserts that found their fingerprint already there.
// With m equally likely cells about S^2 / 2m samples collide.
constexpr int SAMPLE = 4096;
constexpr int SAMPLE_SLOTS = 2 * SAMPLE;

template <int DD>
__global__ void __launch_bounds__(1024) sample_collisions_kernel(const int32_t* __restrict__ pts, int64_t n,
                                                                 uint32_t s, int32_t* out) {
  __shared__ uint32_t set[SAMPLE_SLOTS];
  for (int t = threadIdx.x; t < SAMPLE_SLOTS; t += blockDim.x) set[t] = 0;
  __syncthreads();
  const int S = (int)min((int64_t)SAMPLE, n);
  int dup = 0;
  for (int t = threadIdx.x; t < S; t += blockDim.x) {
    const int64_t i = (int64_t)t * n / S;
    uint64_t h = 0x9e3779b97f4a7c15ull;
#pragma unroll
    for (int k = 0; k < DD; ++k) {
      const uint32_t c = ((uint32_t)pts[i * DD + k] ^ 0x80000000u) / s;  // (x - INT32_MIN) / s
      h = mix64(h ^ (c + 0x632be59bd9b4e019ull + (h << 6)));
    }
    const uint32_t f = (uint32_t)(h >> 32) | 1u;  // non-zero fingerprint
    uint32_t slot = (uint32_t)h & (SAMPLE_SLOTS - 1);
    while (true) {
      const uint32_t prev = atomicCAS(set + slot, 0u, f);
      if (prev == 0u) break;
      if (prev == f) { ++dup; break; }
      slot = (slot + 1) & (SAMPLE_SLOTS - 1);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) dup += __shfl_xor_sync(DB_FULL, dup, o);
  if ((threadIdx.x & 31) == 0 && dup) atomicAdd(out, dup);
}

void bbox(Ctx& c, const int32_t* pts, int64_t n, int d, uint32_t s, int32_t* lohi) {
  bbox_init_kernel<<<1, 32, 0, c.st>>>(lohi);
  c.launched();
  by_dim(d, [&](auto Dc) {
    constexpr int DD = decltype(Dc)::value;
    c.fork();  // the one-block sample runs beside the bounding box
    sample_collisions_kernel<DD><<<1, 1024, 0, c.side>>>(pts, n, s, lohi + 16);
    c.launched();
    bbox_kernel<DD><<<grid_for(n, 256, c.sms * 8), 256, 0, c.st>>>(pts, n, lohi);
    c.launched();
    c.join();
  });
}

// key = sum_k ((x_k - lo_k) div s) << shift_k; idx = input row; plus the
// 256-bin histogram of each of the `passes` 8-bit digits (onesweep's single
// up-front histogram), aggregated per warp with __match_any_sync before the
// shared atomics so that skewed digits (one value in most keys) do not
// serialise.
template <typename K, int DD>
__global__ void __launch_bounds__(256) keys_kernel(const int32_t* __restrict__ pts, uint32_t n,
                                                   Geo g, uint64_t magic, int passes,
                                                   K* __restrict__ keys, uint32_t* __restrict__ idx,
                                                   uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[8 * 256];
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t start = blockIdx.x * blockDim.x + threadIdx.x;
  // every thread runs the same number of iterations so the warp-level match is full
  const uint32_t iters = (n + stride - 1) / stride;
  for (uint32_t it = 0; it < iters; ++it) {
    const uint32_t i = start + it * stride;
    const bool valid = i < n;
    K key = 0;
    if (valid) {
#pragma unroll
      for (int k = 0; k < DD; ++k) {
        // x - lo in [0, 2^32): exact as an unsigned 32-bit difference
        const uint32_t off = (uint32_t)__ldg(pts + (uint64_t)i * DD + k) - (uint32_t)g.lo[k];
        const uint32_t ck = magic ? (uint32_t)__umul64hi((uint64_t)off, magic) : off;
        key |= (K)ck << g.shift[k];
      }
      keys[i] = key;
      idx[i] = i;
    }
    const uint32_t vmask = __ballot_sync(DB_FULL, valid);
    for (int p = 0; p < passes; ++p) {
      const uint32_t dg = (uint32_t)(key >> (8 * p)) & 255u;
      // a digit shared by the whole warp (clustered data) is one atomic; otherwise
      // one atomic per lane (uniform data: conflicts are rare)
      const uint32_t d0 = __shfl_sync(DB_FULL, dg, 0);
      if (__all_sync(DB_FULL, !valid || dg == d0)) {
        if ((threadIdx.x & 31) == 0 && vmask) atomicAdd(sh + p * 256 + d0, __popc(vmask));
      } else if (valid) {
        atomicAdd(sh + p * 256 + dg, 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * 256; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, sh[i]);
}

void cell_keys_and_sort(Ctx& c, const int32_t* pts, int64_t n, const Geo& g, bool key64,
                        void** sorted_keys, uint32_t** sorted_idx, int* passes_out) {
  const int passes = (int)((g.bits + 7) / 8);
  *passes_out = passes;
  // magic = ceil(2^64 / s) for s >= 2 (s = 1: identity)
  const uint64_t magic =
      g.s > 1 ? (uint64_t)((((unsigned __int128)1 << 64) + g.s - 1) / g.s) : 0;
  uint32_t* hist = c.alloc<uint32_t>(8 * 256);
  c.zero(hist, sizeof(uint32_t) * 8 * 256);
  uint32_t* v0 = c.alloc<uint32_t>(n);
  uint32_t* v1 = c.alloc<uint32_t>(n);
  const unsigned grid = grid_for(n, 256, c.sms * 8);
  if (key64) {
    uint64_t* k0 = c.alloc<uint64_t>(n);
    uint64_t* k1 = c.alloc<uint64_t>(n);
    by_dim(g.d, [&](auto Dc) {
      constexpr int DD = decltype(Dc)::value;
      keys_kernel<uint64_t, DD><<<grid, 256, 0, c.st>>>(pts, (uint32_t)n, g, magic, passes, k0, v0, hist);
    });
    c.launched();
    uint64_t* ko; uint32_t* vo;
    radix_sort_pairs_u64(c, k0, v0, k1, v1, (uint32_t)n, passes, hist, &ko, &vo);
    *sorted_keys = ko; *sorted_idx = vo;
  } else {
    uint32_t* k0 = c.alloc<uint32_t>(n);
    uint32_t* k1 = c.alloc<uint32_t>(n);
    by_dim(g.d, [&](auto Dc) {
      constexpr int DD = decltype(Dc)::value;
      keys_kernel<uint32_t, DD><<<grid, 256, 0, c.st>>>(pts, (uint32_t)n, g, magic, passes, k0, v0, hist);
    });
    c.launched();
    uint32_t* ko; uint32_t* vo;
    radix_sort_pairs_u32(c, k0, v0, k1, v1, (uint32_t)n, passes, hist, &ko, &vo);
    *sorted_keys = ko; *sorted_idx = vo;
  }
}

}  // namespace db
