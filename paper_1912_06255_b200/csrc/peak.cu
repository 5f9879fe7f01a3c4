// peak.cu — U1 `peak_dist`: the measured throughput of
// the exact distance predicate on this GPU, the denominator of the a6/a8
// roofline fractions. MarkCore (Alg 2) and the BCP of
// ClusterCore (Alg 3) are, per unit of work, one distance test
// ||p - q||^2 <= eps^2; the paper analyses MarkCore as
// O(n minPts) such tests.
//
// The kernel runs the SHIPPED predicate (common.cuh `within`, the same
// template the stage kernels instantiate) on a shared-memory tile of
// candidates against queries held in registers — the shape of the brick
// MarkCore (one candidate loaded from shared memory per test) at QT = 1, and
// a register tile that amortises the candidate load over QT queries at
// QT = 2, 4. Variants: 0 = uint32 `__sad` path (shipped for every BASELINE
// config), 1 = the 64-bit clamped path (shipped for wide inputs), 2 = fp64
// (north_star's "int64/fp64 pipe peak"; exact here because coordinates are
// < 2^12), 3 = the brick MarkCore's predicate (d = 3: candidates packed
// {x | y << 16, z} in an 8-byte shared-memory row, `brick_within`).
// Coordinates come from a counter-based hash on the device (no upload);
// about half the pairs pass, so the compare is data-dependent.
#include "internal.h"

namespace db {

constexpr int PK_M = 1024;       // candidates per shared-memory tile
constexpr int PK_THREADS = 256;

__device__ __forceinline__ uint32_t pk_hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int DIM, int V>
__device__ __forceinline__ bool pk_test(const int32_t* q, const int32_t* c, uint32_t clampc, uint64_t eps2) {
  if constexpr (V == 0) return within<DIM, false>(q, c, clampc, eps2);
  else if constexpr (V == 1) return within<DIM, true>(q, c, clampc, eps2);
  else {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      const double t = (double)q[k] - (double)c[k];
      acc = fma(t, t, acc);
    }
    return acc <= (double)eps2;
  }
}

// candidate m of the tile, as the stage kernels load a D-padded point
template <int DP>
__device__ __forceinline__ void pk_load(const int32_t* tile, int m, int32_t* x) {
  if constexpr (DP == 2) {
    const int2 v = reinterpret_cast<const int2*>(tile)[m];
    x[0] = v.x; x[1] = v.y;
  } else if constexpr (DP == 4) {
    const int4 v = reinterpret_cast<const int4*>(tile)[m];
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
  } else {
    const int4 a = reinterpret_cast<const int4*>(tile)[2 * m], b = reinterpret_cast<const int4*>(tile)[2 * m + 1];
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
}

// variant 3: the brick kernel's packed rows and predicate (d = 3)
template <int QT>
__global__ void __launch_bounds__(PK_THREADS) peak_brick_kernel(int64_t reps, uint32_t eps2,
                                                                unsigned long long* hits) {
  __shared__ uint2 tile[PK_M];
  for (int m = threadIdx.x; m < PK_M; m += blockDim.x) {
    const uint32_t x = pk_hash(blockIdx.x * 7919u + m * 131u) & 4095u,
                   y = pk_hash(blockIdx.x * 7919u + m * 131u + 1) & 4095u,
                   z = pk_hash(blockIdx.x * 7919u + m * 131u + 2) & 4095u;
    tile[m] = make_uint2(x | (y << 16), z);
  }
  uint32_t q[QT][3];
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int j = 0; j < QT; ++j)
#pragma unroll
    for (int k = 0; k < 3; ++k) q[j][k] = pk_hash(0x9e3779b9u ^ (tid * QT + j) * 17u + k) & 4095u;
  __syncthreads();
  uint32_t cnt[QT];
#pragma unroll
  for (int j = 0; j < QT; ++j) cnt[j] = 0;
  for (int64_t r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int m = 0; m < PK_M; ++m) {
      const uint2 c = tile[m];
#pragma unroll
      for (int j = 0; j < QT; ++j) cnt[j] += brick_within(q[j], c, eps2) ? 1u : 0u;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < QT; ++j) s += cnt[j];
  block_add_u64(s, hits);
}

template <int DIM, int V, int QT>
__global__ void __launch_bounds__(PK_THREADS) peak_dist_kernel(int64_t reps, uint32_t clampc, uint64_t eps2,
                                                               unsigned long long* hits) {
  constexpr int DP = DIM <= 2 ? 2 : (DIM <= 4 ? 4 : 8);
  __shared__ __align__(16) int32_t tile[PK_M * DP];
  for (int i = threadIdx.x; i < PK_M * DP; i += blockDim.x) {
    const int m = i / DP, k = i % DP;
    tile[i] = k < DIM ? (int32_t)(pk_hash(blockIdx.x * 7919u + m * 131u + k) & 4095u) : 0;
  }
  int32_t q[QT][DIM];
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int j = 0; j < QT; ++j)
#pragma unroll
    for (int k = 0; k < DIM; ++k) q[j][k] = (int32_t)(pk_hash(0x9e3779b9u ^ (tid * QT + j) * 17u + k) & 4095u);
  __syncthreads();
  uint32_t cnt[QT];
#pragma unroll
  for (int j = 0; j < QT; ++j) cnt[j] = 0;
  for (int64_t r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int m = 0; m < PK_M; ++m) {
      int32_t c[DP];
      pk_load<DP>(tile, m, c);
#pragma unroll
      for (int j = 0; j < QT; ++j) cnt[j] += pk_test<DIM, V>(q[j], c, clampc, eps2) ? 1u : 0u;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < QT; ++j) s += cnt[j];
  block_add_u64(s, hits);
}

}  // namespace db

using namespace db;

extern "C" int dbscan_peak_dist(int32_t d, int32_t variant, int32_t qt, int64_t reps, void* stream,
                                double* tests_per_s, double* ms_out, int64_t* tests_out, int64_t* hits_out) {
  if (d < 1 || d > 8 || variant < 0 || variant > 3 || (variant == 3 && d != 3) || !(qt == 1 || qt == 2 || qt == 4) ||
      reps < 1 || !tests_per_s)
    return DBSCAN_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return DBSCAN_ECUDA;
  }
  // eps^2 = half the mean squared distance of uniform [0, 4096)^d points
  // (~half the pairs pass); the 32-bit path is exact (d * 4096^2 < 2^32)
  const uint64_t half = (uint64_t)d * 4096ull * 4096ull / 12ull;
  uint64_t eps = 0;
  while ((eps + 1) * (eps + 1) <= half) ++eps;
  const uint32_t clampc = (uint32_t)eps + 1;
  const unsigned blocks = (unsigned)sms * 8;  // 8 CTAs of 256 threads per SM: full occupancy
  unsigned long long* dh = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (cudaMallocAsync(&dh, sizeof(unsigned long long), st) != cudaSuccess ||
      cudaMemsetAsync(dh, 0, sizeof(unsigned long long), st) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    (void)cudaGetLastError();
    return DBSCAN_ECUDA;
  }
  auto go = [&](auto dimc, auto vc, auto qc) {
    constexpr int DIM = decltype(dimc)::value, V = decltype(vc)::value, QT = decltype(qc)::value;
    peak_dist_kernel<DIM, V, QT><<<blocks, PK_THREADS, 0, st>>>(1, clampc, eps * eps, dh);  // warm-up
    cudaMemsetAsync(dh, 0, sizeof(unsigned long long), st);
    cudaEventRecord(e0, st);
    peak_dist_kernel<DIM, V, QT><<<blocks, PK_THREADS, 0, st>>>(reps, clampc, eps * eps, dh);
    cudaEventRecord(e1, st);
  };
  auto by_q = [&](auto dimc, auto vc) {
    if (qt == 1) go(dimc, vc, std::integral_constant<int, 1>());
    else if (qt == 2) go(dimc, vc, std::integral_constant<int, 2>());
    else go(dimc, vc, std::integral_constant<int, 4>());
  };
  auto brick = [&](auto qc) {
    constexpr int QT = decltype(qc)::value;
    peak_brick_kernel<QT><<<blocks, PK_THREADS, 0, st>>>(1, (uint32_t)(eps * eps), dh);  // warm-up
    cudaMemsetAsync(dh, 0, sizeof(unsigned long long), st);
    cudaEventRecord(e0, st);
    peak_brick_kernel<QT><<<blocks, PK_THREADS, 0, st>>>(reps, (uint32_t)(eps * eps), dh);
    cudaEventRecord(e1, st);
  };
  auto by_v = [&](auto dimc) {
    if (variant == 3) {
      if (qt == 1) brick(std::integral_constant<int, 1>());
      else if (qt == 2) brick(std::integral_constant<int, 2>());
      else brick(std::integral_constant<int, 4>());
    } else if (variant == 0) by_q(dimc, std::integral_constant<int, 0>());
    else if (variant == 1) by_q(dimc, std::integral_constant<int, 1>());
    else by_q(dimc, std::integral_constant<int, 2>());
  };
  switch (d) {
    case 1: by_v(std::integral_constant<int, 1>()); break;
    case 2: by_v(std::integral_constant<int, 2>()); break;
    case 3: by_v(std::integral_constant<int, 3>()); break;
    case 4: by_v(std::integral_constant<int, 4>()); break;
    case 5: by_v(std::integral_constant<int, 5>()); break;
    case 6: by_v(std::integral_constant<int, 6>()); break;
    case 7: by_v(std::integral_constant<int, 7>()); break;
    default: by_v(std::integral_constant<int, 8>()); break;
  }
  unsigned long long h = 0;
  float ms = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, dh, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaFreeAsync(dh, st);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return DBSCAN_ECUDA;
  }
  const double tests = (double)blocks * PK_THREADS * qt * (double)PK_M * (double)reps;
  *tests_per_s = tests / (ms / 1e3);
  if (ms_out) *ms_out = ms;
  if (tests_out) *tests_out = (int64_t)tests;
  if (hits_out) *hits_out = (int64_t)h;
  return DBSCAN_OK;
}
