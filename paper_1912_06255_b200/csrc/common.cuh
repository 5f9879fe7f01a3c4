// common.cuh — device-side building blocks shared by every stage of the
// B200 DBSCAN path: grid geometry, the exact distance predicates, union-find,
// warp/block scans and the decoupled look-back primitive.
//
// Product code. It never includes, links or calls anything under oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define DB_WARP 32
#define DB_FULL 0xffffffffu

namespace db {

// ---------------------------------------------------------------------------
// Work counters of the measurement build (make count: libdbscan_b200_count.so,
// -DDB_COUNT_WORK): every distance test of MarkCore (slot 0, a6), of the BCP
// in ClusterCore (slot 1, a8) and of ClusterBorder (slot 2, a10) adds one to a
// per-translation-unit device counter, summed into stats[] after the call
// (DBSCAN_STAT_*_TESTS). bench.py runs that build in a separate, untimed pass
// to get the algorithmic work behind the a6/a8/a10 roofline fractions; the
// product build compiles the macros away.
// ---------------------------------------------------------------------------
#ifdef DB_COUNT_WORK
static __device__ unsigned long long db_work_ctr[4];
#define DB_WORK(slot) atomicAdd(&::db::db_work_ctr[slot], 1ull)
#define DB_WORK_N(slot, n) atomicAdd(&::db::db_work_ctr[slot], (unsigned long long)(n))
#else
#define DB_WORK(slot) ((void)0)
#define DB_WORK_N(slot, n) ((void)0)
#endif

// ---------------------------------------------------------------------------
// Grid geometry (reading 5).
// Integer cell side s = isqrt(floor(eps^2/d)) + 1 so that two points of one
// cell differ by <= s-1 per axis and d (s-1)^2 <= eps^2 (same cell => within
// eps). Cell coordinate c_k = (x_k - lo_k) div s (half-open boxes,
// origin at the per-axis minimum). The packed cell key puts axis 0 in the most
// significant bits: key = sum_k c_k << shift_k, with w_k = bits(maxc_k).
// ---------------------------------------------------------------------------
struct Geo {
  int32_t  d;           // dimension
  int32_t  D;           // padded dimension of the sorted point array (2, 4 or 8)
  uint32_t s;           // integer cell side
  uint32_t bits;        // total key width (<= 63)
  int32_t  lo[8];       // per-axis minimum coordinate
  uint32_t maxc[8];     // per-axis maximum lattice coordinate
  uint32_t shift[8];    // bit position of axis k in the key
  uint32_t width[8];    // bit width of axis k
  uint64_t eps2;        // eps^2
  uint32_t clampc;      // eps + 1: Lemma 3 clamp (reading 4)
  uint32_t R;           // max |delta| of lattice coordinates between neighbour cells
  uint64_t eps;         // eps
  uint32_t at;          // rho-approximate DBSCAN (row f4): sub-cell side t >= 2; 0 = exact
  uint64_t eps2_apx;    // rho-approximate: floor((eps (1 + rho'))^2), rho' <= rho dyadic; 0 = exact
  uint32_t apxc;        // rho-approximate: per-axis clamp (> sqrt(eps2_apx))
};

__device__ __forceinline__ uint32_t cell_coord(uint64_t key, const Geo& g, int k) {
  return (uint32_t)((key >> g.shift[k]) & ((g.width[k] == 32) ? 0xffffffffull
                                                              : ((1ull << g.width[k]) - 1)));
}

// Squared gap between two lattice cells (or cell boxes) along one axis, in
// coordinate units: the closest integer coordinates of cells differing by
// delta != 0 are (|delta|-1)*s + 1 apart (reading 7). Clamped at
// eps+1 so the squared sum stays < 2^62 (d (eps+1)^2 < 2^62 is checked on the
// host); a clamped term alone already exceeds eps^2.
__device__ __forceinline__ uint64_t gap_term(uint32_t delta, const Geo& g) {
  if (delta == 0) return 0;
  uint64_t gap = (uint64_t)(delta - 1) * g.s + 1;
  if (gap > g.clampc) gap = g.clampc;
  return gap * gap;
}

// ---------------------------------------------------------------------------
// Exact distance predicate ||a-b||^2 <= eps^2 on int32 coordinates
// (closed neighbourhood). Every caller compares points of cells
// at most R apart per axis (stencil / neighbour cells), so |a_k - b_k| <=
// (R+1)s - 1. 32-bit path (reading 4): sum_k |a_k - b_k|^2 <= eps^2
// with |a_k - b_k| = __sad(a_k, b_k, 0), exact in uint32 because the host
// chooses it only when d ((R+1)s - 1)^2 < 2^32.
// Padded coordinates are 0 on both sides and contribute nothing.
// 64-bit path: 64-bit differences clamped at eps+1 (Lemma 3: a clamped term
// alone exceeds eps^2) and 64-bit sums (d (eps+1)^2 < 2^62).
// ---------------------------------------------------------------------------
template <int D, bool WIDE>
struct Pt;

template <> struct Pt<2, false> { int2 v; };
template <> struct Pt<2, true>  { int2 v; };
template <> struct Pt<4, false> { int4 v; };
template <> struct Pt<4, true>  { int4 v; };
template <> struct Pt<8, false> { int4 a, b; };
template <> struct Pt<8, true>  { int4 a, b; };

template <int D>
struct PtLoad {
  // Load point j of a D-padded array (16-byte rows for D=4, 8 for D=2, 32 for D=8).
  __device__ __forceinline__ static void load(const int32_t* __restrict__ P, int64_t j, int32_t* x);
};
template <> struct PtLoad<2> {
  __device__ __forceinline__ static void load(const int32_t* __restrict__ P, int64_t j, int32_t* x) {
    int2 v = __ldg(reinterpret_cast<const int2*>(P) + j);
    x[0] = v.x; x[1] = v.y;
  }
};
template <> struct PtLoad<4> {
  __device__ __forceinline__ static void load(const int32_t* __restrict__ P, int64_t j, int32_t* x) {
    int4 v = __ldg(reinterpret_cast<const int4*>(P) + j);
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
  }
};
template <> struct PtLoad<8> {
  __device__ __forceinline__ static void load(const int32_t* __restrict__ P, int64_t j, int32_t* x) {
    const int4* q = reinterpret_cast<const int4*>(P) + 2 * j;
    int4 a = __ldg(q), b = __ldg(q + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
};

template <int D, bool WIDE>
__device__ __forceinline__ bool within(const int32_t* a, const int32_t* b, uint32_t clampc,
                                       uint64_t eps2) {
  if constexpr (!WIDE) {
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const uint32_t t = __sad(a[k], b[k], 0u);
      acc += t * t;
    }
    return acc <= (uint32_t)eps2;
  } else {
    uint64_t acc = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      int64_t t = (int64_t)a[k] - (int64_t)b[k];
      uint64_t u = (uint64_t)(t < 0 ? -t : t);
      if (u > clampc) u = clampc;
      acc += u * u;
    }
    return acc <= eps2;
  }
}

// The brick MarkCore's predicate (sparse.cu): ||p - q||^2 <= eps^2 on 3D
// coordinates relative to the halo's origin, q packed {x | y << 16, z} (exact:
// each squared difference < 2^32 / 3). Also run by U1 (peak.cu, variant 3).
__device__ __forceinline__ bool brick_within(const uint32_t* p, uint2 q, uint32_t eps2) {
  const uint32_t dx = __sad(p[0], q.x & 0xffffu, 0u), dy = __sad(p[1], q.x >> 16, 0u), dz = __sad(p[2], q.y, 0u);
  return dx * dx + dy * dy + dz * dz <= eps2;
}

// Connectivity test of two core points in ClusterCore (Alg 3, the BCP).
// Exact DBSCAN: ||a-b|| <= eps. rho-approximate DBSCAN (row f4, Gan and Tao,
// PAPER.md P:L225-235): the points are snapped to sub-cells of integer side
// t (a grid aligned with the cells' origin lo) and connected when the two
// sub-cell boxes are within eps: sum_k gap_k^2 <= eps^2 with gap_k =
// (|dq_k|-1) t + 1 for sub-cell index difference dq_k != 0 (the exact box
// gap, as for cells, reading 7). A pair within eps always passes
// (the box gap is at most the point distance); a passing pair is within
// eps + 2 (t-1) sqrt(d) <= eps (1 + rho) because the host picks the largest
// t with 2 (t-1) sqrt(d) <= eps rho.
// The sub-cell snap is done once per point (connect_prep: identity for the
// exact test, sub-cell indices for the approximate one) and the test runs on
// the prepared values (connect_q); connect_test = both.
template <int D>
__device__ __forceinline__ void connect_prep(const int32_t* x, const Geo& g, int32_t* q) {
#pragma unroll
  for (int k = 0; k < D; ++k)
    q[k] = (g.at && k < g.d) ? (int32_t)(((uint32_t)x[k] - (uint32_t)g.lo[k]) / g.at) : x[k];
}

template <int D, bool WIDE>
__device__ __forceinline__ bool connect_q(const int32_t* qa, const int32_t* qb, const Geo& g) {
  if (g.at == 0) return within<D, WIDE>(qa, qb, g.clampc, g.eps2);
  uint64_t acc = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < g.d) {
      const uint32_t dq = __sad(qa[k], qb[k], 0u);
      uint64_t gap = dq ? (uint64_t)(dq - 1) * g.at + 1 : 0;
      if (gap > g.clampc) gap = g.clampc;
      acc += gap * gap;
    }
  }
  return acc <= g.eps2;
}

// rho-approximate cell-level cut-off (row f4; the paper's quadtree search
// "terminates once a node's sub-cell is completely contained in the
// eps(1+rho)-radius", at the root: the cell): two core cells
// whose lattice boxes are entirely within eps(1+rho) of each other may be
// connected without any point test — every pair of their points is within
// eps(1+rho), so connecting them is allowed, and the pairs within eps are
// connected as required. Cells differing by delta along an axis have points
// at most (|delta| + 1) s - 1 apart along it.
__device__ __forceinline__ bool apx_cells_within(uint64_t ka, uint64_t kb, const Geo& g) {
  if (!g.eps2_apx) return false;
  uint64_t acc = 0;
  for (int k = 0; k < g.d; ++k) {
    const uint32_t a = cell_coord(ka, g, k), b = cell_coord(kb, g, k);
    const uint64_t dl = a > b ? a - b : b - a;
    uint64_t m = (dl + 1) * (uint64_t)g.s - 1;
    if (m > g.apxc) m = g.apxc;
    acc += m * m;
  }
  return acc <= g.eps2_apx;
}

template <int D, bool WIDE>
__device__ __forceinline__ bool connect_test(const int32_t* a, const int32_t* b, const Geo& g) {
  int32_t qa[D], qb[D];
  connect_prep<D>(a, g, qa);
  connect_prep<D>(b, g, qb);
  return connect_q<D, WIDE>(qa, qb, g);
}

// Squared distance from point p to the integer box of cell `key`, clamped as
// above: [lo_k + c_k s, lo_k + c_k s + s - 1] per axis. Used by the BCP filter
// ("filter out points further than eps from the other cell").
// slack (rho-approximate DBSCAN): each per-axis gap is first reduced by
// slack = 2(t-1), the most the two sub-cell boxes of connect_test reach past
// their points; the filter then keeps every point that can pass the test.
template <int D>
__device__ __forceinline__ bool near_box(const int32_t* p, const int64_t* blo, const Geo& g, uint32_t slack = 0) {
  uint64_t acc = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < g.d) {
      int64_t x = p[k], lo = blo[k], hi = blo[k] + (int64_t)g.s - 1;
      int64_t t = x < lo ? lo - x : (x > hi ? x - hi : 0);
      t = t > (int64_t)slack ? t - (int64_t)slack : 0;
      uint64_t u = (uint64_t)t;
      if (u > g.clampc) u = g.clampc;
      acc += u * u;
    }
  }
  return acc <= g.eps2;
}

// Squared gap between the box [qlo, qhi] (the bounding box of some query
// points) and the integer box of a cell with lower corner blo, clamped as in
// near_box: <= eps^2 unless no point of the cell is within eps of any point
// in [qlo, qhi].
template <int D>
__device__ __forceinline__ bool near_box2(const int32_t* qlo, const int32_t* qhi, const int64_t* blo, const Geo& g) {
  uint64_t acc = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (k < g.d) {
      const int64_t lo = blo[k], hi = blo[k] + (int64_t)g.s - 1;
      const int64_t t = qlo[k] > hi ? qlo[k] - hi : (qhi[k] < lo ? lo - qhi[k] : 0);
      uint64_t u = (uint64_t)t;
      if (u > g.clampc) u = g.clampc;
      acc += u * u;
    }
  }
  return acc <= g.eps2;
}

template <int D>
__device__ __forceinline__ void cell_box_lo(uint64_t key, const Geo& g, int64_t* blo) {
#pragma unroll
  for (int k = 0; k < D; ++k)
    blo[k] = (k < g.d) ? (int64_t)g.lo[k] + (int64_t)cell_coord(key, g, k) * (int64_t)g.s : 0;
}

// ---------------------------------------------------------------------------
// Lock-free union-find over cells: parent[x] <= x
// always (a root is only ever linked under a smaller root), find uses path
// halving with plain stores (benign races: any stored value is an ancestor),
// link uses atomicCAS on the larger root and retries on failure.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t x) {
  volatile uint32_t* p = parent;
  while (true) {
    uint32_t px = p[x];
    if (px == x) return x;
    uint32_t gx = p[px];
    if (gx == px) return px;
    p[x] = gx;  // path halving
    x = gx;
  }
}

// Root through L1-cached loads, no writes. A cached parent value may be stale
// but is always an ancestor taken at some earlier time (values only move up
// the tree, ids strictly decrease along every chain, so the walk ends), and
// components only merge: equal stale roots prove a and b connected, unequal
// ones prove nothing. Keeps the Find filter off the one L2 line of a large
// component's root, which every volatile Find reads (same-address hot spot).
__device__ __forceinline__ uint32_t uf_root_cached(const uint32_t* parent, uint32_t x) {
  while (true) {
    const uint32_t px = __ldca(parent + x);
    if (px == x) return x;
    x = px;
  }
}

// Find(a) == Find(b): the cached walk first, the coherent one if it differs.
__device__ __forceinline__ bool uf_same(uint32_t* parent, uint32_t a, uint32_t b) {
  if (uf_root_cached(parent, a) == uf_root_cached(parent, b)) return true;
  return uf_find(parent, a) == uf_find(parent, b);
}

// Find(a) == Find(b) with the parents compared first: equal parents (both
// ancestors) prove the pair connected with two loads spread over the array,
// none of them on the root's line. Pays off after a flatten pass
// (parent[x] = root), when most pairs share one root.
__device__ __forceinline__ bool uf_same_hop(uint32_t* parent, uint32_t a, uint32_t b) {
  volatile uint32_t* p = parent;
  if (p[a] == p[b]) return true;
  return uf_find(parent, a) == uf_find(parent, b);
}

__device__ __forceinline__ void uf_link(uint32_t* parent, uint32_t a, uint32_t b) {
  while (true) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a < b) { uint32_t t = a; a = b; b = t; }
    uint32_t old = atomicCAS(parent + a, a, b);
    if (old == a) return;
    a = old;
  }
}

// ---------------------------------------------------------------------------
// Scans.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(DB_FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan; returns the block total through *total.
// `smem` must hold 33 T. All threads of the block must call it.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) smem[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T w = lane < nw ? smem[lane] : T(0);
    T wi = warp_inclusive_scan(w);
    if (lane < nw) smem[lane] = wi - w;
    if (lane == nw - 1) smem[32] = wi;
  }
  __syncthreads();
  T res = inc - v + smem[wid];
  *total = smem[32];
  __syncthreads();
  return res;
}

// Decoupled look-back (single-pass chained scan): status words hold a 2-bit
// flag (1 = aggregate of this tile, 2 = inclusive prefix) and a 62-bit value.
constexpr uint64_t LB_AGG = 1ull << 62;
constexpr uint64_t LB_INC = 2ull << 62;
constexpr uint64_t LB_VAL = (1ull << 62) - 1;

__device__ __forceinline__ void lb_publish(uint64_t* st, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(st), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t lb_read(const uint64_t* st) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(st) : "memory");
  return v;
}

// Exclusive prefix of tile `tile` for one lane of status (stride `stride`
// between tiles): publishes the aggregate, walks back, publishes the inclusive
// value, returns the exclusive prefix. Called by one thread per status lane.
__device__ __forceinline__ uint64_t lb_exclusive(uint64_t* status, int64_t tile, int64_t stride,
                                                 uint64_t agg) {
  if (tile == 0) {
    lb_publish(status, LB_INC | agg);
    return 0;
  }
  lb_publish(status + tile * stride, LB_AGG | agg);
  uint64_t excl = 0;
  int64_t t = tile - 1;
  while (true) {
    uint64_t s = lb_read(status + t * stride);
    if ((s & ~LB_VAL) == 0) continue;  // predecessor not published yet: spin
    excl += s & LB_VAL;
    if (s & LB_INC) break;
    --t;
  }
  lb_publish(status + tile * stride, LB_INC | (excl + agg));
  return excl;
}

// The same look-back by a whole warp (call from every lane of ONE warp; the
// result is valid in every lane): the lanes read 32 predecessors at once,
// wait until all of them have published, and stop at the nearest inclusive
// prefix — a chain of aggregate-only tiles costs one round trip per 32 tiles.
__device__ __forceinline__ uint64_t lb_exclusive_warp(uint64_t* status, int64_t tile, int64_t stride,
                                                      uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) lb_publish(status, LB_INC | agg);
    return 0;
  }
  if (lane == 0) lb_publish(status + tile * stride, LB_AGG | agg);
  uint64_t excl = 0;
  int64_t t = tile - 1;
  while (true) {
    const int64_t tt = t - lane;
    uint64_t s = tt >= 0 ? lb_read(status + tt * stride) : (LB_INC | 0ull);
    while (!__all_sync(0xffffffffu, (s & ~LB_VAL) != 0))
      if ((s & ~LB_VAL) == 0) s = lb_read(status + tt * stride);
    const uint32_t inc = __ballot_sync(0xffffffffu, (s & LB_INC) != 0);
    const int k = inc ? __ffs(inc) - 1 : 31;  // lanes 0..k count
    uint64_t v = lane <= k ? (s & LB_VAL) : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc) break;
    t -= 32;
  }
  if (lane == 0) lb_publish(status + tile * stride, LB_INC | (excl + agg));
  return excl;
}

// Add v over the whole block to *dst with ONE atomic (thread 0). Every thread
// of the block must call it. Same-address atomics serialise in L2 (about one
// per clock), so per-thread or per-warp counters over millions of items cost
// hundreds of microseconds; per-block aggregation removes that.
__device__ __forceinline__ void block_add_u64(unsigned long long v, unsigned long long* dst) {
  __shared__ unsigned long long s_part[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(DB_FULL, v, o);
  __syncthreads();  // s_part is free (a previous call may still be reading it)
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) t += s_part[w];
    if (t) atomicAdd(dst, t);
  }
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// One-dimensional TMA bulk copy global -> shared (cp.async.bulk, SASS
// UBLKCP) completing on an mbarrier: one elected thread moves a whole
// contiguous chunk, so a block's input arrives with no per-thread load
// latency chains. dst, src and bytes must be multiples of 16.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  }
}

// Hash of a packed cell key into an open-addressing table of 16-byte slots.
// Keys that differ only in the low 3 bits (consecutive cells along the last
// axis) land in the same 8-slot (128-byte) group, so stencil probes of
// neighbouring cells share cache lines.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}
__device__ __forceinline__ uint64_t slot_of(uint64_t key, uint64_t mask) {
  return ((mix64(key >> 3) << 3) | (key & 7)) & mask;
}

constexpr uint64_t EMPTY_KEY = ~0ull;  // never a valid key (keys use <= 63 bits)

struct __align__(16) Slot {
  unsigned long long key;
  uint32_t val;
  uint32_t pad;
};

__device__ __forceinline__ uint32_t hash_lookup(const Slot* __restrict__ T, uint64_t mask,
                                                uint64_t key) {
  uint64_t h = slot_of(key, mask);
  while (true) {
    uint4 s = __ldg(reinterpret_cast<const uint4*>(T + h));
    uint64_t k = ((uint64_t)s.y << 32) | s.x;
    if (k == key) return s.z;
    if (k == EMPTY_KEY) return 0xffffffffu;
    h = (h + 1) & mask;
  }
}

}  // namespace db
