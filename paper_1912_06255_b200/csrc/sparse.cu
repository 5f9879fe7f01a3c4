// sparse.cu — the cell-centric path for sparse lattices (d <= 3, few points
// per cell, e.g. BASELINE configs[4] "3D uniform fill": 8.9M cells of ~1.1
// points). It computes exactly what the CSR path computes (rows a4-a10 of
// SURVEY §8(a)) but never materialises neighbour lists: with ~26 non-empty
// neighbours of ~1 point per cell, building and re-reading a CSR costs more
// than walking the stencil again.
//
//  * Cell lookup (a4): a rank directory over the lattice padded by R cells.
//    One 16-byte entry per 32 lattice cells holds that word of the occupancy
//    bitmap, the next word and the number of occupied cells before it (L2
//    resident: 21 MB for c5). Cell ids follow key order, which is the
//    lattice's linear order, so one load answers "which cells of this run of
//    up to 32 lattice cells exist, and what are their ids". The exact stencil
//    (reading 7) is a union of COLUMNS, runs of consecutive cells
//    along the last axis (25 in 3D, 5 in 2D); a column's cells have
//    consecutive ids and their points are one contiguous range of Ps.
//    Out-of-range neighbours land in the padding (no range checks).
//  * MarkCore (a6, Alg 2): 3D lattices with 0.15-0.3 points per
//    cell and R = 2 (c5): bricks of 16^3 cells staged with their halo in
//    shared memory, a thread per own point walking the 25 column ranges in
//    one branch-free loop (sp_core_brick_kernel); otherwise a thread per
//    point over the columns on the directory (sp_core_kernel). Counting stops
//    at minPts; a cell with |g| >= minPts is all core.
//  * a7: a thread per 8 cells counts core points; mixed cells are
//    partitioned core-first (core.cu); a second directory covers only the
//    cells holding core points, with the list of those cells in linear order.
//  * ClusterCore (a8, Alg 3): over the core cells, the lanes of a
//    warp take (core cell g, back column) items — back columns hold the
//    cells before g in linear order, so each pair is seen once, from its
//    higher id ("g > h") — probe the core directory and test the
//    core cells found: small BCPs directly (cheaper than the Finds that could
//    prune them), larger ones after a Find check through the warp BCP kernel
//    (cluster.cu). When most cells hold core points, the gap-0 columns run
//    first and the rest with Find first.
//  * ClusterBorder (a10, Alg 4): from the core cells (a warp per
//    core cell: candidates of its 25 columns laid out flat over the lanes,
//    labels added to lock-free 4-slot sets in input order), or, when the
//    non-core points are fewer than the core cells, from the points (a
//    thread per non-core point on the core directory). Larger sets are
//    enumerated without storage in ascending order.
#include <algorithm>
#include <array>
#include <map>

#include "internal.h"

namespace db {

constexpr int SP_MAXL = 4;
constexpr int SP_MAX_COLS = 32;  // lane per column in the MarkCore warp (3D: 25)
constexpr uint32_t MISS = 0xffffffffu;
constexpr uint32_t SP_SMALL = 64;

constexpr int BRK = 16;                  // brick side in cells
constexpr int BRK_R = 2;                 // halo (R = 2; the usual case for d = 3)
constexpr int BRK_H = BRK + 2 * BRK_R;   // 20
constexpr int BRK_COLS = BRK_H * BRK_H;  // halo columns
constexpr int BRK_CAP = 2400;            // halo points held in shared memory (c5: mean 1,864, sd 43)
constexpr int BRK_THREADS = 512;
constexpr int BRK_PER = (BRK_COLS + BRK_THREADS - 1) / BRK_THREADS;
constexpr int BRK_MAXC = (2 * BRK_R + 1) * (2 * BRK_R + 1);  // stencil columns at R = 2: 25

// stencil columns for the brick kernel, nearest first: window of column k of
// a cell at abs row index i = abs_flat[i + A[k]] .. abs_flat[i + B[k]]
// (the cell-level stencil; the kernel walks the sub-cell tables below and
// uses these only to count Alg 2's work in the measurement build)
struct BrickCols {
  int32_t A[BRK_MAXC], B[BRK_MAXC];  // byte offsets (2 per abs entry)
  int32_t ncols;
  uint32_t thr[3];                   // sub-cell thresholds t_1..t_3 of a cell offset (BRK_SUB per axis)
  int32_t nwmax;                     // most windows of a sub-cell stencil
};

// Sub-cell stencils (DESIGN.md §5 "MarkCore"): a point's offset inside its
// cell, o_k = x_k - lo_k - c_k s in [0, s), falls in one of BRK_SUB
// sub-intervals per axis (j_k = #{i : o_k >= t_i}); for each of the
// BRK_SUB^3 sub-cells the windows are the cells whose box lies within eps of
// the sub-cell's box (the exact gap of reading 7 between the sub-interval and
// the cell) — a subset of the cell-level stencil that still holds every point
// within eps of any point of the sub-cell, so the count is unchanged.
// Entry (uint16): byte offset A of the window's first abs entry relative to
// the point's own (column, z) entry, + 2048, in bits 0-11; the window's span
// in bytes (2 per cell) in bits 12-15. Nearest column first.
constexpr int BRK_SUB = 4;
constexpr int BRK_NSUB = BRK_SUB * BRK_SUB * BRK_SUB;
struct BrickTab {
  uint16_t w[BRK_NSUB][BRK_MAXC];
  uint8_t nw[BRK_NSUB];
};

struct SpArgs {
  Geo g;
  uint64_t stride[3];
  const uint4* dir;          // all cells: {bits of word w, bits of w+1, cells before w, 0}
  const uint4* cdir;         // cells with core points, same layout
  const uint32_t* core_list; // cells with core points in linear order (rank in cdir -> id)
  uint32_t ncore;
  const long long* coff;     // stencil columns: start offset (padded linear units), nearest first
  const uint32_t* cmask;     // stencil columns: (1 << width) - 1
  int ncols;
  const long long* bcoff;    // back columns (cells before g in linear order)
  const uint32_t* bcmask;
  int nbcols;
  int nbnear;                // back columns at gap 0 (first in the list): ClusterCore's first pass
  int nbmid;                 // back columns adjacent laterally (gap <= d - 1): the second pass
  uint32_t ncells;
  const uint32_t* cell_start;
  const uint64_t* cell_key;
  const uint32_t* cell_of;
  int32_t* Ps;
  uint32_t* idx;
  uint8_t* core_s;
  uint32_t* core_cnt;
  int64_t min_pts;
  uint32_t* counters;        // [1] brick overflow, [2] large pairs, [3] mixed cells,
                             // [4] core cells, [5] core points (one u64 atomic)
  uint32_t* mixed_list;
  uint32_t* core_tmp;        // cells with core points, unordered (count in counters[4])
  const uint32_t* cell_label;
  uint32_t* parent;
  uint2* large;
  uint32_t large_cap;
  uint32_t* bcnt;            // [n] input order
  uint32_t* tmp_lab;         // [n*SP_MAXL] label sets by sorted position (MISS = empty slot)
  uint8_t* tmp_n;            // [n] by sorted position: 0 no label, 1 labels in tmp_lab, 0xff overflowed
  uint32_t* ovf_list;        // sorted positions of overflowed sets (count in ovf_count)
  uint32_t* ovf_count;
  unsigned long long* nborder;
  const uint32_t* cpre;      // [ncore + 1] core points before each core cell (core_list order)
  const uint64_t* clin;      // [ncore] padded linear lattice index of each core cell (by rank)
  const uint32_t* ccnt;      // [ncore] core points of each core cell (by rank)
  const int4* cpts;          // core points in core_list order: {x, y, z (0 in 2D), cell id}
  uint64_t ncpts;            // core points
  int64_t n;
};

// Cells of the lattice run start .. start+width-1 (mask = (1 << width) - 1,
// width <= 32): returns how many exist; *id0 = the first one's id (rank).
__device__ __forceinline__ uint32_t dir_probe(const uint4* __restrict__ dir, uint64_t start, uint32_t mask,
                                              uint32_t* id0) {
  const uint4 e = __ldg(dir + (start >> 5));
  const uint32_t b0 = (uint32_t)start & 31u;
  const uint32_t bits = __funnelshift_r(e.x, e.y, b0) & mask;
  if (!bits) return 0;
  *id0 = e.z + __popc(e.x & ((1u << b0) - 1u));
  return __popc(bits);
}

// rank of an occupied lattice cell
__device__ __forceinline__ uint32_t dir_rank(const uint4* __restrict__ dir, uint64_t lin) {
  const uint4 e = __ldg(dir + (lin >> 5));
  return e.z + __popc(e.x & ((1u << ((uint32_t)lin & 31u)) - 1u));
}

template <int DIM>
__device__ __forceinline__ uint64_t cell_lin(uint64_t key, const SpArgs& a) {
  uint64_t lin = 0;
#pragma unroll
  for (int k = 0; k < DIM; ++k) lin += (uint64_t)(cell_coord(key, a.g, k) + a.g.R) * a.stride[k];
  return lin;
}

template <int D>
__device__ __forceinline__ void load_pt(const int32_t* __restrict__ Ps, uint32_t j, int32_t* x) {
  PtLoad<D>::load(Ps, j, x);
}

// ||p - q||^2 <= eps^2 over the first DIM coordinates (the padding is 0 on
// both sides; skipping it saves an axis in 3D)
template <int DIM, int D, bool WIDE>
__device__ __forceinline__ bool within_dim(const int32_t* p, const int32_t* q, const Geo& g) {
  int32_t a[D], b[D];
#pragma unroll
  for (int k = 0; k < D; ++k) { a[k] = k < DIM ? p[k] : 0; b[k] = k < DIM ? q[k] : 0; }
  return within<D, WIDE>(a, b, g.clampc, g.eps2);
}

// ------------------------------------------------------------- directories
// every cell (list = NULL), or the cells list[0 .. *count) (grid-stride)
__global__ void dir_set_kernel(const uint64_t* __restrict__ cell_key, uint32_t ncells, SpArgs a,
                               const uint32_t* __restrict__ list, const uint32_t* __restrict__ count,
                               uint32_t* bm) {
  const uint32_t m = list ? *count : ncells;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
    const uint32_t i = list ? list[t] : t;
    const uint64_t key = cell_key[i];
    uint64_t lin = 0;
    for (int k = 0; k < a.g.d; ++k) lin += (uint64_t)(cell_coord(key, a.g, k) + a.g.R) * a.stride[k];
    atomicOr(bm + (lin >> 5), 1u << (lin & 31));
  }
}

__global__ void popc_kernel(const uint32_t* __restrict__ bm, uint64_t words, uint32_t* __restrict__ cnt) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < words) cnt[i] = __popc(bm[i]);
}

__global__ void dir_pack_kernel(const uint32_t* __restrict__ bm, const uint32_t* __restrict__ pre, uint64_t words,
                                uint4* __restrict__ dir) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < words) dir[i] = make_uint4(bm[i], i + 1 < words ? bm[i + 1] : 0u, pre[i], 0u);
}

// core_list[rank in cdir] = cell id, for every cell holding core points
// (from the unordered list core_tmp[0 .. counters[4]))
// (also, by rank, each core cell's core count and padded lattice index: the
// packed core points of the one-pass ClusterCore are built from them)
__global__ void core_list_kernel(SpArgs a, uint32_t* __restrict__ core_list, uint32_t* __restrict__ ccnt,
                                 uint64_t* __restrict__ clin) {
  const uint32_t m = a.counters[4];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
    const uint32_t g = a.core_tmp[t];
    uint64_t lin = 0;
    const uint64_t key = a.cell_key[g];
    for (int k = 0; k < a.g.d; ++k) lin += (uint64_t)(cell_coord(key, a.g, k) + a.g.R) * a.stride[k];
    const uint32_t r = dir_rank(a.cdir, lin);
    core_list[r] = g;
    ccnt[r] = a.core_cnt[g];
    clin[r] = lin;
  }
}

// largest cell size (block max, one atomic per block)
__global__ void __launch_bounds__(256) cell_max_kernel(const uint32_t* __restrict__ cell_start,
                                                       uint32_t ncells, uint32_t* mx) {
  uint32_t m = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += gridDim.x * blockDim.x)
    m = max(m, cell_start[i + 1] - cell_start[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(DB_FULL, m, o));
  __shared__ uint32_t sm[8];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, sm[w]);
    atomicMax(mx, m);
  }
}

// ------------------------------------------------------------ MarkCore (a6)
// Thread per sorted point (Alg 2): a dense cell (|g| >= minPts)
// is all core; otherwise count the points within eps over the
// stencil columns, nearest column first, stopping at minPts. The own cell
// lies in the central column and passes the same test (same cell => within
// eps; p counts itself). Consecutive lanes hold consecutive sorted
// points (mostly one cell or its last-axis neighbours), so their column
// probes and point loads hit the same lines. The range loop is unrolled by U:
// U candidate loads in flight per thread, ceil(max range / U) iterations per
// column for the warp. Measured alternatives on c5: a warp per
// cell (latency-bound), a flat or two-phase per-point loop, U = 4, and
// symmetric counting with atomics were all slower.
// fb != NULL (after the brick kernel): runs only if *fb is set, and only on
// the points of bricks that overflowed (core_s still 0xff).
template <int DIM, int D, bool WIDE, int U>
__global__ void __launch_bounds__(256) sp_core_kernel(SpArgs a, const uint32_t* fb) {
  if (fb && *fb == 0) return;
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  for (int i = threadIdx.x; i < a.ncols; i += blockDim.x) { s_off[i] = a.coff[i]; s_mask[i] = a.cmask[i]; }
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < a.n && (!fb || a.core_s[j] == 0xff)) {
    const uint32_t g = a.cell_of[j];
    const uint32_t m = a.cell_start[g + 1] - a.cell_start[g];
    if ((int64_t)m >= a.min_pts) {
      a.core_s[j] = 1;  // dense cell
    } else {
      const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
      int32_t p[D];
      load_pt<D>(a.Ps, j, p);
      const uint32_t need = (uint32_t)min(a.min_pts, (int64_t)0xffffffff);
      uint32_t count = 0;
      for (int c = 0; c < a.ncols && count < need; ++c) {
        uint32_t id0;
        const uint32_t nc = dir_probe(a.dir, base + (uint64_t)s_off[c], s_mask[c], &id0);
        if (!nc) continue;
        const uint32_t ue = a.cell_start[id0 + nc];
        for (uint32_t u = a.cell_start[id0]; u < ue && count < need; u += U) {
          int32_t q[U][D];
#pragma unroll
          for (int k = 0; k < U; ++k)
            if (u + k < ue) load_pt<D>(a.Ps, u + k, q[k]);
#pragma unroll
          for (int k = 0; k < U; ++k)
            if (u + k < ue) count += within_dim<DIM, D, WIDE>(p, q[k], a.g);
          DB_WORK_N(0, min((uint32_t)U, ue - u));
          DB_WORK_N(3, min((uint32_t)U, ue - u));
        }
      }
      a.core_s[j] = count >= need;
    }
  }
}

// Brick variant of MarkCore (d = 3, R = 2; the default for 3D sparse
// lattices). A CTA takes a brick of BRK^3 lattice cells and stages the points
// of the brick and of its R-cell halo in shared memory: every halo column (a
// run of BRK_H cells along z) is one contiguous range of Ps, found with one
// directory probe and brought in by ONE TMA bulk copy (cp.async.bulk,
// completing on an mbarrier), with, per halo column, the positions of its
// cells' first points (abs). Then a thread per own point counts over the
// stencil columns from shared memory only (Alg 2; nearest column
// first, stopping at minPts; a dense cell is all core), in two
// phases:
//  A. the stencil columns' windows [z - m, z + m] are read from abs with
//     column offsets that are kernel parameters (constant-bank operands in a
//     fully unrolled loop) and the NON-EMPTY ones appended to a per-thread
//     list (interleaved by thread: conflict-free);
//  B. one flat loop over the listed candidates: a step fetches the next
//     list entry when the current range is spent and tests one candidate —
//     every step is a distance test, and empty columns cost no step.
// A brick whose halo holds more than BRK_CAP points sets *overflow and leaves
// its points to the thread kernel (core_s stays 0xff for them).

struct BrickSmem {
  union {
    int4 raw[BRK_CAP];                     // the halo's points as copied (x, y, z, 0)
    uint32_t list[BRK_MAXC][BRK_THREADS];  // phase A: non-empty windows, start | end << 16
  };
  uint2 pts[BRK_CAP];                    // the same points relative to the halo's origin:
                                         // {x | y << 16, z} (< 2^16: s BRK_H < 2^16 / sqrt 3)
  uint16_t abs[BRK_COLS][BRK_H + 1];     // per column: index in pts of its cell z (z = BRK_H: end)
  int32_t gdelta[BRK_COLS];              // sorted position - index in pts, per column
  uint32_t obase[BRK_COLS];              // prefix of the own points per column
  BrickTab tab;                          // sub-cell stencils
  uint32_t cbits[BRK_COLS];              // per column: occupancy of its BRK_H cells
  uint32_t crank[BRK_COLS];              // per column: id of its first occupied cell
  unsigned long long scan[33];
  uint32_t total, own;
  uint64_t bar;
};


__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}


template <bool WIDE>
__global__ void __launch_bounds__(BRK_THREADS, 2) sp_core_brick_kernel(SpArgs a, const BrickCols cols,
                                                                    const BrickTab* __restrict__ gtab,
                                                                    uint32_t nby, uint32_t nbz,
                                                                    uint32_t* overflow) {
  extern __shared__ __align__(16) uint8_t brick_raw[];
  BrickSmem& S = *reinterpret_cast<BrickSmem*>(brick_raw);
  {  // sub-cell stencils (read from L2 by every CTA: 3.3 KB)
    static_assert(sizeof(BrickTab) % 4 == 0, "BrickTab copied by words");
    const uint32_t* src = reinterpret_cast<const uint32_t*>(gtab);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&S.tab);
    for (int i = threadIdx.x; i < (int)(sizeof(BrickTab) / 4); i += BRK_THREADS) dst[i] = __ldg(src + i);
  }
  const uint32_t bid = blockIdx.x;
  const uint32_t bz = bid % nbz, by = (bid / nbz) % nby, bx = bid / (nbz * nby);
  const uint64_t Dx = a.g.maxc[0] + 1 + 2 * BRK_R, Dy = a.g.maxc[1] + 1 + 2 * BRK_R,
                 Dz = a.g.maxc[2] + 1 + 2 * BRK_R;
  // padded lattice coordinates of the halo origin: own cells start at +R
  const uint64_t X0 = (uint64_t)bx * BRK, Y0 = (uint64_t)by * BRK, Z0 = (uint64_t)bz * BRK;
  if (threadIdx.x == 0) {
    mbar_init(&S.bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- phase 0: a thread per halo column — one directory word pair covers its
  // BRK_H cells (b0 + 20 <= 51 bits); cell ends are independent loads
  uint32_t len[BRK_PER], own[BRK_PER], g0s[BRK_PER];
#pragma unroll
  for (int q = 0; q < BRK_PER; ++q) {
    const int cc = threadIdx.x * BRK_PER + q;
    len[q] = own[q] = g0s[q] = 0;
    if (cc >= BRK_COLS) continue;
    const uint32_t hx = cc / BRK_H, hy = cc % BRK_H;
    const uint64_t X = X0 + hx, Y = Y0 + hy;
    uint32_t bits = 0, r = 0;
    if (X < Dx && Y < Dy) {
      const uint32_t hz = (uint32_t)min((uint64_t)BRK_H, Dz - Z0);
      const uint64_t lin0 = (X * Dy + Y) * Dz + Z0;
      const uint4 e = __ldg(a.dir + (lin0 >> 5));
      const uint32_t b0 = (uint32_t)lin0 & 31u;
      bits = __funnelshift_r(e.x, e.y, b0) & ((1u << hz) - 1u);
      r = e.z + __popc(e.x & ((1u << b0) - 1u));
    }
    const uint32_t g0 = __ldg(a.cell_start + r);
    uint32_t run = 0, o0 = 0, o1 = 0;
#pragma unroll
    for (int z = 0; z < BRK_H; ++z) {
      if (z == BRK_R) o0 = run;
      if (z == BRK_R + BRK) o1 = run;
      S.abs[cc][z] = (uint16_t)min(run, 65535u);  // (made absolute below)
      if ((bits >> z) & 1u) run = __ldg(a.cell_start + r + __popc(bits & ((2u << z) - 1u))) - g0;
    }
    S.abs[cc][BRK_H] = (uint16_t)min(run, 65535u);
    S.cbits[cc] = bits;
    S.crank[cc] = r;
    len[q] = run;
    g0s[q] = g0;
    own[q] = (hx >= BRK_R && hx < BRK_R + BRK && hy >= BRK_R && hy < BRK_R + BRK) ? o1 - o0 : 0u;
  }
  // column bases (all halo points) and own-point prefixes: one 64-bit scan
  uint32_t el;
  {
    unsigned long long sv = 0;
#pragma unroll
    for (int q = 0; q < BRK_PER; ++q) sv += (unsigned long long)len[q] | ((unsigned long long)own[q] << 32);
    unsigned long long tot;
    const unsigned long long ex = block_exclusive_scan<unsigned long long>(sv, S.scan, &tot);
    el = (uint32_t)ex;
    uint32_t eo = (uint32_t)(ex >> 32);
#pragma unroll
    for (int q = 0; q < BRK_PER; ++q) {
      const int cc = threadIdx.x * BRK_PER + q;
      if (cc < BRK_COLS) S.obase[cc] = eo;
      eo += own[q];
    }
    if (threadIdx.x == 0) {
      S.total = (uint32_t)tot;
      S.own = (uint32_t)(tot >> 32);
      // (a column over 65535 points also overflows: tot would exceed BRK_CAP)
      if ((uint32_t)(tot >> 32) > 0 && (uint32_t)tot <= BRK_CAP) mbar_expect_tx(&S.bar, (uint32_t)tot * 16u);
    }
  }
  __syncthreads();
  const uint32_t total = S.total, nown = S.own;
  if (nown == 0) return;
  if (total > BRK_CAP) {
    if (threadIdx.x == 0) atomicExch(overflow, 1u);
    return;  // the thread kernel takes this brick's points (core_s left at 0xff)
  }
  // ---- phase 0b: one TMA bulk copy per non-empty halo column; abs made absolute
#pragma unroll
  for (int q = 0; q < BRK_PER; ++q) {
    const int cc = threadIdx.x * BRK_PER + q;
    if (cc >= BRK_COLS) continue;
    if (len[q]) bulk_copy(&S.raw[el], reinterpret_cast<const int4*>(a.Ps) + g0s[q], len[q] * 16u, &S.bar);
#pragma unroll
    for (int z = 0; z <= BRK_H; ++z) S.abs[cc][z] += (uint16_t)el;
    S.gdelta[cc] = (int32_t)(g0s[q] - el);
    el += len[q];
  }
  __syncthreads();
  mbar_wait(&S.bar, 0);
  // ---- points relative to the halo's origin (lattice coordinate X0 - R of
  // halo cell 0): 16 bits per axis, half the shared-memory wavefronts of a
  // candidate load, squared distances exact in 32 bits
  {
    const uint32_t ox = (uint32_t)a.g.lo[0] + (uint32_t)(X0 - BRK_R) * a.g.s;
    const uint32_t oy = (uint32_t)a.g.lo[1] + (uint32_t)(Y0 - BRK_R) * a.g.s;
    const uint32_t oz = (uint32_t)a.g.lo[2] + (uint32_t)(Z0 - BRK_R) * a.g.s;
    for (uint32_t k = threadIdx.x; k < total; k += BRK_THREADS) {
      const int4 v = S.raw[k];
      S.pts[k] = make_uint2(((uint32_t)v.x - ox) | (((uint32_t)v.y - oy) << 16), (uint32_t)v.z - oz);
    }
  }
  __syncthreads();  // (phase A's lists overwrite raw)
  // ---- a thread per own point
  const uint32_t need = (uint32_t)min(a.min_pts, (int64_t)0xffffffff);
  const uint32_t eps2 = (uint32_t)a.g.eps2;
  const uint16_t* abs_flat = &S.abs[0][0];
  for (uint32_t t = threadIdx.x; t < nown; t += blockDim.x) {
    // its column: the last one whose own prefix is <= t (never an empty one)
    int cc = 0;
#pragma unroll
    for (int step = 256; step; step >>= 1)
      if (cc + step < BRK_COLS && S.obase[cc + step] <= t) cc += step;
    const uint16_t* col = S.abs[cc];
    const uint32_t i = t - S.obase[cc] + col[BRK_R];  // index in pts
    // its cell: the last own z whose start is <= i
    int hz = BRK_R;
#pragma unroll
    for (int step = 8; step; step >>= 1)
      if (col[hz + step] <= i) hz += step;
    const uint32_t j = (uint32_t)((int32_t)i + S.gdelta[cc]);  // sorted position
    // (a core point adds one to its cell's core count, core_cnt zeroed before
    // the kernel: a7's sp_cells then reads the counts instead of the flags)
    const uint32_t cell = S.crank[cc] + __popc(S.cbits[cc] & ((1u << hz) - 1u));
    if ((int64_t)(col[hz + 1] - col[hz]) >= a.min_pts) {  // dense cell
      a.core_s[j] = 1;
      atomicAdd(a.core_cnt + cell, 1u);
      continue;
    }
    const uint2 pv = S.pts[i];
    const uint32_t p[3] = {pv.x & 0xffffu, pv.x >> 16, pv.y};
    // its sub-cell: offsets inside the cell (halo coordinates hx, hy, hz)
    uint32_t sub = 0;
    {
      const uint32_t hxyz[3] = {(uint32_t)cc / BRK_H, (uint32_t)cc % BRK_H, (uint32_t)hz};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint32_t o = p[k] - hxyz[k] * a.g.s;
        sub = sub * BRK_SUB + (o >= cols.thr[0]) + (o >= cols.thr[1]) + (o >= cols.thr[2]);
      }
    }
    // (32-bit shared-memory addresses: no 64-bit pointer arithmetic per window)
    const uint32_t base = smem_addr(abs_flat + cc * (BRK_H + 1) + hz);
#ifdef DB_COUNT_WORK
    {  // Alg 2's work: the tests of the cell-level stencil walk,
       // nearest column first, stopping at minPts (what slot 0 counts on the
       // other MarkCore paths)
      uint32_t alg2 = 0, cnt = 0;
      for (int k = 0; k < cols.ncols && cnt < need; ++k)
        for (uint32_t u = lds_u16(base + cols.A[k]), ue = lds_u16(base + cols.B[k]); u < ue && cnt < need; ++u) {
          cnt += brick_within(p, S.pts[u], eps2) ? 1u : 0u;
          ++alg2;
        }
      DB_WORK_N(3, alg2);
    }
#endif
    // phase A: the non-empty windows of the sub-cell's stencil, nearest first
    // (table rows are padded with empty windows to nwmax: no per-lane trip count)
    const uint32_t L = smem_addr(&S.list[0][threadIdx.x]);
    uint32_t Lw = L;
    const uint32_t tw = smem_addr(&S.tab.w[sub][0]);
#pragma unroll
    for (int k = 0; k < BRK_MAXC; ++k) {
      if (k < cols.nwmax) {
        const uint32_t e = lds_u16(tw + 2 * k);
        const uint32_t wa = base + (e & 0xfffu) - 2048u;
        const uint32_t lo = lds_u16(wa), hi = lds_u16(wa + (e >> 12));
        if (lo < hi) {
          sts_u32(Lw, __byte_perm(lo, hi, 0x5410));  // lo | hi << 16
          Lw += 4 * BRK_THREADS;
        }
      }
    }
    const uint32_t Lend = Lw;
    // phase B: every step tests one candidate (the own window is never empty)
    uint32_t count = 0, u = 0, u1 = 0, Lr = L;
    for (;;) {
      if (u >= u1) {
        if (Lr == Lend) break;
        const uint32_t w = lds_u32(Lr);
        Lr += 4 * BRK_THREADS;
        u = w & 0xffffu;
        u1 = w >> 16;
      }
      DB_WORK(0);
      count += brick_within(p, S.pts[u], eps2) ? 1u : 0u;
      ++u;
      if (count >= need) break;
    }
    a.core_s[j] = count >= need;
    if (count >= need) atomicAdd(a.core_cnt + cell, 1u);
  }
}

// Thread per cell: core count (a7); mixed cells are listed for the partition.
constexpr int SC_CELLS = 8;  // consecutive cells per thread in sp_cells (fewer blocks, fewer atomics)

// counted (after the brick kernel): core_cnt already holds the counts unless a
// brick overflowed (its points went to the thread kernel)
__global__ void __launch_bounds__(256) sp_cells_kernel(SpArgs a, const uint32_t* counted) {
  const bool have = counted && *counted == 0;
  const uint32_t g0 = (blockIdx.x * blockDim.x + threadIdx.x) * SC_CELLS;
  uint32_t ncc = 0, nmx = 0, kpts = 0;
  uint8_t flags[SC_CELLS];  // bit 0 core cell, bit 1 mixed
#pragma unroll
  for (int q = 0; q < SC_CELLS; ++q) {
    const uint32_t g = g0 + q;
    flags[q] = 0;
    if (g < a.ncells) {
      const uint32_t s = a.cell_start[g], e = a.cell_start[g + 1], m = e - s;
      uint32_t k = 0;
      if ((int64_t)m >= a.min_pts) k = m;
      else if (have) k = a.core_cnt[g];
      else
        for (uint32_t u = s; u < e; ++u) k += a.core_s[u];
      if (!have) a.core_cnt[g] = k;
      flags[q] = (k > 0 ? 1 : 0) | (k > 0 && k < m ? 2 : 0);
      ncc += k > 0;
      nmx += k > 0 && k < m;
      kpts += k;
    }
  }
  // one 64-bit block scan for three block totals: core cells (bits 0-15),
  // mixed cells (16-31) and core points (32-63); core cells (unordered, for
  // the core directory) and mixed cells (for the partition) are appended
  // with one 64-bit atomic per block for core cells + core points (same-
  // address atomics from many blocks serialise) and one for mixed cells
  __shared__ uint64_t s_scan[33];
  __shared__ uint32_t s_base, s_cbase;
  uint64_t tot;
  const uint64_t ex = block_exclusive_scan<uint64_t>(
      (uint64_t)ncc | ((uint64_t)nmx << 16) | ((uint64_t)kpts << 32), s_scan, &tot);
  if (threadIdx.x == 0) {
    const uint64_t nc = tot & 0xffffu, nm = (tot >> 16) & 0xffffu;
    if (nc) s_cbase = (uint32_t)atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 4),
                                          (unsigned long long)(nc | ((tot >> 32) << 32)));
    if (nm) s_base = atomicAdd(a.counters + 3, (uint32_t)nm);
  }
  __syncthreads();
  uint32_t pc = s_cbase + (uint32_t)(ex & 0xffffu), pm = s_base + (uint32_t)((ex >> 16) & 0xffffu);
#pragma unroll
  for (int q = 0; q < SC_CELLS; ++q) {
    if (flags[q] & 1) a.core_tmp[pc++] = g0 + q;
    if (flags[q] & 2) a.mixed_list[pm++] = g0 + q;
  }
}

// ---------------------------------------------------------- ClusterCore (a8)
// Over the core cells (core_list, linear order): a warp takes 32 of them and
// its lanes run over the (core cell g, back column) items; each probes the
// core directory and tests the core cells h found (h < g in linear order:
// every pair once):
//  * small pairs (|A| |B| <= SP_SMALL core points; ~1x1 on sparse lattices):
//    the BCP test itself is cheaper than the two Finds that could prune it,
//    so it runs directly (early exit at the first pair within eps,
//    P:L642-644) and Links on success;
//  * larger pairs are skipped if Find(g) == Find(h) and queued
//    for the warp BCP kernel (cluster.cu), which re-checks Find first.
// APX: the rho-approximate connectivity test (row f4), a separate
// instantiation so that the exact kernel keeps its register budget.
// Two launches: back columns [0, nbnear) (gap 0: the pairs most likely to
// connect, tested directly), then the rest with Find first — on data where
// most cells join one component the second pass is pruned almost entirely
// instead of testing and linking every pair against one contended root.
template <int DIM, int D, bool WIDE, bool BY_CELLS, bool APX>
__global__ void __launch_bounds__(256) sp_pairs_kernel(SpArgs a, unsigned long long* tested, int col_lo,
                                                       int col_hi, bool find_first) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];

  const int nb = col_hi - col_lo;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    s_off[i] = a.bcoff[col_lo + i];
    s_mask[i] = a.bcmask[col_lo + i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t mine = 0;
  // BY_CELLS: chunks of 32 consecutive cells, the core ones found by a ballot;
  // else chunks of 32 consecutive core cells from core_list
  const uint32_t limit = BY_CELLS ? a.ncells : a.ncore;
  for (uint32_t r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; r0 < limit; r0 += nwarps * 32) {
    uint32_t cm = 0xffffffffu, k;
    if (BY_CELLS) {
      const uint32_t gl = r0 + lane;
      cm = __ballot_sync(DB_FULL, gl < a.ncells && a.core_cnt[gl] > 0);
      k = __popc(cm);
    } else {
      k = min(32u, a.ncore - r0);
    }
    const uint32_t items = k * (uint32_t)nb;
    // warp-uniform rounds of 32 items, reconverged after each: left to
    // independent thread scheduling the lanes drift apart over their runs and
    // the h loop issued with ~3 of 32 lanes active (ncu, uniform-3d eps=1000)
    for (uint32_t it0 = 0; it0 < items; it0 += 32) {
      __syncwarp();
      const uint32_t it = it0 + lane;
      if (it >= items) continue;
      const uint32_t ci = it / nb, col = it - ci * nb;
      const uint32_t g = BY_CELLS ? r0 + (uint32_t)__fns(cm, 0, ci + 1) : a.core_list[r0 + ci];
      const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
      uint32_t id0;
      const uint32_t nc = dir_probe(a.cdir, base + (uint64_t)s_off[col], s_mask[col], &id0);
      if (!nc) continue;
      const uint32_t kg = a.core_cnt[g], sg = a.cell_start[g];
      for (uint32_t r = id0; r < id0 + nc; ++r) {
        const uint32_t h = a.core_list[r];
        const uint32_t kh = a.core_cnt[h];
        if (find_first && uf_same_hop(a.parent, g, h)) continue;
        if (APX && apx_cells_within(a.cell_key[g], a.cell_key[h], a.g)) {
          uf_link(a.parent, g, h);  // (rho-approximate: no point test needed)
          continue;
        }
        if ((uint64_t)kg * kh > SP_SMALL) {
          if (uf_find(a.parent, g) == uf_find(a.parent, h)) continue;
          const uint32_t slot = atomicAdd(a.counters + 2, 1u);
          if (slot < a.large_cap) { a.large[slot] = make_uint2(g, h); continue; }
          // list full: test the pair here (correct, only slower)
        }
        ++mine;
        const uint32_t sh = a.cell_start[h];
        bool hit = false;
        for (uint32_t u = sg; u < sg + kg && !hit; ++u) {
          int32_t p[D];
          load_pt<D>(a.Ps, u, p);
          for (uint32_t v = sh; v < sh + kh; ++v) {
            int32_t q[D];
            load_pt<D>(a.Ps, v, q);
            DB_WORK(1);
            if (APX ? connect_test<D, WIDE>(p, q, a.g) : within_dim<DIM, D, WIDE>(p, q, a.g)) {
              hit = true;
              break;
            }
          }
        }
        if (hit) uf_link(a.parent, g, h);
      }
    }
  }
  block_add_u64(mine, tested);
}

// Core points packed in core_list order (cells with core points in linear
// order): the core points of the core cells found by one probe of the core
// directory (ranks id0 .. id0 + nc) are one contiguous range of cpts, so a
// pair search reads no per-cell tables for the cells it finds.
template <int D>
__global__ void sp_core_pack_kernel(SpArgs a, int4* __restrict__ cpts) {
  // a warp per 32 core cells, lanes over their core points
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; r0 < a.ncore; r0 += nwarps * 32) {
    const uint32_t r1 = min(r0 + 32, a.ncore);
    const uint32_t q0 = a.cpre[r0], q1 = a.cpre[r1];
    for (uint32_t q = q0 + lane; q < q1; q += 32) {
      // its cell: the last rank in r0 .. r1 whose start is <= q
      uint32_t r = r0;
#pragma unroll
      for (int step = 16; step; step >>= 1)
        if (r + step < r1 && a.cpre[r + step] <= q) r += step;
      const uint32_t h = a.core_list[r];
      int32_t p[D];
      load_pt<D>(a.Ps, a.cell_start[h] + (q - a.cpre[r]), p);
      cpts[q] = make_int4(p[0], p[1], D > 2 ? p[2] : 0, (int32_t)h);
    }
  }
}

// ClusterCore on the packed core points (one pass over the back columns, no
// Find filter; Alg 3): the lanes of a warp take (core cell g,
// back column) items; a probe of the core directory gives the core cells of
// the column run and, through cpre, their core points as one range; each is
// tested against g's core points and a hit links g with the point's cell
// (pairs are seen once, from the higher id, as in sp_pairs_kernel). Pairs
// with more than SP_SMALL point pairs go to the warp BCP as before.
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_pairs_cp_kernel(SpArgs a, unsigned long long* tested) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  const int nb = a.nbcols;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    s_off[i] = a.bcoff[i];
    s_mask[i] = a.bcmask[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t mine = 0;
  for (uint32_t r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; r0 < a.ncore; r0 += nwarps * 32) {
    const uint32_t k = min(32u, a.ncore - r0);
    const uint32_t items = k * (uint32_t)nb;
    for (uint32_t it0 = 0; it0 < items; it0 += 32) {
      __syncwarp();
      const uint32_t it = it0 + lane;
      if (it >= items) continue;
      const uint32_t ci = it / nb, col = it - ci * nb;
      const uint32_t r = r0 + ci;
      uint32_t id0;
      const uint32_t nc = dir_probe(a.cdir, a.clin[r] + (uint64_t)s_off[col], s_mask[col], &id0);
      if (!nc) continue;
      const uint32_t g = a.core_list[r];
      const uint32_t pb = a.cpre[r], pe = a.cpre[r + 1];
      const uint32_t qb = a.cpre[id0], qe = a.cpre[id0 + nc];
      if ((uint64_t)(pe - pb) * (qe - qb) <= SP_SMALL) {
        uint32_t last = MISS;  // (the cell linked last: its other points need no test)
        for (uint32_t q = qb; q < qe; ++q) {
          const int4 qv = __ldg(a.cpts + q);
          if ((uint32_t)qv.w == last) continue;
          const int32_t qq[4] = {qv.x, qv.y, qv.z, 0};
          ++mine;
          for (uint32_t u = pb; u < pe; ++u) {
            const int4 pv = __ldg(a.cpts + u);
            const int32_t pp[4] = {pv.x, pv.y, pv.z, 0};
            DB_WORK(1);
            if (within_dim<DIM, 4, WIDE>(pp, qq, a.g)) {
              uf_link(a.parent, g, (uint32_t)qv.w);
              last = (uint32_t)qv.w;
              break;
            }
          }
        }
        continue;
      }
      // larger: per found cell, as sp_pairs_kernel (big pairs to the warp BCP)
      const uint32_t kg = pe - pb;
      for (uint32_t rr = id0; rr < id0 + nc; ++rr) {
        const uint32_t h = a.core_list[rr];
        const uint32_t hb = a.cpre[rr], he = a.cpre[rr + 1];
        if ((uint64_t)kg * (he - hb) > SP_SMALL) {
          if (uf_find(a.parent, g) == uf_find(a.parent, h)) continue;
          const uint32_t slot = atomicAdd(a.counters + 2, 1u);
          if (slot < a.large_cap) { a.large[slot] = make_uint2(g, h); continue; }
        }
        ++mine;
        bool hit = false;
        for (uint32_t u = pb; u < pe && !hit; ++u) {
          const int4 pv = __ldg(a.cpts + u);
          const int32_t pp[4] = {pv.x, pv.y, pv.z, 0};
          for (uint32_t v = hb; v < he; ++v) {
            const int4 qv = __ldg(a.cpts + v);
            const int32_t qq[4] = {qv.x, qv.y, qv.z, 0};
            DB_WORK(1);
            if (within_dim<DIM, 4, WIDE>(pp, qq, a.g)) { hit = true; break; }
          }
        }
        if (hit) uf_link(a.parent, g, h);
      }
    }
  }
  block_add_u64(mine, tested);
}

// --------------------------------------------------------- ClusterBorder (a10)
// Does core cell h hold a core point within eps of p? Core points are first in
// their cell (a7), so they are Ps[cell_start[h] .. + core_cnt[h]).
template <int DIM, int D, bool WIDE>
__device__ __forceinline__ bool sp_core_within(const SpArgs& a, const int32_t* p, uint32_t h) {
  const uint32_t sh = a.cell_start[h], kh = a.core_cnt[h];
  for (uint32_t v = sh; v < sh + kh; ++v) {
    int32_t q[D];
    load_pt<D>(a.Ps, v, q);
    DB_WORK(2);
    if (within_dim<DIM, D, WIDE>(p, q, a.g)) return true;
  }
  return false;
}

// Smallest label > `after` among clusters with a core point within eps of p
// (storage-free enumeration for points with more than SP_MAXL labels).
template <int DIM, int D, bool WIDE>
__device__ uint32_t sp_next_label(const SpArgs& a, const long long* s_off, const uint32_t* s_mask,
                                  const int32_t* p, uint32_t g, uint64_t base, int64_t after) {
  uint32_t best = MISS;
  for (int c = 0; c < a.ncols; ++c) {
    uint32_t id0;
    const uint32_t nc = dir_probe(a.cdir, base + (uint64_t)s_off[c], s_mask[c], &id0);
    for (uint32_t r = id0; r < id0 + nc; ++r) {
      const uint32_t h = a.core_list[r];
      const uint32_t lab = a.cell_label[h];
      if ((int64_t)lab <= after || lab >= best) continue;
      if (h == g || sp_core_within<DIM, D, WIDE>(a, p, h)) best = lab;
    }
  }
  return best;
}

// tmp_n[j] |= v with a 32-bit atomic on the word holding the byte; returns the
// byte's previous value. (0xff | 1 = 0xff: an overflow flag is never undone.)
__device__ __forceinline__ uint32_t flag_or(uint8_t* tmp_n, uint32_t j, uint32_t v) {
  uint32_t* w = reinterpret_cast<uint32_t*>(tmp_n + (j & ~3u));
  const uint32_t sh = (j & 3u) * 8u;
  return (atomicOr(w, v << sh) >> sh) & 255u;
}

// A label set passed SP_MAXL labels: flag it (first flagger lists it for the
// enumeration kernel, which then writes its exact count).
__device__ __forceinline__ void flag_overflow(const SpArgs& a, uint32_t j) {
  if (flag_or(a.tmp_n, j, 0xffu) != 0xffu) a.ovf_list[atomicAdd(a.ovf_count, 1u)] = j;
}

// Point-centric ClusterBorder, for lattices where almost every point is core
// (few non-core points, millions of core cells): a thread per non-core point
// walks the stencil columns on the core directory, tests the core points of
// each core cell found whose label it does not hold yet, and writes its label
// set (ascending order is the fill's job) with no atomics — one thread owns
// the row. More than SP_MAXL labels: flagged, enumerated later.
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256, 4) sp_border_point_kernel(SpArgs a) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  for (int i = threadIdx.x; i < a.ncols; i += blockDim.x) { s_off[i] = a.coff[i]; s_mask[i] = a.cmask[i]; }
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n || a.core_s[j]) return;
  const uint32_t g = a.cell_of[j];
  const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
  int32_t p[D];
  load_pt<D>(a.Ps, j, p);
  uint32_t L[SP_MAXL];
#pragma unroll
  for (int k = 0; k < SP_MAXL; ++k) L[k] = MISS;
  int nl = 0;
  bool ovf = false;
  for (int c = 0; c < a.ncols && !ovf; ++c) {
    uint32_t id0;
    const uint32_t nc = dir_probe(a.cdir, base + (uint64_t)s_off[c], s_mask[c], &id0);
    for (uint32_t r = id0; r < id0 + nc && !ovf; ++r) {
      const uint32_t h = a.core_list[r];
      const uint32_t lab = a.cell_label[h];
      bool have = false;
#pragma unroll
      for (int k = 0; k < SP_MAXL; ++k) have |= L[k] == lab;
      if (have || !sp_core_within<DIM, D, WIDE>(a, p, h)) continue;
      if (nl == SP_MAXL) { ovf = true; break; }
#pragma unroll
      for (int k = 0; k < SP_MAXL; ++k)
        if (k == nl) L[k] = lab;
      ++nl;
    }
  }
  if (ovf) {  // (counted as a border point below; its count comes from the enumeration)
    flag_overflow(a, j);
  } else if (nl) {
    *reinterpret_cast<uint4*>(a.tmp_lab + (size_t)j * SP_MAXL) = make_uint4(L[0], L[1], L[2], L[3]);
    a.tmp_n[j] = 1;
    a.bcnt[a.idx[j]] = (uint32_t)nl;
  }
  if (ovf || nl) atomicAdd(a.nborder, 1ull);
}

// Core-centric ClusterBorder. Alg 4 asks, for every non-core point p, which
// clusters have a core point within eps of p. On a sparse
// lattice most stencil cells of p hold no core point (c5: 8% of points are
// core), so the search runs from the other side: a warp per core cell h.
// Lane k probes stencil column k on the directory of all cells; a warp scan
// of the column sizes lays the candidate points out flat, and the lanes take
// them 32 at a time (lane -> column by a shuffle search), so the lanes stay
// busy whatever the column sizes. Every non-core candidate p is tested
// against h's core points; on a hit label(h) joins p's label set, a
// lock-free set of SP_MAXL slots (atomicCAS into the first slot that is
// empty or already holds the label; slots fill in order, so a label appears
// once). A point whose set overflows is flagged and enumerated later without
// storage (sp_next_label). "Core point within eps" is symmetric, so both
// sides find the same pairs; p's own cell is h's centre column (same cell =>
// within eps, the test passes).
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_border_emit_kernel(SpArgs a) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  for (int i = threadIdx.x; i < a.ncols; i += blockDim.x) { s_off[i] = a.coff[i]; s_mask[i] = a.cmask[i]; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  uint32_t nb = 0;  // border points found first by this thread
  for (uint32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < a.ncore; r += nwarps) {
    const uint32_t h = a.core_list[r];
    const uint64_t base = cell_lin<DIM>(a.cell_key[h], a);
    const uint32_t sh = a.cell_start[h], kh = a.core_cnt[h];
    const uint32_t lab = a.cell_label[h];
    uint32_t lo = 0, len = 0;
    if (lane < a.ncols) {
      uint32_t id0;
      const uint32_t nc = dir_probe(a.dir, base + (uint64_t)s_off[lane], s_mask[lane], &id0);
      if (nc) {
        lo = a.cell_start[id0];
        len = a.cell_start[id0 + nc] - lo;
      }
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(DB_FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t total = __shfl_sync(DB_FULL, incl, 31);
    const uint32_t excl = incl - len;
    for (uint32_t t0 = 0; t0 < total; t0 += 32) {
      const uint32_t t = t0 + lane;
      // column of candidate t: the last lane whose exclusive start is <= t
      int k = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const uint32_t e = __shfl_sync(DB_FULL, excl, k + step);
        if (e <= t) k += step;
      }
      const uint32_t u = __shfl_sync(DB_FULL, lo, k) + t - __shfl_sync(DB_FULL, excl, k);
      if (t >= total || a.core_s[u]) continue;
      int32_t p[D];
      load_pt<D>(a.Ps, u, p);
      const uint32_t iu = __ldg(a.idx + u);  // (issued with the point: no wait after the CAS)
      bool hit = false;
      for (uint32_t v = sh; v < sh + kh && !hit; ++v) {
        int32_t q[D];
        load_pt<D>(a.Ps, v, q);
        DB_WORK(2);
        hit = within_dim<DIM, D, WIDE>(p, q, a.g);
      }
      if (!hit) continue;
      // label sets by sorted position: the candidates of one core cell lie in
      // its neighbouring columns, so the atomics of a warp hit nearby lines
      uint32_t* L = a.tmp_lab + (size_t)u * SP_MAXL;
      // slots fill in order, so a label appears once; the thread that fills
      // slot s adds one to the point's count (input order) and, for slot 0,
      // marks it as a border point
      bool placed = false;
#pragma unroll
      for (int s = 0; s < SP_MAXL; ++s) {
        const uint32_t old = atomicCAS(L + s, MISS, lab);
        if (old == MISS) {
          if (s == 0) {
            flag_or(a.tmp_n, u, 1u);
            ++nb;
          }
          atomicAdd(a.bcnt + iu, 1u);
        }
        if (old == MISS || old == lab) { placed = true; break; }
      }
      if (!placed) flag_overflow(a, u);  // more than SP_MAXL labels: enumerated later
    }
  }
  block_add_u64(nb, a.nborder);
}

// Overflowed label sets (more than SP_MAXL labels; ovf_list): their exact
// size by storage-free enumeration, written to the point's input index.
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256, 4) sp_border_ovf_kernel(SpArgs a) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  for (int k = threadIdx.x; k < a.ncols; k += blockDim.x) { s_off[k] = a.coff[k]; s_mask[k] = a.cmask[k]; }
  __syncthreads();
  const uint32_t m = *a.ovf_count;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
    const uint32_t j = a.ovf_list[t];
    const uint32_t g = a.cell_of[j];
    const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
    int32_t p[D];
    load_pt<D>(a.Ps, j, p);
    uint32_t cnt = 0;
    int64_t after = -1;
    while (true) {
      const uint32_t nx = sp_next_label<DIM, D, WIDE>(a, s_off, s_mask, p, g, base, after);
      if (nx == MISS) break;
      ++cnt;
      after = nx;
    }
    a.bcnt[a.idx[j]] = cnt;
  }
}

// Thread per sorted position: the point's row of the CSR (at its input
// index), the set sorted by a 4-input network (unused slots are ~0 and sort
// last), or the enumeration for an overflowed set.
template <int DIM, int D, bool WIDE>
__global__ void __launch_bounds__(256) sp_border_fill_kernel(SpArgs a, const int64_t* __restrict__ border_off,
                                                             int32_t* __restrict__ border_ids) {
  __shared__ long long s_off[SP_MAX_COLS];
  __shared__ uint32_t s_mask[SP_MAX_COLS];
  for (int k = threadIdx.x; k < a.ncols; k += blockDim.x) { s_off[k] = a.coff[k]; s_mask[k] = a.cmask[k]; }
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  const uint32_t f = a.tmp_n[j];
  if (!f) return;  // no label (core and noise points)
  const bool ovf = f == 0xffu;
  uint4 v = make_uint4(MISS, MISS, MISS, MISS);
  if (!ovf) v = *reinterpret_cast<const uint4*>(a.tmp_lab + (size_t)j * SP_MAXL);
  const int64_t o = border_off[a.idx[j]];
  if (!ovf) {
    auto cs = [](uint32_t& x, uint32_t& y) { const uint32_t lo = min(x, y), hi = max(x, y); x = lo; y = hi; };
    cs(v.x, v.y); cs(v.z, v.w); cs(v.x, v.z); cs(v.y, v.w); cs(v.y, v.z);
    const uint32_t L[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (L[q] != MISS) border_ids[o + q] = (int32_t)L[q];
    return;
  }
  const uint32_t g = a.cell_of[j];
  const uint64_t base = cell_lin<DIM>(a.cell_key[g], a);
  int32_t p[D];
  load_pt<D>(a.Ps, j, p);
  int64_t after = -1, w = 0;
  while (true) {
    const uint32_t nx = sp_next_label<DIM, D, WIDE>(a, s_off, s_mask, p, g, base, after);
    if (nx == MISS) break;
    border_ids[o + w++] = (int32_t)nx;
    after = nx;
  }
}

// ----------------------------------------------------------------- host
template <typename F>
static void by_dim_sp(int d, bool wide, F&& f) {
  auto w = [&](auto Dm, auto Dp) {
    if (wide) f(Dm, Dp, std::true_type());
    else f(Dm, Dp, std::false_type());
  };
  if (d == 1) w(std::integral_constant<int, 1>(), std::integral_constant<int, 2>());
  else if (d == 2) w(std::integral_constant<int, 2>(), std::integral_constant<int, 2>());
  else w(std::integral_constant<int, 3>(), std::integral_constant<int, 4>());
}

static unsigned __int128 padded_volume(const Geo& g) {
  unsigned __int128 vol = 1;
  for (int k = 0; k < g.d; ++k) vol *= (unsigned __int128)g.maxc[k] + 1 + 2 * (unsigned __int128)g.R;
  return vol;
}

// Stencil columns: the offsets (and self) grouped by all but
// the last axis; each group is |delta_last| <= m, one column of width 2m + 1.
// Returns {squared gap of the prefix, {start offset, mask}} nearest first;
// *back gets the columns of cells before the centre in linear order.
typedef std::vector<std::pair<unsigned __int128, std::pair<long long, uint32_t>>> Cols;
static Cols stencil_columns(const Geo& g, const uint64_t* stride, Cols* back,
                            std::vector<int8_t>* geom = nullptr /* dx, dy, mz per column (d = 3) */) {
  const std::vector<int8_t> offs = stencil_offsets(g);
  const int noffs = (int)(offs.size() / g.d);
  std::map<std::vector<int>, int> colm;
  colm[std::vector<int>(g.d > 1 ? g.d - 1 : 0, 0)] = 0;
  for (int t = 0; t < noffs; ++t) {
    std::vector<int> pfx(offs.begin() + (size_t)t * g.d, offs.begin() + (size_t)t * g.d + g.d - 1);
    const int v = offs[(size_t)t * g.d + g.d - 1];
    int& mm = colm[pfx];
    mm = std::max(mm, v < 0 ? -v : v);
  }
  Cols cols;
  std::vector<std::pair<unsigned __int128, std::array<int8_t, 3>>> gg3;
  back->clear();
  for (auto& [pfx, mm] : colm) {
    int first = 0;  // sign of the first non-zero prefix component
    for (int v : pfx)
      if (v) { first = v < 0 ? -1 : 1; break; }
    unsigned __int128 gap = 0;
    long long off = -(long long)mm;
    for (int k = 0; k + 1 < g.d; ++k) {
      const int v = pfx[k] < 0 ? -pfx[k] : pfx[k];
      if (v) { const unsigned __int128 gg = (unsigned __int128)(v - 1) * g.s + 1; gap += gg * gg; }
      off += (long long)pfx[k] * (long long)stride[k];
    }
    const uint32_t full = (uint32_t)((1ull << (2 * mm + 1)) - 1);
    cols.push_back({gap, {off, full}});
    if (g.d == 3) gg3.push_back({gap, {(int8_t)pfx[0], (int8_t)pfx[1], (int8_t)mm}});
    if (first < 0) back->push_back({gap, {off, full}});
    else if (first == 0 && mm > 0) back->push_back({gap, {off, (uint32_t)((1ull << mm) - 1)}});
  }
  auto by_gap = [](const auto& x, const auto& y) { return x.first < y.first; };
  std::stable_sort(cols.begin(), cols.end(), by_gap);
  std::stable_sort(back->begin(), back->end(), by_gap);
  if (geom) {
    std::stable_sort(gg3.begin(), gg3.end(), by_gap);
    geom->clear();
    for (auto& e : gg3) geom->insert(geom->end(), e.second.begin(), e.second.end());
  }
  return cols;
}

// Sub-cell stencils of the brick kernel (d = 3, R = 2): sub-interval j of
// an axis holds the cell offsets [t_j, t_{j+1}) with t_0 = 0, t_j = j s /
// BRK_SUB, t_BRK_SUB = s (s < BRK_SUB: one sub-interval, thresholds s). A
// cell at lattice delta v along an axis is at gap v s - (t_{j+1} - 1) (v > 0),
// t_j - (v s + s - 1) (v < 0), 0 (v = 0) from the sub-interval: the distance
// between their closest integer coordinates. Windows keep the cells with
// sum of squared gaps <= eps^2, per column one z-run (the condition is convex
// in v), ordered by the column's lateral gap.
// Rows are padded with empty windows (A = 0, span 0); returns the longest row.
static int brick_tables(const Geo& g, uint32_t thr[3], BrickTab* tab) {
  int nwmax = 0;
  const int64_t s = g.s;
  const int nsub = s >= BRK_SUB ? BRK_SUB : 1;
  int64_t t[BRK_SUB + 1];
  for (int j = 0; j <= BRK_SUB; ++j) t[j] = j < nsub ? j * s / nsub : s;
  for (int j = 0; j < 3; ++j) thr[j] = (uint32_t)t[j + 1];
  auto gap = [&](int j, int v) -> int64_t {
    if (v > 0) return v * s - (t[j + 1] - 1);
    if (v < 0) return t[j] - (v * s + s - 1);
    return 0;
  };
  const int R = BRK_R;
  for (int jx = 0; jx < BRK_SUB; ++jx)
    for (int jy = 0; jy < BRK_SUB; ++jy)
      for (int jz = 0; jz < BRK_SUB; ++jz) {
        const int o = (jx * BRK_SUB + jy) * BRK_SUB + jz;
        std::vector<std::pair<uint64_t, uint16_t>> ws;
        if (jx < nsub && jy < nsub && jz < nsub) {
          for (int dx = -R; dx <= R; ++dx)
            for (int dy = -R; dy <= R; ++dy) {
              const uint64_t gx = (uint64_t)gap(jx, dx), gy = (uint64_t)gap(jy, dy);
              const uint64_t lat = gx * gx + gy * gy;
              int zlo = 1, zhi = 0;
              for (int dz = -R; dz <= R; ++dz) {
                const uint64_t gz = (uint64_t)gap(jz, dz);
                if (lat + gz * gz <= g.eps2) { zlo = std::min(zlo, dz); zhi = std::max(zhi, dz); }
              }
              if (zlo > zhi) continue;
              const int dc = (dx * BRK_H + dy) * (BRK_H + 1);
              const int A = 2 * (dc + zlo), span = 2 * (zhi - zlo + 1);
              if (A + 2048 < 0 || A + 2048 > 0xfff || span > 15) throw Error(-4, "brick_tables: entry out of range");
              ws.push_back({lat, (uint16_t)((A + 2048) | (span << 12))});
            }
          std::stable_sort(ws.begin(), ws.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        }
        if (ws.size() > (size_t)BRK_MAXC) throw Error(-4, "brick_tables: too many windows");
        tab->nw[o] = (uint8_t)ws.size();
        nwmax = std::max(nwmax, (int)ws.size());
        for (int k = 0; k < BRK_MAXC; ++k) tab->w[o][k] = k < (int)ws.size() ? ws[k].second : (uint16_t)2048;
      }
  return nwmax;
}

bool sparse_applicable(const Geo& g, int64_t n, uint32_t ncells, bool forced) {
  if (g.d > 3) return false;
  // 4 bits per lattice cell (two directories of 16 B per 32 cells): keep them
  // within ~64 bytes per point
  if (padded_volume(g) > (unsigned __int128)128 * n + (1u << 24)) return false;
  uint64_t stride[3] = {0, 0, 0};
  unsigned __int128 vol = 1;
  for (int k = g.d - 1; k >= 0; --k) {
    stride[k] = (uint64_t)vol;
    vol *= (unsigned __int128)g.maxc[k] + 1 + 2 * (unsigned __int128)g.R;
  }
  Cols back;
  if (stencil_columns(g, stride, &back).size() > (size_t)SP_MAX_COLS) return false;
  if (forced) return true;
  return (uint64_t)n <= (uint64_t)SPARSE_MEAN_PER_CELL * ncells;
}

// Build a directory over the padded lattice for every cell (list = NULL) or
// the cells list[0 .. *count).
static uint4* build_dir(Ctx& c, const SpArgs& a, uint64_t words, const uint32_t* list,
                        const uint32_t* count) {
  uint32_t* bm = c.alloc<uint32_t>(words);
  uint32_t* wcnt = c.alloc<uint32_t>(words);
  uint32_t* pre = c.alloc<uint32_t>(words + 1);
  uint4* dir = c.alloc<uint4>(words);
  c.zero(bm, sizeof(uint32_t) * words);
  dir_set_kernel<<<grid_for(a.ncells, 256, c.sms * 8), 256, 0, c.st>>>(a.cell_key, a.ncells, a, list, count, bm);
  c.launched();
  popc_kernel<<<grid_for((int64_t)words, 256, 1 << 30), 256, 0, c.st>>>(bm, words, wcnt);
  c.launched();
  exclusive_scan_u32_u32(c, wcnt, pre, (int64_t)words);
  dir_pack_kernel<<<grid_for((int64_t)words, 256, 1 << 30), 256, 0, c.st>>>(bm, pre, words, dir);
  c.launched();
  return dir;
}

uint32_t sparse_pipeline(Ctx& c, const Geo& g, const CellsView& cv, int32_t* Ps, uint32_t* idx,
                         uint8_t* core_s, uint32_t* core_cnt, int64_t n, int64_t min_pts, bool wide,
                         const uint4* dir, bool brick_ok, SparseOut* o) {
  SpArgs a{};
  a.g = g;
  unsigned __int128 vol = 1;
  for (int k = g.d - 1; k >= 0; --k) {
    a.stride[k] = (uint64_t)vol;
    vol *= (unsigned __int128)g.maxc[k] + 1 + 2 * (unsigned __int128)g.R;
  }
  a.ncells = cv.ncells;
  a.cell_start = cv.cell_start;
  a.cell_key = cv.cell_key;
  a.cell_of = cv.cell_of;
  a.Ps = Ps;
  a.idx = idx;
  a.core_s = core_s;
  a.core_cnt = core_cnt;
  a.min_pts = min_pts;
  a.n = n;
  a.counters = o->counters;  // [4], zeroed by the caller
  Cols back;
  const Cols cols = stencil_columns(g, a.stride, &back);
  if ((int)cols.size() > SP_MAX_COLS) throw Error(-4, "sparse path: too many stencil columns");
  // Global MarkCore bound (Alg 2's count can never exceed the points of the
  // stencil cells, reading 13): if (stencil cells) x (largest cell) < minPts
  // no point can be core and the caller takes the all-noise exit.
  uint64_t stencil_cells = 0;
  for (auto& e : cols) stencil_cells += (uint64_t)__builtin_popcount(e.second.second);
  if (!dir && (uint64_t)min_pts > stencil_cells) {  // (the lattice sort checked it already)
    uint32_t* mx = c.alloc<uint32_t>(1);
    c.zero(mx, sizeof(uint32_t));
    cell_max_kernel<<<grid_for(cv.ncells, 256, c.sms * 8), 256, 0, c.st>>>(cv.cell_start, cv.ncells, mx);
    c.launched();
    if ((uint64_t)c.read(mx) * stencil_cells < (uint64_t)min_pts) return 0;  // no core point
  }
  auto upload = [&](const Cols& cs, const long long** off, const uint32_t** mask) {
    std::vector<long long> co;
    std::vector<uint32_t> cm;
    for (auto& e : cs) { co.push_back(e.second.first); cm.push_back(e.second.second); }
    co.push_back(0);
    cm.push_back(0);
    long long* dco = c.alloc<long long>(co.size());
    uint32_t* dcm = c.alloc<uint32_t>(cm.size());
    c.upload(dco, co.data(), co.size());
    c.upload(dcm, cm.data(), cm.size());
    *off = dco;
    *mask = dcm;
  };
  upload(cols, &a.coff, &a.cmask);
  a.ncols = (int)cols.size();
  upload(back, &a.bcoff, &a.bcmask);
  a.nbcols = (int)back.size();
  a.nbnear = 0;
  while (a.nbnear < a.nbcols && back[a.nbnear].first == 0) ++a.nbnear;
  a.nbmid = a.nbnear;
  // (columns whose lateral offsets are all within 1 have gap <= d - 1)
  while (a.nbmid < a.nbcols && back[a.nbmid].first <= (unsigned)(g.d - 1)) ++a.nbmid;
  // a4: directory of all cells
  const uint64_t words = ((uint64_t)vol + 31) / 32 + 1;
  a.dir = dir ? dir : build_dir(c, a, words, nullptr, nullptr);
  // a6: MarkCore — bricks staged in shared memory (d = 3, R = 2), else a
  // thread per point over the stencil columns (U = 2)
  c.stage(DBSCAN_STAGE_MARKCORE);
  // bricks hold BRK_CAP / BRK_H^3 = 0.30 points per halo cell: taken when the
  // mean over the lattice is at most 0.27 (denser data would overflow them:
  // at 0.27 a halo holds 2,160 points on average, sd 46)
  // ... and at least 0.15: below it most halo columns are empty and the
  // per-brick staging costs more than it saves (measured: 0.08 points per
  // cell 1.32 ms against 0.93 ms for the thread kernel; 0.23 (c5) 1.04 / 1.07)
  // (halo-relative coordinates: 3 (s BRK_H)^2 < 2^32 for exact 32-bit squares)
  o->brick = brick_ok && g.d == 3 && g.R == BRK_R && !g.at && (unsigned __int128)n * 100 <= vol * 27 &&
             (unsigned __int128)n * 20 >= vol * 3 && 3ull * ((uint64_t)g.s * BRK_H) * ((uint64_t)g.s * BRK_H) < (1ull << 32) &&
             g.eps2 < (1ull << 32);
  BrickTab tab{};
  uint32_t thr[3] = {0, 0, 0};
  if (o->brick) brick_tables(g, thr, &tab);
  if (o->brick) {
    std::vector<int8_t> geom;
    stencil_columns(g, a.stride, &back, &geom);
    BrickCols bc{};
    bc.ncols = (int)(geom.size() / 3);
    if (bc.ncols > BRK_MAXC) throw Error(-4, "sparse path: too many stencil columns for the brick kernel");
    for (int k = 0; k < bc.ncols; ++k) {
      const int dc = ((int)geom[3 * k] * BRK_H + geom[3 * k + 1]) * (BRK_H + 1), mz = geom[3 * k + 2];
      bc.A[k] = 2 * (dc - mz);
      bc.B[k] = 2 * (dc + mz + 1);
    }
    for (int k = 0; k < 3; ++k) bc.thr[k] = thr[k];
    bc.nwmax = 0;
    for (int k = 0; k < BRK_NSUB; ++k) bc.nwmax = std::max(bc.nwmax, (int32_t)tab.nw[k]);
    BrickTab* dtab = c.alloc<BrickTab>(1);
    c.upload(dtab, &tab, 1);
    const uint32_t nb[3] = {(g.maxc[0] + BRK) / BRK, (g.maxc[1] + BRK) / BRK, (g.maxc[2] + BRK) / BRK};
    const uint64_t nbricks = (uint64_t)nb[0] * nb[1] * nb[2];
    if (nbricks >= (1ull << 31)) throw Error(-4, "sparse path: brick grid too large");
    DB_CUDA(cudaMemsetAsync(core_s, 0xff, (size_t)n, c.st));
    c.zero(core_cnt, sizeof(uint32_t) * cv.ncells);  // (the brick kernel counts core points per cell)
    const size_t smem = sizeof(BrickSmem);
    by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
      constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
      constexpr bool W = decltype(Wd)::value;
      if constexpr (DIM == 3) {
        auto kern = sp_core_brick_kernel<W>;
        DB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)nbricks, BRK_THREADS, smem, c.st>>>(a, bc, dtab, nb[1], nb[2], a.counters + 1);
        c.launched();
        sp_core_kernel<DIM, D, W, 2><<<grid_for(n, 256, 1 << 30), 256, 0, c.st>>>(a, a.counters + 1);
        c.launched();
      }
    });
  } else {
    by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
      constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
      constexpr bool W = decltype(Wd)::value;
      sp_core_kernel<DIM, D, W, 2><<<grid_for(n, 256, 1 << 30), 256, 0, c.st>>>(a, nullptr);
    });
    c.launched();
  }
  // a7: core counts, core-first partition of mixed cells
  c.stage(DBSCAN_STAGE_COMPACT);
  a.mixed_list = c.alloc<uint32_t>(cv.ncells);
  a.core_tmp = c.alloc<uint32_t>(cv.ncells);
  sp_cells_kernel<<<grid_for(((int64_t)cv.ncells + SC_CELLS - 1) / SC_CELLS, 256, 1 << 30), 256, 0, c.st>>>(
      a, o->brick ? a.counters + 1 : nullptr);
  c.launched();
  partition_mixed(c, g, cv, a.mixed_list, a.counters + 3, core_cnt, Ps, idx, core_s, n);
  // directory of the cells holding core points, and their list in linear order
  a.cdir = build_dir(c, a, words, a.core_tmp, a.counters + 4);
  uint32_t* core_list = c.alloc<uint32_t>(cv.ncells);
  a.core_list = core_list;
  uint32_t* ccnt = c.alloc<uint32_t>(cv.ncells);
  uint64_t* clin = c.alloc<uint64_t>(cv.ncells);
  core_list_kernel<<<grid_for(cv.ncells, 256, c.sms * 8), 256, 0, c.st>>>(a, core_list, ccnt, clin);
  a.ccnt = ccnt;
  a.clin = clin;
  c.launched();
  const uint32_t* hc = c.fetch(a.counters, 6);  // [1] brick overflow, [4] core cells, [5] core points
  c.sync();
  a.ncore = hc[4];
  if (o->brick && hc[1]) o->brick = 2;
  const uint64_t core_pts = hc[5];
  a.ncpts = core_pts;
  // ClusterBorder from the side with less work: the non-core points when they
  // are fewer than the core cells (almost every point core), else the cells
  o->point_border = (uint64_t)n - core_pts < (uint64_t)a.ncore;
  o->stash = new SpArgs(a);
  o->core_list = core_list;
  o->ncore = a.ncore;
  return a.ncore;
}

void sparse_cluster(Ctx& c, const Geo& g, const CellsView& cv, const int32_t* Ps,
                    const uint32_t* core_cnt, bool wide, uint32_t* parent,
                    unsigned long long* tested, SparseOut* o) {
  SpArgs& a = *(SpArgs*)o->stash;
  a.parent = parent;
  a.large_cap = a.ncore + 4096;
  a.large = c.alloc<uint2>(a.large_cap);
  uf_init_list(c, parent, a.core_list, a.ncore);  // (Find and Link touch core cells only)
  if (a.nbcols > 0 && a.ncore > 0) {
    const unsigned grid = grid_for(((int64_t)cv.ncells + 31) / 32 * 32, 256, c.sms * 16);
    c.zero(a.counters + 2, sizeof(uint32_t));
    by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
      constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
      constexpr bool W = decltype(Wd)::value;
      // (two passes only when most cells hold core points: on sparse core
      // cells (c5: 8%) the second probe pass costs more than it prunes)
      // (with two: gap 0, then gap 1, then the rest, flattening in between)
      const bool two = 2ull * a.ncore >= cv.ncells;
      if (!two && !g.at && !(o->flags & DBSCAN_F_NO_PACKED_CORE)) {
        // one pass on the packed core points
        uint32_t* cpre = c.alloc<uint32_t>((size_t)a.ncore + 1);
        int4* cpts = c.alloc<int4>(std::max<uint64_t>(a.ncpts, 1));
        exclusive_scan_u32_u32(c, a.ccnt, cpre, a.ncore);  // (counts by rank: core_list_kernel)
        a.cpre = cpre;
        a.cpts = cpts;
        sp_core_pack_kernel<D><<<grid_for(((int64_t)a.ncore + 31) / 32 * 32, 256, c.sms * 16), 256, 0, c.st>>>(a, cpts);
        c.launched();
        sp_pairs_cp_kernel<DIM, D, W><<<grid_for(((int64_t)a.ncore + 31) / 32 * 32, 256, c.sms * 16), 256, 0,
                                        c.st>>>(a, tested);
        c.launched();
        o->passes = 1;
        return;
      }
      const int cut[4] = {0, two ? a.nbnear : a.nbcols, two ? a.nbmid : a.nbcols, a.nbcols};
      for (int pass = 0; pass < 3; ++pass) {
        const int lo = cut[pass], hi = cut[pass + 1];
        if (lo == hi) continue;
        if (g.at) sp_pairs_kernel<DIM, D, W, true, true><<<grid, 256, 0, c.st>>>(a, tested, lo, hi, pass > 0);
        else sp_pairs_kernel<DIM, D, W, true, false><<<grid, 256, 0, c.st>>>(a, tested, lo, hi, pass > 0);
        c.launched();
        ++o->passes;
        if (two && hi < a.nbcols) uf_flatten(c, parent, a.core_list, a.ncore);
      }
    });
    bcp_large(c, g, cv, Ps, core_cnt, parent, a.large, a.counters + 2, a.large_cap, wide);
  }
}

void sparse_border(Ctx& c, const Geo& g, const uint32_t* cell_label, const int32_t* cluster, int64_t n,
                   bool wide, int64_t* border_off, unsigned long long* nborder, SparseOut* o) {
  SpArgs& a = *(SpArgs*)o->stash;
  a.cell_label = cell_label;
  a.bcnt = c.alloc<uint32_t>(n);
  a.tmp_lab = c.alloc<uint32_t>((size_t)n * SP_MAXL);
  a.tmp_n = c.alloc<uint8_t>((size_t)n + 4);  // (+4: flag_or's 32-bit word at the end)
  a.ovf_count = c.alloc<uint32_t>(1);
  a.ovf_list = c.alloc<uint32_t>(n);
  c.zero(a.ovf_count, sizeof(uint32_t));
  a.nborder = nborder;
  // core-centric: label sets of SP_MAXL slots per point (input order), empty = ~0
  DB_CUDA(cudaMemsetAsync(a.tmp_lab, 0xff, sizeof(uint32_t) * (size_t)n * SP_MAXL, c.st));
  c.zero(a.tmp_n, (size_t)n + 4);
  c.zero(a.bcnt, sizeof(uint32_t) * (size_t)n);  // (counts are added or written for border points only)
  by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
    constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
    constexpr bool W = decltype(Wd)::value;
    if (o->point_border)
      sp_border_point_kernel<DIM, D, W><<<grid_for(n, 256, 1 << 30), 256, 0, c.st>>>(a);
    else
      sp_border_emit_kernel<DIM, D, W><<<grid_for((int64_t)a.ncore * 32, 256, c.sms * 16), 256, 0, c.st>>>(a);
    c.launched();
    sp_border_ovf_kernel<DIM, D, W><<<c.sms * 2, 256, 0, c.st>>>(a);
    c.launched();
  });
  (void)cluster;
  // (no border point at all: the scan writes zeros without reading the counts)
  exclusive_scan_u32_i64(c, a.bcnt, border_off, n, nborder);
}

void sparse_border_fill(Ctx& c, const Geo& g, bool wide, const int64_t* border_off,
                        int32_t* border_ids, SparseOut* o) {
  SpArgs& a = *(SpArgs*)o->stash;
  by_dim_sp(g.d, wide, [&](auto Dm, auto Dp, auto Wd) {
    constexpr int DIM = decltype(Dm)::value, D = decltype(Dp)::value;
    constexpr bool W = decltype(Wd)::value;
    sp_border_fill_kernel<DIM, D, W><<<grid_for(a.n, 256, 1 << 30), 256, 0, c.st>>>(a, border_off, border_ids);
  });
  c.launched();
}

void sparse_release(SparseOut* o) {
  delete (SpArgs*)o->stash;
  o->stash = nullptr;
}

}  // namespace db
