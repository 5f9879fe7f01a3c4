/*
 * dbscan.h — exact Euclidean DBSCAN for integer points on one B200 (sm_100a).
 *
 * C ABI of libdbscan_b200.so (paper_1912_06255_b200/). Plain pointers and
 * sizes only; no C++ or torch types cross this boundary.
 *
 * What it computes — PAPER.md §2 "DBSCAN Definition":
 *   a point p is CORE iff |{q in P : ||p - q|| <= eps}| >= min_pts  (p counts
 *   itself, duplicates count with multiplicity); core points joined by a chain
 *   of core points with consecutive distances <= eps form one cluster; a
 *   non-core point belongs to every cluster that has a core point within eps
 *   (BORDER), or to none (NOISE). The result is unique.
 * How — the paper's grid method, Alg 1: Cells (grid + radix sort
 *   + hash), MarkCore (Alg 2), ClusterCore with BCP
 *   tests and a lock-free union-find (Alg 3),
 *   ClusterBorder (Alg 4); neighbouring cells by stencil (d <= 3)
 *   or a cell tree (d >= 4). See DESIGN.md.
 *
 * Exactness: coordinates are int32; distances are compared squared and
 * exactly against eps^2 (readings 1-4). The output is bit-identical
 * to the CPU oracle (oracle/) and independent of scheduling.
 */
#ifndef DBSCAN_B200_H
#define DBSCAN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
#define DBSCAN_OK       0
#define DBSCAN_EINVAL  -1 /* n < 0 or n > 2^31-1; d < 1 or d > 8; eps < 1; min_pts < 1;
                             NULL pts with n > 0; NULL out; contradictory flags */
#define DBSCAN_ERANGE  -2 /* packed cell key needs > 63 bits, or d*(eps+1)^2 >= 2^62 */
#define DBSCAN_ENOMEM  -3 /* device or host allocation failed */
#define DBSCAN_ECUDA   -4 /* any other CUDA error; detail via dbscan_error_string */

/* ---- flags --------------------------------------------------------------- */
#define DBSCAN_F_DEVICE_IO     1u  /* pts and every output are DEVICE pointers; outputs the
                                      library allocates are cudaMallocAsync'd on `stream` */
#define DBSCAN_F_TIMING        2u  /* fill out->stage_ms with CUDA-event times (adds a sync) */
#define DBSCAN_F_CALLER_OUT    4u  /* out->core, out->cluster, out->border_off are caller-
                                      allocated ([n], [n], [n+1]; host or device per
                                      F_DEVICE_IO). out->border_ids may also be set, with
                                      its capacity (elements) in out->nnz: it is used when
                                      the result fits, else the library allocates one    */
#define DBSCAN_F_FORCE_STENCIL 8u  /* neighbour cells by stencil enumeration for every d */
#define DBSCAN_F_FORCE_TREE   16u  /* neighbour cells by the cell tree for every d */
#define DBSCAN_F_FORCE_WIDE   32u  /* 64-bit distance arithmetic even where 32-bit is exact */
#define DBSCAN_F_NO_WAVES     64u  /* ClusterCore in one wave (ablation of the wave schedule) */
#define DBSCAN_F_NO_SPARSE   128u  /* never take the cell-centric sparse-lattice path         */
#define DBSCAN_F_FORCE_SPARSE 256u /* take the sparse path whenever d <= 3 and the lattice
                                      directory fits (otherwise it is chosen by occupancy)   */
#define DBSCAN_F_RADIX_GROUP 512u  /* group points by cell with the LSD radix sort only (never
                                      the hash-table or lattice counting sorts)              */
#define DBSCAN_F_LATTICE_GROUP 1024u /* skip the hash counting sort: use the lattice counting
                                      sort whenever d <= 3 and its lattice fits               */
#define DBSCAN_F_COUNT_WORK  2048u /* reserved (accepted, no effect): distance tests are counted
                                      by the measurement build libdbscan_b200_count.so
                                      (`make count`), see DBSCAN_STAT_COUNTING_BUILD         */
#define DBSCAN_F_QUADTREE    4096u /* our-exact-qt: MarkCore's
                                      RangeCount on cells with >= 256 points traverses a
                                      per-cell tree instead of scanning (CSR path)           */
#define DBSCAN_F_NO_QBOUND  16384u /* never run the sub-cell lower bounds before MarkCore (row f2)  */
#define DBSCAN_F_FORCE_QBOUND 32768u /* run them whatever minPts (testing; CSR path)              */
#define DBSCAN_F_NBR_TWO_PASS 65536u /* all-pairs neighbour search (d >= 4) with a counting pass
                                      and a filling pass even where the one-pass search with
                                      candidate-capacity rows fits (testing)                  */
#define DBSCAN_F_NO_BRICK    8192u /* sparse path, d = 3: MarkCore with a thread per point
                                      instead of the shared-memory brick kernel (testing)    */
#define DBSCAN_F_NO_PACKED_CORE 131072u /* sparse path: ClusterCore's one-pass pair search on the
                                      per-cell tables instead of the packed core points
                                      (testing)                                               */

/* ---- stage timers (indices into stage_ms) -------------------------------- */
#define DBSCAN_STAGE_BBOX      0  /* a1: bounding box                                  */
#define DBSCAN_STAGE_KEYS      1  /* a1: cell keys + digit histograms                  */
#define DBSCAN_STAGE_SORT      2  /* a2: LSD radix sort of (key, index)                */
#define DBSCAN_STAGE_SEGMENT   3  /* a3: cell segmentation + point gather              */
#define DBSCAN_STAGE_HASH      4  /* a4: cell hash table (reported inside NEIGHBORS)     */
#define DBSCAN_STAGE_NEIGHBORS 5  /* a5: neighbour-cell CSR (stencil or tree)          */
#define DBSCAN_STAGE_MARKCORE  6  /* a6: MarkCore (Alg 2)                              */
#define DBSCAN_STAGE_COMPACT   7  /* a7: core-first compaction per cell                */
#define DBSCAN_STAGE_CLUSTER   8  /* a8: ClusterCore: BCP + union-find (Alg 3)         */
#define DBSCAN_STAGE_LABELS    9  /* a9: canonical labels                              */
#define DBSCAN_STAGE_BORDER   10  /* a10: ClusterBorder CSR (Alg 4)                    */
#define DBSCAN_STAGE_TOTAL    11  /* whole call on the stream                          */
#define DBSCAN_NSTAGES        12

/* ---- counters (indices into stats) --------------------------------------- */
#define DBSCAN_STAT_NCELLS        0  /* non-empty cells                                  */
#define DBSCAN_STAT_KEY_BITS      1  /* packed cell-key width                            */
#define DBSCAN_STAT_SORT_PASSES   2  /* radix passes run                                 */
#define DBSCAN_STAT_NBR_ENTRIES   3  /* neighbour CSR entries (excluding self)           */
#define DBSCAN_STAT_CORE_CELLS    4  /* cells holding >= 1 core point                     */
#define DBSCAN_STAT_PAIRS         5  /* candidate core-cell pairs (g > h)                */
#define DBSCAN_STAT_PAIRS_TESTED  6  /* pairs that reached a BCP test (not pruned by Find)*/
#define DBSCAN_STAT_LAUNCHES      7  /* kernels launched by this call                    */
#define DBSCAN_STAT_WIDE          8  /* 1 if the 64-bit distance path ran                */
#define DBSCAN_STAT_TREE          9  /* 1 if neighbour cells came from the cell tree      */
#define DBSCAN_STAT_CELL_SIDE    10  /* integer cell side s                              */
#define DBSCAN_STAT_DENSE_DIR    11  /* 1 if cells were found through a dense directory   */
#define DBSCAN_STAT_SPARSE       12  /* 1 if the cell-centric sparse-lattice path ran       */
#define DBSCAN_STAT_HASH_GROUP   13  /* grouping: 1 hash counting sort, 2 lattice counting sort,
                                        0 LSD radix sort + segmentation                      */
#define DBSCAN_STAT_MARKCORE_TESTS 14 /* distance tests of MarkCore, a6 (measurement build only) */
#define DBSCAN_STAT_QT_NODES     15  /* tree nodes built with F_QUADTREE                         */
#define DBSCAN_STAT_APPROX_SIDE  16  /* dbscan_approx: sub-cell side t of the connectivity test
                                        (0: the test is exact)                                */
#define DBSCAN_STAT_BRICK        17  /* sparse MarkCore: 1 brick kernel, 2 brick kernel with
                                        overflowed bricks taken by the thread kernel, 0 none  */
#define DBSCAN_STAT_POINT_BORDER 18  /* sparse ClusterBorder from the non-core points (1) or from
                                        the core cells (0)                                    */
#define DBSCAN_STAT_SPARSE_PASSES 19 /* sparse ClusterCore: pair-search launches over the back columns
                                        (1; 3 when most cells hold core points: gap-0 columns, then
                                        laterally adjacent ones, then the rest, flattened between) */
#define DBSCAN_STAT_BCP_TESTS    20  /* distance tests of the BCPs of ClusterCore, a8 (measurement
                                        build only)                                           */
#define DBSCAN_STAT_BORDER_TESTS 21  /* distance tests of ClusterBorder, a10 (measurement build)  */
#define DBSCAN_STAT_COUNTING_BUILD 22 /* 1 in libdbscan_b200_count.so (built with -DDB_COUNT_WORK:
                                        every distance test adds to a device counter; not
                                        thread-safe across concurrent calls, measurement only),
                                        0 in the product library                              */
#define DBSCAN_STAT_QB_DECIDED   23  /* MarkCore points proved core by the sub-cell lower bounds
                                        (row f2, minPts >= 2000 on the CSR path); -1: not run  */
#define DBSCAN_STAT_MARKCORE_ALG2 24 /* MarkCore work of Alg 2 as written: the tests of
                                        the cell-level stencil walk, nearest column first, stopping
                                        at minPts (measurement build only; equals MARKCORE_TESTS
                                        except where the brick kernel's sub-cell stencils skip
                                        candidates)                                            */
#define DBSCAN_NSTATS            32  /* (25-31 reserved) */

typedef struct dbscan_result {
  int64_t  n;
  uint8_t *core;        /* [n]   1 = core point                                          */
  int32_t *cluster;     /* [n]   core: canonical cluster id = minimum input index of a
                                 core point of its cluster; non-core: -1                 */
  int64_t *border_off;  /* [n+1] CSR over ALL points in input order; rows of core and
                                 noise points are empty; border_off[0] = 0               */
  int32_t *border_ids;  /* [nnz] each non-core point's cluster ids, ascending, distinct  */
  int64_t  nnz;         /* border_off[n]                                                  */
  int64_t  n_core, n_border, n_noise, n_clusters;
  float    stage_ms[DBSCAN_NSTAGES]; /* filled with F_TIMING, else 0                     */
  int64_t  stats[DBSCAN_NSTATS];
  uint32_t flags;       /* flags of the call that produced this result                  */
  void    *priv;        /* library bookkeeping; do not touch                             */
} dbscan_result;

/*
 * dbscan — run exact DBSCAN.
 *   pts      [n*d] int32, row-major (point i = pts[i*d .. i*d+d-1]); host or device
 *            memory per F_DEVICE_IO. Owned by the caller, read only. No alignment needed.
 *   n        number of points, 0 <= n <= 2^31-1.  n = 0 returns empty outputs.
 *   d        dimension, 1..8.
 *   eps      radius, >= 1; the predicate is  sum_k (x_k - y_k)^2 <= eps^2  (closed).
 *   min_pts  >= 1; min_pts > n makes every point noise.
 *   flags    DBSCAN_F_* bits.
 *   stream   cudaStream_t to run on (NULL = legacy default stream). The call blocks
 *            until its work on `stream` is done (with F_DEVICE_IO the outputs are then
 *            final in device memory; without it they are in host memory). It reads a
 *            few scalars back during the call (cell count, border count, ...).
 *   out      result; zeroed on entry unless F_CALLER_OUT (then core/cluster/border_off
 *            must be set by the caller). On error *out is left with every library-
 *            allocated pointer NULL and nothing leaks.
 * Ownership: the caller releases library-allocated outputs with dbscan_result_free.
 * Threads: concurrent calls on different streams (any host threads) are safe. Shared
 *   state: a mutex-protected process-wide pool of workspaces (dbscan_release_workspace),
 *   and a mutex that serialises the host-to-device input copies of concurrent host-path
 *   calls (each call computes while the next one's input is in flight).
 * Returns DBSCAN_OK or a negative code above.
 */
int dbscan(const int32_t *pts, int64_t n, int32_t d, int64_t eps, int64_t min_pts,
           uint32_t flags, void *stream, dbscan_result *out);

/*
 * dbscan_approx — rho-approximate DBSCAN (Gan and Tao; §2 P:L225-235,
 * §"Approximate DBSCAN" P:L1037-1058).
 *   Same arguments, outputs and conventions as dbscan(), plus rho > 0. Core
 *   flags and the border rule are those of DBSCAN; core points within eps are
 *   always in one cluster, core points farther apart than eps (1 + rho) are
 *   connected only through chains of closer pairs, and pairs in between may or
 *   may not be connected. Several outputs are valid; cluster ids stay canonical
 *   (minimum input index of a core point of the cluster).
 *   Connectivity test: both points snapped to sub-cells of integer side t, the
 *   largest with 2 (t-1) sqrt(d) <= eps rho, connected when the sub-cell boxes
 *   are within eps (stats[DBSCAN_STAT_APPROX_SIDE] = t; t = 1 is exact DBSCAN).
 * Returns DBSCAN_EINVAL for rho outside (0, 1e6].
 */
int dbscan_approx(const int32_t *pts, int64_t n, int32_t d, int64_t eps, int64_t min_pts, double rho,
                  uint32_t flags, void *stream, dbscan_result *out);

/* Release what the library allocated in *r (never caller-owned F_CALLER_OUT buffers).
 * Device outputs are released with cudaFreeAsync on the stream of the dbscan() call,
 * which must still exist; work queued on that stream before the free may still use
 * them. Safe on a zeroed result. */
void dbscan_result_free(dbscan_result *r);

/* A call's temporaries (device memory, 1 MB of pinned host memory, events, a
 * second stream) come from a workspace taken from a process-wide pool and
 * returned when the call ends, so calls make no allocator call per temporary and
 * concurrent calls (any threads) use different workspaces. A workspace's device
 * memory grows after a call that needed more and is kept. This frees the idle
 * workspaces (those of calls in flight are kept); later calls allocate again. */
void dbscan_release_workspace(void);

/* Static description of a code, with the detail of this thread's last error. */
const char *dbscan_error_string(int code);

/* Name of stage i (0 <= i < DBSCAN_NSTAGES) for reports. */
const char *dbscan_stage_name(int i);

/*
 * dbscan_peak_dist — U1 microbenchmark (SURVEY §2.7 `peak_dist`, §8(d)): the
 * measured throughput of the exact distance predicate ||p-q||^2 <= eps^2
 * (P:L199-202), the unit of work of MarkCore (Alg 2; O(n minPts) tests,
 * P:L1106-1121) and of the BCP (Alg 3). It is the denominator of
 * the a6/a8 roofline fractions that bench.py reports. Not part of DBSCAN.
 *   d        dimension 1..8 (candidates stored D-padded as the stage kernels do)
 *   variant  0: the shipped uint32 `__sad` predicate; 1: the shipped 64-bit
 *            clamped predicate; 2: an fp64 FMA predicate (north_star's fp64 pipe);
 *            3: the brick MarkCore's predicate on 8-byte packed rows (d = 3 only)
 *   qt       queries held in registers per thread (1, 2 or 4) against a
 *            1024-point shared-memory tile of candidates (one tile load per
 *            candidate serves qt tests)
 *   reps     passes over the tile (about 90 us each on a B200 at qt = 1)
 *   stream   cudaStream_t (NULL = legacy default); the call synchronises it
 *   out: *tests_per_s; optional *ms (CUDA-event time of the timed launch, after
 *   one untimed launch), *tests, *hits (tests that passed: about half).
 * Returns DBSCAN_OK, DBSCAN_EINVAL (bad argument) or DBSCAN_ECUDA.
 */
int dbscan_peak_dist(int32_t d, int32_t variant, int32_t qt, int64_t reps, void *stream,
                     double *tests_per_s, double *ms, int64_t *tests, int64_t *hits);

/* Library version, as 10000*major + 100*minor + patch. */
int dbscan_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DBSCAN_B200_H */
