/*
 * oracle/o1_bruteforce.c — O1: exact DBSCAN straight from the definition.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this code.
 * The product path (paper_1912_06255_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with it.
 *
 * Definition followed (§2 "DBSCAN Definition"):
 *   p is core  iff |{p_i in P : d(p, p_i) <= eps}| >= minPts
 *   core p, q share a cluster iff an eps-chain of core points joins them
 *   non-core p belongs to every cluster with a core q, d(p,q) <= eps
 *   border = non-core in >= 1 cluster; noise = non-core in none
 * Readings (DESIGN.md §"Readings"): the neighbourhood is closed (<= eps);
 * p counts itself; duplicates count with multiplicity; Euclidean distance is
 * compared squared and exactly against eps^2 in 128-bit integers (no slack);
 * a cluster is named by the minimum input index of its core points; border
 * label sets are ascending and distinct; cluster[] of a non-core point is -1.
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): hand-computed vectors
 * tests/golden/*.txt, sklearn.cluster.DBSCAN core set / core partition /
 * border-vs-noise, scipy connected components at minPts = 1, all-noise and
 * one-cluster closed forms, invariants, permutation invariance.
 *
 * Plain, slow, O(n^2): no grid, no blocking, no reordering.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;

/* squared Euclidean distance, exact for any int32 coordinates */
static i128 dist2(const int32_t *a, const int32_t *b, int d) {
  i128 s = 0;
  for (int k = 0; k < d; ++k) {
    i128 t = (i128)a[k] - (i128)b[k];
    s += t * t;
  }
  return s;
}

static void set_threads(int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
}

/* Step 1 for a subset: cnt[s] = |{j : dist2(p_sample[s], p_j) <= eps^2}| (self included). */
void o1_counts_for(const int32_t *pts, int64_t n, int32_t d, int64_t eps,
                   const int64_t *sample, int64_t k, int64_t *cnt, int threads) {
  set_threads(threads);
  const i128 e2 = (i128)eps * (i128)eps;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t s = 0; s < k; ++s) {
    const int32_t *p = pts + sample[s] * d;
    int64_t c = 0;
    for (int64_t j = 0; j < n; ++j)
      if (dist2(p, pts + j * d, d) <= e2) ++c;
    cnt[s] = c;
  }
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* Sorted distinct labels {label[q] : core[q], dist2(p, q) <= eps^2} for one p.
 * buf must hold n entries; returns the number written. */
static int64_t labels_near(const int32_t *pts, int64_t n, int32_t d, i128 e2,
                           const uint8_t *core, const int32_t *label,
                           int64_t i, int32_t *buf) {
  int64_t m = 0;
  const int32_t *p = pts + i * d;
  for (int64_t j = 0; j < n; ++j)
    if (core[j] && dist2(p, pts + j * d, d) <= e2) buf[m++] = label[j];
  qsort(buf, (size_t)m, sizeof(int32_t), cmp_i32);
  int64_t u = 0;
  for (int64_t t = 0; t < m; ++t)
    if (u == 0 || buf[u - 1] != buf[t]) buf[u++] = buf[t];
  return u;
}

/*
 * Full DBSCAN from the definition. Outputs (caller-allocated):
 *   core[n], cluster[n], border_off[n+1]; *border_ids is malloc'd here
 *   (free with o1_free). Returns 0, or -1 on allocation failure.
 */
int o1_dbscan(const int32_t *pts, int64_t n, int32_t d, int64_t eps, int64_t min_pts,
              uint8_t *core, int32_t *cluster, int64_t *border_off,
              int32_t **border_ids, int threads) {
  set_threads(threads);
  const i128 e2 = (i128)eps * (i128)eps;
  *border_ids = NULL;
  border_off[0] = 0;
  if (n == 0) return 0;

  /* Steps 1-2: neighbourhood counts and core flags. */
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int64_t j = 0; j < n; ++j)
      if (dist2(pts + i * d, pts + j * d, d) <= e2) ++c;
    core[i] = (uint8_t)(c >= min_pts);
  }

  /* Step 3: clusters of core points = eps-chains. BFS from the
   * smallest unlabelled core index, so each label is its cluster's minimum
   * core index. */
  for (int64_t i = 0; i < n; ++i) cluster[i] = -1;
  int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  if (!queue) return -1;
  for (int64_t i = 0; i < n; ++i) {
    if (!core[i] || cluster[i] != -1) continue;
    int64_t head = 0, tail = 0;
    cluster[i] = (int32_t)i;
    queue[tail++] = i;
    while (head < tail) {
      int64_t u = queue[head++];
      for (int64_t j = 0; j < n; ++j)
        if (core[j] && cluster[j] == -1 && dist2(pts + u * d, pts + j * d, d) <= e2) {
          cluster[j] = (int32_t)i;
          queue[tail++] = j;
        }
    }
  }
  free(queue);

  /* Step 4: border sets for non-core points. */
  int64_t *cnt = (int64_t *)calloc((size_t)n, sizeof(int64_t));
  if (!cnt) return -1;
#pragma omp parallel
  {
    int32_t *buf = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i)
      if (!core[i]) cnt[i] = labels_near(pts, n, d, e2, core, cluster, i, buf);
    free(buf);
  }
  for (int64_t i = 0; i < n; ++i) border_off[i + 1] = border_off[i] + cnt[i];
  int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(border_off[n] + 1));
  if (!ids) { free(cnt); return -1; }
#pragma omp parallel
  {
    int32_t *buf = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i)
      if (!core[i] && cnt[i]) {
        int64_t m = labels_near(pts, n, d, e2, core, cluster, i, buf);
        memcpy(ids + border_off[i], buf, sizeof(int32_t) * (size_t)m);
      }
    free(buf);
  }
  free(cnt);
  *border_ids = ids;
  return 0;
}

/*
 * Sampled check helper (for full-size configs the O(n^2) oracle cannot run):
 * for each sampled point s, the sorted distinct labels of core points within
 * eps, taken from the GIVEN core[] / label[] arrays (P:L211-215 applied to a
 * candidate labelling). Writes counts to cnt[k]; if ids != NULL also the
 * labels, row s starting at off[s] (caller computed from a first call).
 */
void o1_labels_near_for(const int32_t *pts, int64_t n, int32_t d, int64_t eps,
                        const uint8_t *core, const int32_t *label,
                        const int64_t *sample, int64_t k, int64_t *cnt,
                        const int64_t *off, int32_t *ids, int threads) {
  set_threads(threads);
  const i128 e2 = (i128)eps * (i128)eps;
#pragma omp parallel
  {
    int32_t *buf = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
#pragma omp for schedule(dynamic, 4)
    for (int64_t s = 0; s < k; ++s) {
      int64_t m = labels_near(pts, n, d, e2, core, label, sample[s], buf);
      cnt[s] = m;
      if (ids) memcpy(ids + off[s], buf, sizeof(int32_t) * (size_t)m);
    }
    free(buf);
  }
}

/*
 * Sampled check helper: for each sampled point s, viol[s] = the number of
 * core points q with dist2(p_s, q) <= eps^2 (closed ball) whose
 * label differs from label[sample[s]]. For a core sample this must be 0
 * (eps-adjacent core points share a cluster). Pinned negatively in
 * tests/test_oracle.py (a split cluster and an exact-eps tie both count).
 */
void o1_core_label_violations(const int32_t *pts, int64_t n, int32_t d, int64_t eps,
                              const uint8_t *core, const int32_t *label,
                              const int64_t *sample, int64_t k, int64_t *viol,
                              int threads) {
  set_threads(threads);
  const i128 e2 = (i128)eps * (i128)eps;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t s = 0; s < k; ++s) {
    int64_t i = sample[s], v = 0;
    for (int64_t j = 0; j < n; ++j)
      if (core[j] && label[j] != label[i] && dist2(pts + i * d, pts + j * d, d) <= e2) ++v;
    viol[s] = v;
  }
}

void o1_free(void *p) { free(p); }
