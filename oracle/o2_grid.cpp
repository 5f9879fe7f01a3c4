/*
 * oracle/o2_grid.cpp — O2: an independent, sequential CPU grid DBSCAN.
 *
 * TEST INFRASTRUCTURE ONLY (and the "simple CPU grid version" baseline that
 * BASELINE.json's north_star asks to be timed beside the GPU). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it. It shares no code with paper_1912_06255_b200/ and makes
 * different free choices wherever the paper leaves one open:
 *
 *   step                      paper                         O2's choice
 *   Cells (Alg 1 l.2)         side eps/sqrt(d), semisort    side s' = max(1, isqrt(floor(eps^2/d)))
 *                             + hash   std::sort of (cell tuple, index),
 *                                                           std::unordered_map of cells
 *   NeighborCells             enumerate / k-d tree          all cells within Chebyshev radius
 *                                      R' = floor(eps/s')+1: full cube
 *                                                           enumeration for d <= 3, all cell
 *                                                           pairs for d >= 4 (a superset; every
 *                                                           distance is still checked exactly)
 *   MarkCore (Alg 2)          count = |g| + sum RangeCount  same, stopping once count >= minPts
 *                                               (reading 13: output unchanged)
 *   ClusterCore (Alg 3)       Find(g) != Find(h), g > h,    same; candidate pairs visited one at a
 *                             Connected = BCP <= eps with   time in ascending lattice gap, BCP by
 *                             filter + early exit           plain double loop over the filtered
 *                                      core points (reading 12: any order)
 *   labels                    uf.Find(g)       min input index of the component's
 *                                                           core points (reading 8)
 *   ClusterBorder (Alg 4)                  same, sorted distinct label sets
 *
 * NeighborCells, MarkCore and ClusterBorder treat cells independently and are
 * spread over host threads with OpenMP (results do not depend on the order);
 * ClusterCore's union-find loop is sequential.
 * Same cell => within eps: points of one cell differ by <= s'-1 per axis, and
 * d (s'-1)^2 <= d s'^2 <= eps^2.
 * Distances are exact: squared, in 128-bit integers, against eps^2.
 * Pinned against O1 on random instances (tests/test_oracle.py).
 */
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <vector>

typedef __int128 i128;

namespace {

i128 dist2(const int32_t *a, const int32_t *b, int d) {
  i128 s = 0;
  for (int k = 0; k < d; ++k) {
    i128 t = (i128)a[k] - (i128)b[k];
    s += t * t;
  }
  return s;
}

int64_t isqrt_floor(i128 v) {  // floor(sqrt(v)) for 0 <= v < 2^126
  if (v <= 0) return 0;
  int64_t r = 0;
  for (int b = 62; b >= 0; --b) {
    int64_t c = r | ((int64_t)1 << b);
    if ((i128)c * c <= v) r = c;
  }
  return r;
}

struct UF {
  std::vector<int64_t> p;
  explicit UF(int64_t n) : p((size_t)n) { std::iota(p.begin(), p.end(), 0); }
  int64_t find(int64_t x) {
    while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
    return x;
  }
  void link(int64_t a, int64_t b) {
    a = find(a); b = find(b);
    if (a != b) p[std::max(a, b)] = std::min(a, b);
  }
};

}  // namespace

extern "C" {

/* Returns 0; -1 on allocation failure; -2 if the lattice exceeds 2^123 cells.
 * Outputs as o1_dbscan. */
int o2_dbscan(const int32_t *pts, int64_t n, int32_t d, int64_t eps, int64_t min_pts,
              uint8_t *core, int32_t *cluster, int64_t *border_off, int32_t **border_ids) {
  *border_ids = nullptr;
  border_off[0] = 0;
  if (n == 0) return 0;
  const i128 e2 = (i128)eps * eps;

  /* ---- Cells (Alg 1 line 2): side s', lattice tuple per point. ---- */
  int64_t s = isqrt_floor(e2 / d);
  if (s < 1) s = 1;
  std::vector<int64_t> lo((size_t)d), ext((size_t)d);
  for (int k = 0; k < d; ++k) {
    int64_t m = pts[k], M = pts[k];
    for (int64_t i = 1; i < n; ++i) {
      m = std::min<int64_t>(m, pts[i * d + k]);
      M = std::max<int64_t>(M, pts[i * d + k]);
    }
    lo[k] = m;
    ext[k] = (M - m) / s + 1;  // lattice extent on axis k
  }
  // mixed-radix cell id: sum_k c_k * prod_{j>k} ext_j
  typedef unsigned __int128 u128;
  {
    long double prod = 1;
    for (int k = 0; k < d; ++k) prod *= (long double)ext[k];
    if (prod >= 1e37L) return -2;  // lattice too large for a 128-bit id
  }
  auto coord = [&](int64_t i, int k) { return ((int64_t)pts[i * d + k] - lo[k]) / s; };
  auto pack = [&](const int64_t *c) {
    u128 key = 0;
    for (int k = 0; k < d; ++k) key = key * (u128)ext[k] + (u128)c[k];
    return key;
  };
  std::vector<u128> pkey((size_t)n);
  {
    std::vector<int64_t> c((size_t)d);
    for (int64_t i = 0; i < n; ++i) {
      for (int k = 0; k < d; ++k) c[k] = coord(i, k);
      pkey[i] = pack(c.data());
    }
  }
  std::vector<int64_t> order((size_t)n);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    if (pkey[a] != pkey[b]) return pkey[a] < pkey[b];
    return a < b;
  });
  std::vector<int64_t> cstart;       // cells: contiguous runs of `order`
  std::vector<int64_t> ckey;         // lattice tuple per cell, flat [nc*d]
  for (int64_t j = 0; j < n; ++j)
    if (j == 0 || pkey[order[j]] != pkey[order[j - 1]]) {
      cstart.push_back(j);
      for (int k = 0; k < d; ++k) ckey.push_back(coord(order[j], k));
    }
  const int64_t nc = (int64_t)cstart.size();
  cstart.push_back(n);
  struct H128 { size_t operator()(u128 v) const {
    uint64_t a = (uint64_t)v, b = (uint64_t)(v >> 64);
    a ^= b * 0x9e3779b97f4a7c15ull; a ^= a >> 31; a *= 0xbf58476d1ce4e5b9ull; a ^= a >> 29;
    return (size_t)a; } };
  std::unordered_map<u128, int64_t, H128> cell_of;
  cell_of.reserve((size_t)nc * 2);
  for (int64_t c = 0; c < nc; ++c) cell_of[pkey[order[cstart[c]]]] = c;
  pkey.clear(); pkey.shrink_to_fit();
  auto csize = [&](int64_t c) { return cstart[c + 1] - cstart[c]; };
  auto ck = [&](int64_t c, int k) { return ckey[(size_t)c * d + k]; };

  /* ---- NeighborCells: Chebyshev radius R' (superset of the exact set). ----
   * Points within eps differ by <= eps per axis, hence their lattice
   * coordinates by <= floor(eps/s') + 1. Memoised as CSR. */
  const int64_t R = eps / s + 1;
  std::vector<int64_t> noff((size_t)nc + 1, 0), nbr;  // excludes the cell itself
  if (d <= 3) {
    std::vector<int64_t> off((size_t)d, -R), q((size_t)d);
    const int64_t Rc = R;  // R' <= sqrt(d) + 2 for every eps, so the cube is small
    std::vector<int64_t> offs;  // flat list of offsets
    while (true) {
      bool zero = true;
      for (int k = 0; k < d; ++k) zero &= off[k] == 0;
      if (!zero) offs.insert(offs.end(), off.begin(), off.end());
      int k = d - 1;
      while (k >= 0 && off[k] == Rc) { off[k] = -Rc; --k; }
      if (k < 0) break;
      ++off[k];
    }
    const size_t no = offs.size() / (size_t)d;
    // two passes (count, fill) so cells can be processed independently
    auto probe = [&](int64_t c, std::vector<int64_t> &q, int64_t *dst) {
      int64_t m = 0;
      for (size_t t = 0; t < no; ++t) {
        bool in = true;
        for (int k = 0; k < d; ++k) {
          q[k] = ck(c, k) + offs[t * d + k];
          in &= q[k] >= 0 && q[k] < ext[k];
        }
        if (!in) continue;
        auto it = cell_of.find(pack(q.data()));
        if (it != cell_of.end()) { if (dst) dst[m] = it->second; ++m; }
      }
      return m;
    };
#pragma omp parallel
    {
      std::vector<int64_t> qq((size_t)d);
#pragma omp for schedule(dynamic, 1024)
      for (int64_t c = 0; c < nc; ++c) noff[c + 1] = probe(c, qq, nullptr);
    }
    for (int64_t c = 0; c < nc; ++c) noff[c + 1] += noff[c];
    nbr.resize((size_t)noff[nc]);
#pragma omp parallel
    {
      std::vector<int64_t> qq((size_t)d);
#pragma omp for schedule(dynamic, 1024)
      for (int64_t c = 0; c < nc; ++c) probe(c, qq, nbr.data() + noff[c]);
    }
  } else {
    // each row scans every other cell in ascending order (rows are
    // independent, so they are spread over threads; the row content and
    // order are those of a sequential scan)
    std::vector<std::vector<int64_t>> tmp((size_t)nc);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t a = 0; a < nc; ++a)
      for (int64_t b = 0; b < nc; ++b) {
        if (b == a) continue;
        bool ok = true;
        for (int k = 0; k < d && ok; ++k) ok = std::llabs(ck(a, k) - ck(b, k)) <= R;
        if (ok) tmp[a].push_back(b);
      }
    for (int64_t c = 0; c < nc; ++c) {
      nbr.insert(nbr.end(), tmp[c].begin(), tmp[c].end());
      noff[c + 1] = (int64_t)nbr.size();
    }
  }

  /* ---- MarkCore (Alg 2). ---- */
  std::vector<uint8_t> cf((size_t)n, 0);  // core flag by input index
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t g = 0; g < nc; ++g) {
    if (csize(g) >= min_pts) {
      for (int64_t j = cstart[g]; j < cstart[g + 1]; ++j) cf[order[j]] = 1;
      continue;
    }
    for (int64_t j = cstart[g]; j < cstart[g + 1]; ++j) {
      const int64_t p = order[j];
      int64_t count = csize(g);
      for (int64_t t = noff[g]; t < noff[g + 1] && count < min_pts; ++t) {
        const int64_t h = nbr[t];
        for (int64_t u = cstart[h]; u < cstart[h + 1] && count < min_pts; ++u)
          if (dist2(pts + p * d, pts + order[u] * d, d) <= e2) ++count;
      }
      if (count >= min_pts) cf[p] = 1;
    }
  }

  /* ---- ClusterCore (Alg 3). ---- */
  std::vector<std::vector<int64_t>> cores((size_t)nc);  // core points per cell
  for (int64_t g = 0; g < nc; ++g)
    for (int64_t j = cstart[g]; j < cstart[g + 1]; ++j)
      if (cf[order[j]]) cores[g].push_back(order[j]);
  struct Pair { i128 gap; int64_t g, h; };
  std::vector<Pair> pairs;
  for (int64_t g = 0; g < nc; ++g) {
    if (cores[g].empty()) continue;
    for (int64_t t = noff[g]; t < noff[g + 1]; ++t) {
      const int64_t h = nbr[t];
      if (h >= g || cores[h].empty()) continue;  // "g > h": higher id checks lower
      i128 gap = 0;  // squared lattice gap, used only as the visiting order
      for (int k = 0; k < d; ++k) {
        int64_t t = std::llabs(ck(g, k) - ck(h, k));
        if (t) gap += (i128)((t - 1) * s + 1) * ((t - 1) * s + 1);
      }
      pairs.push_back({gap, g, h});
    }
  }
  std::sort(pairs.begin(), pairs.end(), [](const Pair &a, const Pair &b) {
    if (a.gap != b.gap) return a.gap < b.gap;
    if (a.g != b.g) return a.g < b.g;
    return a.h < b.h;
  });
  // integer box of cell c on axis k: [lo + key*s, lo + key*s + s - 1]
  auto box_d2 = [&](const int32_t *p, int64_t c) {
    i128 acc = 0;
    for (int k = 0; k < d; ++k) {
      int64_t blo = lo[k] + ck(c, k) * s, bhi = blo + s - 1, x = p[k];
      int64_t t = x < blo ? blo - x : (x > bhi ? x - bhi : 0);
      acc += (i128)t * t;
    }
    return acc;
  };
  UF uf(nc);
  std::vector<int64_t> fa, fb;
  for (const Pair &pr : pairs) {
    if (uf.find(pr.g) == uf.find(pr.h)) continue;
    // filter: core points further than eps from the other cell
    fa.clear(); fb.clear();
    for (int64_t p : cores[pr.g]) if (box_d2(pts + p * d, pr.h) <= e2) fa.push_back(p);
    for (int64_t q : cores[pr.h]) if (box_d2(pts + q * d, pr.g) <= e2) fb.push_back(q);
    bool hit = false;
    for (size_t a = 0; a < fa.size() && !hit; ++a)
      for (size_t b = 0; b < fb.size(); ++b)
        if (dist2(pts + fa[a] * d, pts + fb[b] * d, d) <= e2) { hit = true; break; }
    if (hit) uf.link(pr.g, pr.h);
  }
  std::vector<int64_t> cmin((size_t)nc, INT64_MAX);  // min core index per root
  for (int64_t g = 0; g < nc; ++g)
    for (int64_t p : cores[g]) { int64_t r = uf.find(g); cmin[r] = std::min(cmin[r], p); }
  for (int64_t i = 0; i < n; ++i) cluster[i] = -1;
  for (int64_t g = 0; g < nc; ++g)
    for (int64_t p : cores[g]) cluster[p] = (int32_t)cmin[uf.find(g)];
  for (int64_t i = 0; i < n; ++i) core[i] = cf[i];

  /* ---- ClusterBorder (Alg 4). ---- */
  std::vector<int64_t> cnt((size_t)n, 0);
  std::vector<std::vector<int32_t>> lab((size_t)n);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t g = 0; g < nc; ++g) {
    std::vector<int32_t> buf;
    if (csize(g) >= min_pts) continue;
    for (int64_t j = cstart[g]; j < cstart[g + 1]; ++j) {
      const int64_t p = order[j];
      if (cf[p]) continue;
      buf.clear();
      for (int64_t q : cores[g]) if (dist2(pts + p * d, pts + q * d, d) <= e2) buf.push_back(cluster[q]);
      for (int64_t t = noff[g]; t < noff[g + 1]; ++t)
        for (int64_t q : cores[nbr[t]])
          if (dist2(pts + p * d, pts + q * d, d) <= e2) buf.push_back(cluster[q]);
      std::sort(buf.begin(), buf.end());
      buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
      cnt[p] = (int64_t)buf.size();
      lab[p] = buf;
    }
  }
  for (int64_t i = 0; i < n; ++i) border_off[i + 1] = border_off[i] + cnt[i];
  int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(border_off[n] + 1));
  if (!ids) return -1;
  for (int64_t i = 0; i < n; ++i)
    if (cnt[i]) std::memcpy(ids + border_off[i], lab[i].data(), sizeof(int32_t) * (size_t)cnt[i]);
  *border_ids = ids;
  return 0;
}

void o2_free(void *p) { free(p); }

}  // extern "C"
