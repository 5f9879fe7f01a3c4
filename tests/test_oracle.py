"""Pins for the CPU oracles (-m "not gpu").

O1 (definition) is pinned to things other than itself:
  * hand-computed golden vectors (tests/golden/, each with its citation);
  * sklearn.cluster.DBSCAN (an independent library): core set, core-point
    partition, border-vs-noise status, and that sklearn's single label for a
    border point lies in our border set;
  * minPts = 1 reduces to connected components of the eps-graph (scipy);
  * closed forms: all pairwise distances > eps => all noise; eps >= diameter
    and n >= minPts => one cluster labelled 0;
  * sklearn radius counts pin the per-point count helper.
O2 (independent grid version, Alg 1-4) is pinned against O1 on random
instances (d = 1..8, ties at exactly eps, duplicates, negative coordinates,
minPts from 1 to n+1) and against the same closed forms.
"""
import numpy as np
import pytest

import datagen
from helpers import as_rows, assert_same, check_invariants, load_golden

GOLD = load_golden()


@pytest.mark.parametrize("g", GOLD, ids=[g.name for g in GOLD])
@pytest.mark.parametrize("which", ["o1", "o2"])
def test_golden(oracle_lib, g, which):
    fn = getattr(oracle_lib, which)
    c = fn(g.pts, g.eps, g.min_pts)
    assert as_rows(c.core, c.cluster, c.border_off, c.border_ids) == g.rows


def _sk(pts, eps, min_pts):
    from sklearn.cluster import DBSCAN
    return DBSCAN(eps=eps, min_samples=min_pts, algorithm="kd_tree").fit(pts.astype(np.float64))


def _instances(seed, count, dmax=7, nmax=300):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        d = int(rng.integers(1, dmax + 1))
        n = int(rng.integers(1, nmax))
        span = int(rng.choice([8, 30, 100, 400]))
        pts = datagen.random_small(rng, n, d, span)
        eps = int(rng.integers(1, max(2, span // 3)))
        min_pts = int(rng.choice([1, 2, 3, 5, 10, max(1, n // 4), n + 1]))
        yield pts, eps, min_pts


def test_o1_vs_sklearn(oracle_lib):
    """sklearn computes |x-y| in float64 and tests <= eps; exact for these
    small integer coordinates (squared distances << 2^52)."""
    for pts, eps, mp in _instances(1, 250):
        c = oracle_lib.o1(pts, eps, mp)
        sk = _sk(pts, eps, mp)
        core = np.zeros(len(pts), bool)
        core[sk.core_sample_indices_] = True
        assert np.array_equal(core, c.core.astype(bool))
        # core partition equal up to renaming
        ci = np.flatnonzero(core)
        pairs = set(zip(c.cluster[ci].tolist(), sk.labels_[ci].tolist()))
        assert len(pairs) == len(set(c.cluster[ci])) == len(set(sk.labels_[ci]))
        ours_of = dict((b, a) for a, b in pairs)
        for i in np.flatnonzero(~core):
            row = c.border_ids[c.border_off[i]:c.border_off[i + 1]]
            if sk.labels_[i] == -1:
                assert len(row) == 0
            else:
                assert ours_of[sk.labels_[i]] in row


def test_o1_invariants_and_counts(oracle_lib):
    from sklearn.neighbors import NearestNeighbors
    for pts, eps, mp in _instances(2, 60, nmax=120):
        c = oracle_lib.o1(pts, eps, mp)
        check_invariants(pts, eps, mp, c)
        nn = NearestNeighbors(radius=eps, algorithm="kd_tree").fit(pts.astype(np.float64))
        ref = np.array([len(r) for r in nn.radius_neighbors(pts.astype(np.float64), return_distance=False)])
        sample = np.arange(len(pts))
        assert np.array_equal(oracle_lib.counts_for(pts, eps, sample), ref)


def test_minpts1_is_connected_components(oracle_lib):
    from scipy.sparse.csgraph import connected_components
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(3)
    for _ in range(40):
        d = int(rng.integers(1, 6))
        n = int(rng.integers(1, 200))
        pts = datagen.random_small(rng, n, d, 60)
        eps = int(rng.integers(1, 15))
        for fn in (oracle_lib.o1, oracle_lib.o2):
            c = fn(pts, eps, 1)
            assert c.core.all() and len(c.border_ids) == 0
            g = cKDTree(pts.astype(np.float64)).sparse_distance_matrix(
                cKDTree(pts.astype(np.float64)), eps + 0.5, output_type="coo_matrix")
            # keep exact pairs only (integer squared distance <= eps^2)
            p64 = pts.astype(np.int64)
            keep = ((p64[g.row] - p64[g.col]) ** 2).sum(1) <= eps * eps
            from scipy.sparse import coo_matrix
            adj = coo_matrix((np.ones(keep.sum()), (g.row[keep], g.col[keep])), shape=(n, n))
            _, comp = connected_components(adj, directed=False)
            first = {}
            for i in range(n):
                first.setdefault(comp[i], i)
            assert np.array_equal(c.cluster, [first[comp[i]] for i in range(n)])


def test_closed_forms(oracle_lib):
    rng = np.random.default_rng(4)
    for _ in range(20):
        d = int(rng.integers(1, 5))
        eps = int(rng.integers(1, 20))
        # lattice with spacing eps+1: every pair farther than eps -> all noise
        m = int(rng.integers(1, 6))
        grid = np.stack(np.meshgrid(*[np.arange(m)] * d, indexing="ij"), -1).reshape(-1, d)
        pts = (grid * (eps + 1) - 7).astype(np.int32)
        for fn in (oracle_lib.o1, oracle_lib.o2):
            c = fn(pts, eps, 2)
            assert not c.core.any() and (c.cluster == -1).all() and c.border_off[-1] == 0
        # eps >= diameter: one cluster labelled 0
        pts = datagen.random_small(rng, int(rng.integers(2, 80)), d, 50)
        diam = int(np.ceil(np.sqrt(d) * 50)) + 1
        for fn in (oracle_lib.o1, oracle_lib.o2):
            c = fn(pts, diam, len(pts))
            assert c.core.all() and (c.cluster == 0).all()


def test_o2_vs_o1_random(oracle_lib):
    """>= 300 random instances, d = 1..8, ties, duplicates, negatives."""
    k = 0
    for pts, eps, mp in _instances(5, 330, dmax=8, nmax=260):
        a = oracle_lib.o1(pts, eps, mp)
        b = oracle_lib.o2(pts, eps, mp)
        assert_same(a, b, f"instance {k}")
        k += 1


def test_o2_vs_o1_clustered(oracle_lib):
    """Seed-spreader shaped instances (dense cells, many neighbours)."""
    for seed, d in [(10, 2), (11, 3), (12, 4), (13, 5), (14, 7)]:
        pts = datagen.seed_spreader(2000, d, 3000, seed, p_step=0.2, noise_frac=0.02)
        for eps, mp in [(100, 10), (60, 30), (200, 100)]:
            assert_same(oracle_lib.o1(pts, eps, mp), oracle_lib.o2(pts, eps, mp), f"ss d={d}")


def test_permutation_invariance(oracle_lib):
    rng = np.random.default_rng(6)
    for pts, eps, mp in _instances(7, 30, nmax=150):
        perm = rng.permutation(len(pts))
        for fn in (oracle_lib.o1, oracle_lib.o2):
            a = fn(pts, eps, mp)
            b = fn(pts[perm], eps, mp)
            assert np.array_equal(a.core[perm], b.core)
            # same partition: labels map through the permutation consistently
            ci = np.flatnonzero(b.core)
            m = {}
            for j in ci:
                m.setdefault(int(b.cluster[j]), int(a.cluster[perm[j]]))
                assert m[int(b.cluster[j])] == int(a.cluster[perm[j]])
            assert len(set(m.values())) == len(m)


def test_c1_full(oracle_lib):
    """configs[0] at full size: O1 == O2, and O1's totals match the survey's
    independent sklearn / cKDTree measurement (9,006 core,
    10 clusters, 994 noise)."""
    cfg = datagen.CONFIGS["c1"]
    pts = cfg.points()
    a = oracle_lib.o1(pts, cfg.eps, cfg.min_pts)
    b = oracle_lib.o2(pts, cfg.eps, cfg.min_pts)
    assert_same(a, b, "c1")
    assert int(a.core.sum()) == 9006
    assert len(set(a.cluster[a.core.astype(bool)].tolist())) == 10
    noise = (~a.core.astype(bool)) & (np.diff(a.border_off) == 0)
    assert int(noise.sum()) == 994
    sk = _sk(pts, cfg.eps, cfg.min_pts)
    assert np.array_equal(np.sort(sk.core_sample_indices_), np.flatnonzero(a.core))


@pytest.mark.parametrize("name", ["c1", "c2", "c5_10"])
def test_generator_sha(name):
    cfg = datagen.CONFIGS[name]
    assert datagen.sha256_prefix(cfg.points()) == cfg.sha


def test_sampled_helpers(oracle_lib):
    """labels_near_for / core_label_violations agree with the full O1 result."""
    pts = datagen.seed_spreader(3000, 3, 5000, 21, p_step=0.1, noise_frac=0.05)
    eps, mp = 150, 20
    c = oracle_lib.o1(pts, eps, mp)
    sample = np.arange(len(pts))
    off, ids = oracle_lib.labels_near_for(pts, eps, c.core, c.cluster, sample)
    nc = np.flatnonzero(~c.core.astype(bool))
    for i in nc:
        assert list(ids[off[i]:off[i + 1]]) == list(c.rows(i))
    v = oracle_lib.core_label_violations(pts, eps, c.core, c.cluster, np.flatnonzero(c.core))
    assert (v == 0).all()


def test_core_label_violations_negative(oracle_lib):
    """Negative pins for core_label_violations: a labelling that
    splits one cluster must count violations, and the closed ball (<= eps,
    P:L201-202) must count a pair at exactly eps, not only pairs inside it."""
    # chain 0 - 3 - 6 - 9 on a line, eps = 3: every gap is exactly eps
    pts = np.array([[0, 0], [3, 0], [6, 0], [9, 0]], dtype=np.int32)
    core = np.ones(4, dtype=np.uint8)
    good = np.zeros(4, dtype=np.int32)
    assert (oracle_lib.core_label_violations(pts, 3, core, good, np.arange(4)) == 0).all()
    # split at the exact-eps gap between points 1 and 2: each sees one violation
    split = np.array([0, 0, 2, 2], dtype=np.int32)
    v = oracle_lib.core_label_violations(pts, 3, core, split, np.arange(4))
    assert v.tolist() == [0, 1, 1, 0]
    # one eps less: no point is within eps of another, the split is not seen
    assert (oracle_lib.core_label_violations(pts, 2, core, split, np.arange(4)) == 0).all()
    # a non-core neighbour with another label is not a violation
    core2 = np.array([1, 1, 0, 1], dtype=np.uint8)
    lab2 = np.array([0, 0, -1, 3], dtype=np.int32)
    assert (oracle_lib.core_label_violations(pts, 3, core2, lab2, np.array([0, 1, 3])) == 0).all()
    # 3-4-5 triangle in 2D at eps = 5 (an exact diagonal tie): points 0 and 2
    tri = np.array([[0, 0], [30, 0], [3, 4]], dtype=np.int32)
    lab3 = np.array([0, 1, 2], dtype=np.int32)
    v = oracle_lib.core_label_violations(tri, 5, np.ones(3, dtype=np.uint8), lab3, np.arange(3))
    assert v.tolist() == [1, 0, 1]
    # a 7D tie (6^2 + 2^2 + 3^2 = 7^2) counts, one unit further does not
    a = np.zeros((2, 7), dtype=np.int32)
    a[1, :3] = [6, 2, 3]
    lab = np.array([0, 1], dtype=np.int32)
    one = np.ones(2, dtype=np.uint8)
    assert oracle_lib.core_label_violations(a, 7, one, lab, np.arange(2)).tolist() == [1, 1]
    a[1, 0] = 7
    assert oracle_lib.core_label_violations(a, 7, one, lab, np.arange(2)).tolist() == [0, 0]
