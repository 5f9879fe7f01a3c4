"""Row f4 — rho-approximate DBSCAN (§2).

CPU (-m "not gpu"): the validity checker oracle/approx.py is pinned against
hand-built cases whose validity follows from the definition: the exact result
is valid for every rho; merging two exact clusters whose closest core pair is
within eps(1+rho) is valid, beyond it is not; splitting an exact cluster, a
non-canonical id, a wrong border row or a wrong core flag are invalid.

GPU (-m gpu): dbscan_approx outputs pass the checker on random and clustered
instances for several rho; with t = 1 (eps rho too small for a sub-cell of
side 2) the output is the exact one, bit for bit.
"""
import numpy as np
import pytest

import datagen
from helpers import assert_same

from oracle import approx as A


def _chain():
    # 1D: exact clusters {0,1,2} (label 0) and {3,4} (label 3); closest core
    # pair 20 -> 35 at distance 15; eps = 10, minPts = 2
    pts = np.array([[0], [10], [20], [35], [45]], np.int32)
    return pts, 10, 2


def test_relaxed_threshold_exact():
    assert A.relaxed_threshold(10, 0.5) == 225
    assert A.relaxed_threshold(10, 0.4) == 196  # the double 0.4 is slightly above 2/5: 196.000...006
    assert A.relaxed_threshold(1000, 0.01) == 1020100


def test_exact_result_is_valid(oracle_lib):
    for seed in range(6):
        rng = np.random.default_rng(seed)
        pts = datagen.random_small(rng, 300, int(rng.integers(1, 5)), 200)
        o = oracle_lib.o1(pts, 12, 4)
        for rho in (0.01, 0.5, 2.0):
            assert A.check(pts, 12, 4, rho, o.core, o.cluster, o.border_off, o.border_ids) == []


def test_merge_within_relaxed_radius_is_valid():
    pts, eps, mp = _chain()
    core = np.ones(5, np.uint8)
    off = np.zeros(6, np.int64)
    ids = np.zeros(0, np.int32)
    merged = np.zeros(5, np.int32)
    assert A.check(pts, eps, mp, 0.5, core, merged, off, ids) == []      # 15 <= 15
    assert A.check(pts, eps, mp, 0.4, core, merged, off, ids) != []      # 15 > 14
    exact = np.array([0, 0, 0, 3, 3], np.int32)
    assert A.check(pts, eps, mp, 0.4, core, exact, off, ids) == []


def test_invalid_outputs_are_rejected():
    pts, eps, mp = _chain()
    core = np.ones(5, np.uint8)
    off = np.zeros(6, np.int64)
    ids = np.zeros(0, np.int32)
    split = np.array([0, 0, 2, 3, 3], np.int32)          # exact cluster split
    assert A.check(pts, eps, mp, 0.5, core, split, off, ids) != []
    wrong_name = np.array([1, 1, 1, 3, 3], np.int32)     # not the minimum index
    assert A.check(pts, eps, mp, 0.5, core, wrong_name, off, ids) != []
    bad_core = core.copy()
    bad_core[4] = 0
    assert A.check(pts, eps, mp, 0.5, bad_core, np.array([0, 0, 0, 3, -1], np.int32), off, ids) != []


def test_border_rows_checked():
    # a border point beside cluster {0,1,2}: point 25 (within 10 of 20)
    pts = np.array([[0], [5], [10], [25], [60]], np.int32)
    eps, mp = 10, 3
    # core: 0 (0,5,10), 5 (all three), 10 (0,5,10) -> 3 >= 3; 25: {10? no: |25-10|=15} -> only itself
    core = np.array([1, 1, 1, 0, 0], np.uint8)
    cl = np.array([0, 0, 0, -1, -1], np.int32)
    off_noise = np.zeros(6, np.int64)
    assert A.check(pts, eps, mp, 0.5, core, cl, off_noise, np.zeros(0, np.int32)) == []
    off_bad = np.array([0, 0, 0, 0, 1, 1], np.int64)
    assert A.check(pts, eps, mp, 0.5, core, cl, off_bad, np.array([0], np.int32)) != []


# ---------------------------------------------------------------- GPU
def _gpu(pts, eps, mp, rho, flags=0):
    torch = pytest.importorskip("torch")
    import paper_1912_06255_b200 as pkg
    r = pkg.dbscan(torch.from_numpy(np.ascontiguousarray(pts, np.int32)).cuda(), eps, mp, rho=rho, flags=flags)
    torch.cuda.synchronize()
    return r, [getattr(r, f).cpu().numpy() for f in ("core", "cluster", "border_off", "border_ids")]


@pytest.mark.gpu
def test_gpu_approx_random_valid():
    import paper_1912_06255_b200 as pkg
    for seed in range(40):
        rng = np.random.default_rng(1000 + seed)
        d = int(rng.integers(1, 6))
        pts = datagen.random_small(rng, int(rng.integers(50, 600)), d, int(rng.choice([100, 400, 3000])))
        eps = int(rng.integers(20, 200))
        mp = int(rng.choice([1, 2, 4, 8]))
        for rho in (0.05, 0.5, 1.5):
            for flags in (0, pkg.F_RADIX_GROUP, pkg.F_FORCE_SPARSE):
                r, out = _gpu(pts, eps, mp, rho, flags)
                assert A.check(pts, eps, mp, rho, *out) == [], (seed, rho, flags)


@pytest.mark.gpu
@pytest.mark.parametrize("d", [2, 3, 5])
def test_gpu_approx_clustered_valid(d):
    pts = datagen.seed_spreader(8_000, d, 6_000, 70 + d, 0.05, noise_frac=0.05)
    for eps, mp, rho in [(150, 10, 0.3), (300, 30, 1.0), (150, 10, 0.01)]:
        r, out = _gpu(pts, eps, mp, rho)
        assert A.check(pts, eps, mp, rho, *out) == [], (d, eps, mp, rho)


@pytest.mark.gpu
def test_gpu_approx_small_rho_is_exact(oracle_lib):
    pts = datagen.seed_spreader(20_000, 3, 20_000, 9, 0.02, noise_frac=0.03)
    r, out = _gpu(pts, 200, 15, 0.001)  # eps rho / (2 sqrt 3) < 1: t = 1
    assert r.stats["approx_side"] == 0

    class R:
        pass
    g = R()
    g.core, g.cluster, g.border_off, g.border_ids = out
    assert_same(g, oracle_lib.o2(pts, 200, 15), "rho small")
    r, out = _gpu(pts, 200, 15, 0.5)
    assert r.stats["approx_side"] >= 2
