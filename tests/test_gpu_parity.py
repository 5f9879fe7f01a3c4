"""Parity of the CUDA path (through the C ABI) with the CPU oracles.

Bar: bit-exact on core[], cluster[], border_off[],
border_ids[] — the method reaches the unique DBSCAN result exactly
 and the labels are canonical, so any difference is a
bug. Small cases compare with O1 (definition); medium and full-size cases
with O2 (independent grid version, itself pinned to O1) plus sampled O1
checks at the full BASELINE.json sizes.
"""
import numpy as np
import pytest

import datagen
from helpers import as_rows, assert_same, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU-only container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1912_06255_b200 as pkg  # noqa: E402

GOLD = load_golden()


def key_bits(pts, eps):
    """Width of the packed cell key, for deciding when ERANGE is legitimate."""
    import math
    d = pts.shape[1]
    s = math.isqrt(eps * eps // d) + 1
    span = pts.astype(np.int64).max(0) - pts.astype(np.int64).min(0)
    return sum(int(v // s).bit_length() for v in span)


def gpu(pts, eps, mp, flags=0, host=False):
    if host:
        return pkg.dbscan(np.ascontiguousarray(pts, np.int32), eps, mp, flags=flags)
    t = torch.from_numpy(np.ascontiguousarray(pts, np.int32)).cuda()
    r = pkg.dbscan(t, eps, mp, flags=flags)
    torch.cuda.synchronize()
    return r


def np_result(r):
    class R:
        pass
    o = R()
    for f in ("core", "cluster", "border_off", "border_ids"):
        v = getattr(r, f)
        setattr(o, f, v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v))
    return o


@pytest.mark.parametrize("g", GOLD, ids=[g.name for g in GOLD])
@pytest.mark.parametrize("host", [False, True])
def test_golden(g, host):
    r = np_result(gpu(g.pts, g.eps, g.min_pts, host=host))
    assert as_rows(r.core, r.cluster, r.border_off, r.border_ids) == g.rows


def _instances(seed, count, dmax=8, nmax=400):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        d = int(rng.integers(1, dmax + 1))
        n = int(rng.integers(1, nmax))
        span = int(rng.choice([8, 30, 100, 400, 5000]))
        pts = datagen.random_small(rng, n, d, span)
        eps = int(rng.integers(1, max(2, span // 3)))
        min_pts = int(rng.choice([1, 2, 3, 5, 10, max(1, n // 4), n + 1]))
        yield pts, eps, min_pts


def run_or_erange(pts, eps, mp, flags=0):
    """GPU result, or None when the call returns ERANGE — allowed only if the
    packed cell key really needs more than 63 bits."""
    try:
        return np_result(gpu(pts, eps, mp, flags))
    except pkg.DBSCANError as e:
        assert e.code == -2 and len(pts) and key_bits(pts, eps) > 63, str(e)
        return None


def test_random_small_vs_o1(oracle_lib):
    """500 random instances: d = 1..8, exact-eps ties, duplicates, negative
    coordinates, minPts from 1 to n+1."""
    ran = 0
    for k, (pts, eps, mp) in enumerate(_instances(100, 500)):
        r = run_or_erange(pts, eps, mp)
        if r is not None:
            assert_same(r, oracle_lib.o1(pts, eps, mp), f"instance {k}")
            ran += 1
    assert ran >= 400


@pytest.mark.parametrize("flags", [pkg.F_FORCE_WIDE, pkg.F_FORCE_TREE, pkg.F_NO_WAVES,
                                   pkg.F_FORCE_WIDE | pkg.F_FORCE_TREE | pkg.F_NO_WAVES,
                                   pkg.F_FORCE_SPARSE, pkg.F_NO_SPARSE,
                                   pkg.F_FORCE_SPARSE | pkg.F_FORCE_WIDE | pkg.F_NO_WAVES,
                                   pkg.F_RADIX_GROUP, pkg.F_RADIX_GROUP | pkg.F_FORCE_SPARSE,
                                   pkg.F_LATTICE_GROUP, pkg.F_LATTICE_GROUP | pkg.F_FORCE_SPARSE,
                                   pkg.F_LATTICE_GROUP | pkg.F_NO_SPARSE,
                                   pkg.F_QUADTREE, pkg.F_QUADTREE | pkg.F_RADIX_GROUP | pkg.F_FORCE_TREE,
                                   pkg.F_FORCE_QBOUND, pkg.F_FORCE_QBOUND | pkg.F_RADIX_GROUP | pkg.F_FORCE_WIDE])
def test_flag_variants_vs_o1(oracle_lib, flags):
    for k, (pts, eps, mp) in enumerate(_instances(200 + flags, 120, dmax=8)):
        r = run_or_erange(pts, eps, mp, flags)
        if r is not None:
            assert_same(r, oracle_lib.o1(pts, eps, mp), f"{flags}/{k}")


def test_force_stencil_high_d_vs_o1(oracle_lib):
    """The stencil path for d = 4..6 must agree with the tree path and O1."""
    for k, (pts, eps, mp) in enumerate(_instances(300, 80, dmax=6)):
        if pts.shape[1] < 4:
            continue
        r = run_or_erange(pts, eps, mp, pkg.F_FORCE_STENCIL)
        if r is not None:
            assert_same(r, oracle_lib.o1(pts, eps, mp), f"{k}")


@pytest.mark.parametrize("grouping", [0, pkg.F_RADIX_GROUP, pkg.F_LATTICE_GROUP], ids=["hash", "radix", "lattice"])
@pytest.mark.parametrize("d", [2, 3, 4, 5, 7, 8])
def test_clustered_medium_vs_o2(oracle_lib, d, grouping):
    """Seed-spreader data with dense cells, many neighbours, border points,
    several tiles of every kernel and ragged tails; both groupings (hash
    counting sort, LSD radix sort)."""
    for seed, n in [(1, 20_001), (2, 45_057)]:
        pts = datagen.seed_spreader(n - n % 100, d, 20000, seed + 10 * d, p_step=0.02, noise_frac=0.03)
        for eps, mp in [(150, 15), (400, 60)]:
            r = run_or_erange(pts, eps, mp, grouping)
            if r is not None:
                assert_same(r, oracle_lib.o2(pts, eps, mp), f"d={d} n={n} eps={eps}")


def test_uniform_medium_vs_o2(oracle_lib):
    """Sparse lattice (c5-like): ~1 point per cell, many 1x1 BCP pairs, many
    border points in several clusters."""
    pts = datagen.uniform(200_000, 3, 12_000, 9)
    for mp in (5, 10, 40):
        assert_same(np_result(gpu(pts, 500, mp)), oracle_lib.o2(pts, 500, mp), f"mp={mp}")


def test_c1_full_vs_o1(oracle_lib):
    cfg = datagen.CONFIGS["c1"]
    pts = cfg.points()
    for host in (False, True):
        assert_same(np_result(gpu(pts, cfg.eps, cfg.min_pts, host=host)),
                    oracle_lib.o1(pts, cfg.eps, cfg.min_pts), "c1")


def test_c2_full_vs_o2(oracle_lib):
    cfg = datagen.CONFIGS["c2"]
    pts = cfg.points()
    assert_same(np_result(gpu(pts, cfg.eps, cfg.min_pts)), oracle_lib.o2(pts, cfg.eps, cfg.min_pts), "c2")


@pytest.mark.parametrize("case", [
    ("single", np.array([[5, 7]], np.int32), 3, 1),
    ("single_noise", np.array([[5, 7]], np.int32), 3, 2),
    ("all_dup", np.full((5000, 3), 42, np.int32), 1, 100),
    ("all_dup_noise", np.full((99, 3), 42, np.int32), 1, 100),
    ("huge_eps", datagen.uniform(3000, 4, 1000, 3), 10_000, 3000),
    ("eps1_d8", datagen.random_small(np.random.default_rng(5), 3000, 8, 4), 1, 3),
    ("d1", datagen.random_small(np.random.default_rng(6), 5000, 1, 20000), 7, 3),
    ("extremes_wide", np.array([[-2**31, 0], [2**31 - 1, 0], [2**31 - 1, 3], [0, 2**31 - 1],
                                [-2**31, -2**31], [-2**31 + 3, -2**31]], np.int32), 3, 1),
    ("big_eps_wide", datagen.random_small(np.random.default_rng(8), 2000, 3, 2**31 - 2, negative=True),
     2**30, 4),
])
def test_edge_cases_vs_o1(oracle_lib, case):
    name, pts, eps, mp = case
    assert_same(np_result(gpu(pts, eps, mp)), oracle_lib.o1(pts, eps, mp), name)


def test_empty():
    for host in (False, True):
        r = np_result(gpu(np.zeros((0, 3), np.int32), 5, 2, host=host))
        assert len(r.core) == 0 and list(r.border_off) == [0] and len(r.border_ids) == 0


@pytest.mark.parametrize("grouping", [0, pkg.F_RADIX_GROUP, pkg.F_LATTICE_GROUP], ids=["hash", "radix", "lattice"])
@pytest.mark.parametrize("n", [4095, 4096, 4097, 8191, 12289])
def test_tile_boundaries_vs_o2(oracle_lib, n, grouping):
    """Ragged tails at the radix (4096), scan (2048) and segment (2048) tiles."""
    pts = datagen.seed_spreader(n - n % 100 + 100, 3, 5000, n, p_step=0.1)[:n]
    assert_same(np_result(gpu(pts, 120, 8, grouping)), oracle_lib.o2(pts, 120, 8), f"n={n}")


def test_deterministic_and_permutation_invariant(oracle_lib):
    pts = datagen.seed_spreader(30_000, 3, 8000, 77, p_step=0.05, noise_frac=0.05)
    a = np_result(gpu(pts, 200, 25))
    b = np_result(gpu(pts, 200, 25))
    assert_same(a, b, "repeat")
    perm = np.random.default_rng(1).permutation(len(pts))
    c = np_result(gpu(pts[perm], 200, 25))
    assert np.array_equal(a.core[perm], c.core)
    m = {}
    for j in np.flatnonzero(c.core):
        m.setdefault(int(c.cluster[j]), int(a.cluster[perm[j]]))
        assert m[int(c.cluster[j])] == int(a.cluster[perm[j]])
    assert len(set(m.values())) == len(m)


def test_stream_and_stats():
    pts = datagen.seed_spreader(20_000, 3, 8000, 3, p_step=0.05)
    s = torch.cuda.Stream()
    t = torch.from_numpy(pts).cuda()
    with torch.cuda.stream(s):
        r = pkg.dbscan(t, 200, 20, timing=True)
    s.synchronize()
    assert r.stage_ms["total"] > 0
    assert r.stats["launches"] > 10
    assert r.stats["ncells"] > 0 and r.n_core + r.n_border + r.n_noise == len(pts)


@pytest.mark.parametrize("flags", [0, pkg.F_NO_SPARSE, pkg.F_RADIX_GROUP, pkg.F_LATTICE_GROUP,
                                   pkg.F_LATTICE_GROUP | pkg.F_NO_SPARSE])
def test_sparse_and_csr_paths_vs_o2(oracle_lib, flags):
    """Both the cell-centric sparse path and the CSR path on sparse lattices
    (1-8 points per cell), 1D-3D, with border points in several clusters."""
    for d, n, hi, eps, mp in [(3, 150_000, 12_000, 500, 8), (2, 120_000, 30_000, 150, 5),
                              (1, 50_000, 200_000, 3, 3), (3, 60_000, 4_000, 300, 20)]:
        pts = datagen.uniform(n, d, hi, d + n)
        r = gpu(pts, eps, mp, flags)
        if not (flags & pkg.F_NO_SPARSE) and d == 3 and hi == 12_000:
            assert r.stats["sparse"] == 1
        expect = 0 if flags & pkg.F_RADIX_GROUP else (2 if flags & pkg.F_LATTICE_GROUP else 1)
        if expect == 2 and r.stats["hash_group"] == 0:
            pass  # lattice too large for the counting sort (d=1 span): radix
        else:
            assert r.stats["hash_group"] == expect
        assert_same(np_result(r), oracle_lib.o2(pts, eps, mp), f"d={d} flags={flags}")


@pytest.mark.parametrize("grouping", [0, pkg.F_RADIX_GROUP, pkg.F_FORCE_WIDE], ids=["lattice", "radix", "wide"])
def test_brick_markcore_vs_o2(oracle_lib, grouping):
    """The 3D brick MarkCore (16^3 cells staged with their halo in shared
    memory) against O2 and against the thread-per-point kernel: lattices with
    ragged brick edges, a dense blob whose brick overflows the shared-memory
    capacity (its points go to the thread kernel), and one cell holding more
    than 65535 points."""
    cases = []
    cases.append((datagen.uniform(150_000, 3, 25_000, 31), 500, 3, 1))
    cases.append((datagen.uniform(100_000, 3, 25_000, 32), 600, 4, 1))
    blob = datagen.uniform(200_000, 3, 28_000, 33)
    blob[:6000] = blob[0] + datagen.uniform(6000, 3, 600, 34)   # ~6000 points in a few cells
    cases.append((blob, 500, 10, 2))
    big = datagen.uniform(260_000, 3, 31_000, 35)
    big[:66_000] = big[0]                                        # one cell, > 65535 points
    cases.append((big, 500, 10, 2))
    # denser than 0.3 points per lattice cell, or sparser than 0.15: the thread kernel alone
    cases.append((datagen.uniform(150_000, 3, 12_000, 36), 500, 8, 0))
    cases.append((datagen.uniform(150_000, 3, 40_000, 37), 500, 3, 0))
    for pts, eps, mp, want in cases:
        r = gpu(pts, eps, mp, grouping)
        assert r.stats["sparse"] == 1 and r.stats["brick"] == want, (r.stats, eps)
        if want == 0:
            assert_same(np_result(r), oracle_lib.o2(pts, eps, mp), f"dense eps={eps}")
            continue
        # (the ClusterBorder / ClusterCore bricks fall back to the core-centric
        # kernels when a brick holds more core points than they stage)
        t = gpu(pts, eps, mp, grouping | pkg.F_NO_BRICK)
        assert t.stats["brick"] == 0
        assert_same(np_result(r), np_result(t), f"brick vs thread eps={eps}")
        assert_same(np_result(r), oracle_lib.o2(pts, eps, mp), f"brick eps={eps}")


def test_brick_subcell_edges_vs_o2(oracle_lib):
    """The brick MarkCore's sub-cell stencils (DESIGN.md §5, 4 sub-intervals
    per axis of a cell): points snapped to the sub-interval edges of their
    cells (offsets 0, t_j - 1, t_j, s - 1 from the cell origin lo + c s) and
    pairs at exactly eps ((300, 400, 0) and (0, 0, 500) apart for eps = 500),
    where a stencil one cell or one sub-interval too small would miss a
    neighbour: same result as O2 and as the thread kernel."""
    eps, mp = 500, 4
    pts = datagen.uniform(150_000, 3, 25_000, 41)
    probe = gpu(pts, eps, mp)
    assert probe.stats["brick"] == 1, probe.stats
    s = int(probe.stats["cell_side"])
    lo = pts.min(axis=0).astype(np.int64)
    edges = np.array(sorted({0, s - 1} | {j * s // 4 for j in (1, 2, 3)} | {j * s // 4 - 1 for j in (1, 2, 3)}))
    rng = np.random.default_rng(42)
    k = 60_000
    rel = pts[:k].astype(np.int64) - lo
    snapped = (rel // s) * s + edges[rng.integers(0, len(edges), size=rel.shape)]
    pts[:k] = (snapped + lo).astype(pts.dtype)
    # exact-eps partners for 20,000 of the snapped points
    off = np.array([[300, 400, 0], [0, 0, 500], [-400, 0, 300], [0, -300, -400]], dtype=np.int64)
    m = 20_000
    pts[k:k + m] = (pts[:m].astype(np.int64) + off[rng.integers(0, 4, size=m)]).astype(pts.dtype)
    pts[:, :] = np.maximum(pts, lo)   # (keep the bounding box's origin)
    pts[k + m] = lo
    r = gpu(pts, eps, mp)
    assert r.stats["brick"] == 1, r.stats
    t = gpu(pts, eps, mp, pkg.F_NO_BRICK)
    assert_same(np_result(r), np_result(t), "brick vs thread at sub-cell edges")
    assert_same(np_result(r), oracle_lib.o2(pts, eps, mp), "brick at sub-cell edges")


@pytest.mark.parametrize("mp", [10, 14])
def test_packed_core_pairs_vs_o2(oracle_lib, mp):
    """Sparse ClusterCore in one pass on the packed core points (core cells
    few relative to all cells): a c5-like lattice plus two dense blobs whose
    core cells hold many core points (pairs above SP_SMALL go to the warp
    BCP); equal to the pass on the per-cell tables (F_NO_PACKED_CORE) and
    to O2."""
    eps = 500
    pts = datagen.uniform(400_000, 3, 35_000, 60 + mp)
    pts[:3000] = pts[0] + datagen.uniform(3000, 3, 900, 61)
    pts[3000:5000] = pts[1] + datagen.uniform(2000, 3, 1500, 62)
    r = gpu(pts, eps, mp)
    assert r.stats["sparse"] == 1 and r.stats["sparse_passes"] == 1, r.stats
    t = gpu(pts, eps, mp, pkg.F_NO_PACKED_CORE)
    assert_same(np_result(r), np_result(t), f"packed vs tables mp={mp}")
    assert_same(np_result(r), oracle_lib.o2(pts, eps, mp), f"packed mp={mp}")


def test_point_centric_border_vs_o2(oracle_lib):
    """Sparse lattice where almost every point is core: ClusterBorder runs from
    the few non-core points (domain-boundary points here) instead of from the
    core cells; same result as O2, border points included."""
    for pts, eps, mp in [(datagen.uniform(200_000, 3, 20_000, 97), 600, 5),
                         (datagen.uniform(100_000, 2, 60_000, 98), 250, 4)]:
        r = gpu(pts, eps, mp)
        assert r.stats["sparse"] == 1 and r.stats["point_border"] == 1, r.stats
        want = oracle_lib.o2(pts, eps, mp)
        assert len(want.border_ids) > 0
        assert_same(np_result(r), want, f"point-centric border eps={eps}")
        t = gpu(pts, eps, mp, pkg.F_NO_SPARSE)
        assert_same(np_result(t), want, "csr")


def test_grouping_choice(oracle_lib):
    """Few cells: the hash counting sort groups the points; many distinct
    cells (uniform 3D, 2M points, ~2M cells) on a lattice too large to count
    over: the radix sort runs; on a small lattice: the lattice counting sort;
    all give the same result."""
    few = datagen.seed_spreader(200_000, 3, 100_000, 5, p_step=0.01)
    r = gpu(few, 1000, 50)
    assert r.stats["hash_group"] == 1 and r.stats["sort_passes"] == 0
    many = datagen.uniform(2_000_000, 3, 1_000_000, 6)
    a = gpu(many, 3000, 3)
    assert a.stats["hash_group"] == 0 and a.stats["sort_passes"] > 0
    b = gpu(many, 3000, 3, pkg.F_RADIX_GROUP)
    assert_same(np_result(a), np_result(b), "hash fallback vs radix")
    assert_same(np_result(a), oracle_lib.o2(many, 3000, 3), "radix vs O2")
    dense = datagen.uniform(2_000_000, 3, 40_000, 7)
    c = gpu(dense, 300, 4)
    assert c.stats["hash_group"] == 2 and c.stats["sparse"] == 1
    assert_same(np_result(c), np_result(gpu(dense, 300, 4, pkg.F_RADIX_GROUP)), "lattice vs radix")
    assert_same(np_result(c), oracle_lib.o2(dense, 300, 4), "lattice vs O2")
    # Alg 2's global bound: no point can reach minPts, nothing is grouped
    e = gpu(dense, 300, 5000)
    assert e.n_core == 0 and e.stats["ncells"] == 0 and e.n_noise == len(dense)


def test_lattice_overflow_falls_back(oracle_lib):
    """More than 255 points in one lattice cell overflows its 8-bit counter:
    the radix sort takes over with the same result."""
    pts = datagen.uniform(300_000, 2, 3000, 8)
    pts[:400] = pts[0]
    r = gpu(pts, 20, 3, pkg.F_LATTICE_GROUP)
    assert r.stats["hash_group"] == 0
    assert_same(np_result(r), np_result(gpu(pts, 20, 3, pkg.F_RADIX_GROUP)), "overflow fallback")
    assert_same(np_result(r), oracle_lib.o2(pts, 20, 3), "overflow fallback vs O2")


@pytest.mark.parametrize("d", [2, 3, 5, 7])
def test_varden_and_sweeps_vs_o2(oracle_lib, d):
    """SURVEY §8(f) f1 on the same kernels: SS-varden (variable-density
    clusters) and eps / minPts sweeps at a size
    the oracle finishes in seconds."""
    L = 1e6 if d <= 3 else 1e5
    pts = datagen.seed_spreader(40_000, d, L / 20, 40 + d, 0.02, varden=True, noise_frac=0.01)
    for eps, mp in [(60, 10), (150, 10), (400, 10), (150, 3), (150, 60), (150, 400)]:
        r = run_or_erange(pts, eps, mp)
        if r is not None:
            assert_same(r, oracle_lib.o2(pts, eps, mp), f"varden d={d} eps={eps} mp={mp}")


def test_host_path_caller_buffers(oracle_lib):
    """Host path with caller-owned (pinned) output buffers, border_ids
    included: used when the result fits, else the library allocates; both
    equal the oracle (the side-stream copies overlap ClusterBorder)."""
    pts = datagen.uniform(60_000, 3, 4_000, 31)
    o = oracle_lib.o2(pts, 300, 20)
    n = len(pts)
    for cap in (n, 1):
        outs = (torch.empty(n, dtype=torch.uint8).pin_memory(), torch.empty(n, dtype=torch.int32).pin_memory(),
                torch.empty(n + 1, dtype=torch.int64).pin_memory(), torch.empty(cap, dtype=torch.int32).pin_memory())
        r = pkg.dbscan(torch.from_numpy(pts).pin_memory(), 300, 20, out=outs)
        got = np_result(r)
        assert len(got.border_ids) == int(got.border_off[-1])
        assert_same(got, o, f"cap={cap}")



@pytest.mark.parametrize("flags", [pkg.F_QUADTREE, pkg.F_QUADTREE | pkg.F_RADIX_GROUP,
                                   pkg.F_QUADTREE | pkg.F_FORCE_WIDE])
@pytest.mark.parametrize("d", [2, 3, 5])
def test_quadtree_vs_o2(oracle_lib, d, flags):
    """Row f2 (our-exact-qt): big cells get range-count trees;
    sparse points beside them count through the trees (minPts large, so the
    counts run long: the paper's "spike" case)."""
    L = 30_000 if d <= 3 else 60_000
    pts = datagen.seed_spreader(60_000, d, L, 50 + d, 0.02, noise_frac=0.05)
    for eps, mp in [(400, 300), (400, 1500), (250, 60)]:
        r = run_or_erange(pts, eps, mp, flags)
        if r is None:
            continue
        assert_same(r, oracle_lib.o2(pts, eps, mp), f"qt d={d} eps={eps} mp={mp} flags={flags}")
    r = gpu(pts, 400, 1500, flags)
    assert r.stats["qt_nodes"] > 0


def test_concurrent_host_calls(oracle_lib):
    """Two host threads, one stream each, calling the blocking host-buffer
    path at once (bench.py's e2e mode): no shared state, same results."""
    import threading
    cases = [(datagen.seed_spreader(40_000, 3, 20_000, 81, 0.02, noise_frac=0.03), 200, 15),
             (datagen.uniform(80_000, 3, 6_000, 82), 300, 10),
             (datagen.seed_spreader(30_000, 5, 30_000, 83, 0.02), 600, 20),
             (datagen.uniform(50_000, 2, 20_000, 84), 150, 6)]
    want = [oracle_lib.o2(p, e, m) for p, e, m in cases]
    got = [None] * len(cases)
    errs = []

    def worker(w):
        try:
            st = torch.cuda.Stream()
            for k in range(w, len(cases), 2):
                for _ in range(3):
                    p, e, m = cases[k]
                    got[k] = np_result(pkg.dbscan(torch.from_numpy(p).pin_memory(), e, m, stream=st))
        except Exception as ex:  # pragma: no cover
            errs.append(ex)
    ths = [threading.Thread(target=worker, args=(w,)) for w in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    for k in range(len(cases)):
        assert_same(got[k], want[k], f"case {k}")


def test_workspace_pool(oracle_lib):
    """Pooled workspaces (include/dbscan.h dbscan_release_workspace): calls of
    growing size (the workspace regrows), short-lived threads calling at once
    on both paths (each takes its own workspace from the pool, the idle ones
    catch up in size), an invalid call in between, and a release of the idle
    workspaces: every result equals the oracle's."""
    import threading
    cases = [(datagen.uniform(2_000, 3, 3_000, 91), 300, 4),
             (datagen.seed_spreader(30_000, 3, 20_000, 92, 0.02, noise_frac=0.03), 200, 15),
             (datagen.uniform(120_000, 3, 9_000, 93), 300, 10),
             (datagen.seed_spreader(25_000, 7, 30_000, 94, 0.02), 900, 20)]
    want = [oracle_lib.o2(p, e, m) for p, e, m in cases]
    pkg.release_workspace()
    for (p, e, m), w in zip(cases, want):  # sequential, growing
        assert_same(np_result(gpu(p, e, m)), w, "sequential")
    with pytest.raises(pkg.DBSCANError):
        gpu(cases[0][0], 0, 4)  # eps = 0: rejected before any kernel
    for rnd in range(3):
        got, errs = {}, []

        def worker(k, host):
            try:
                p, e, m = cases[k]
                st = torch.cuda.Stream()
                if host:
                    r = pkg.dbscan(torch.from_numpy(p).pin_memory(), e, m, stream=st)
                else:
                    t = torch.from_numpy(np.ascontiguousarray(p)).cuda()
                    with torch.cuda.stream(st):
                        r = pkg.dbscan(t, e, m, stream=st)
                    st.synchronize()
                got[(k, host)] = np_result(r)
            except Exception as ex:  # pragma: no cover
                errs.append(ex)
        ths = [threading.Thread(target=worker, args=(k, h)) for k in range(len(cases)) for h in (False, True)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        assert not errs, errs
        for (k, h), r in got.items():
            assert_same(r, want[k], f"round {rnd} case {k} host {h}")
        if rnd == 1:
            pkg.release_workspace()


def test_host_path_constant_outputs(oracle_lib):
    """Host path: outputs that are constant are written on the host (all noise:
    core 0, cluster -1, border_off 0; no border point: border_off 0); pinned
    caller buffers pre-filled with garbage must come back exactly right."""
    pts = datagen.uniform(300_000, 3, 3_000, 71)        # dense: every point core, no border point
    noise = datagen.uniform(300_000, 3, 1_000_000, 72)  # sparse: minPts unreachable
    for p, eps, mp in [(pts, 100, 4), (noise, 50, 50), (pts[:5000], 40, 10_000)]:
        want = oracle_lib.o2(p, eps, mp)
        n = len(p)
        outs = (torch.full((n,), 7, dtype=torch.uint8).pin_memory(), torch.full((n,), 7, dtype=torch.int32).pin_memory(),
                torch.full((n + 1,), 7, dtype=torch.int64).pin_memory(), torch.full((n,), 7, dtype=torch.int32).pin_memory())
        r = pkg.dbscan(torch.from_numpy(np.ascontiguousarray(p)).pin_memory(), eps, mp, out=outs)
        assert_same(np_result(r), want, f"eps={eps} minPts={mp}")
        assert len(want.border_ids) == 0


@pytest.mark.parametrize("d,hi", [(5, 20_000), (7, 10_300)])
def test_cell_tree_at_scale_vs_o2(oracle_lib, d, hi):
    """The cell tree (Morton-ordered BVH over the cells, the GPU form of the
    paper's k-d tree range queries) is the default neighbour
    search for d >= 4 above 131,072 cells: uniform 5D / 7D points with ~one
    point per cell and ~10 eps-neighbours each (core, border and noise
    points, tens to hundreds of clusters) — a multi-block bottom-up build and
    deep DFS queries — against O2 (all-pairs cell scan, independent code)."""
    pts = datagen.uniform(160_000, d, hi, 41 + d)
    r = gpu(pts, 2000, 10)
    assert r.stats["tree"] == 1 and r.stats["ncells"] > 131_072, r.stats
    want = oracle_lib.o2(pts, 2000, 10)
    assert want.core.sum() > 10_000 and len(want.border_ids) > 10_000
    assert_same(np_result(r), want, f"cell tree d={d}")


@pytest.mark.parametrize("flags", [pkg.F_FORCE_SPARSE, 0, pkg.F_NO_SPARSE])
def test_sparse_three_pass_cluster_vs_o2(oracle_lib, flags):
    """Sparse ClusterCore in three launches (gap-0 back columns, laterally
    adjacent columns, the rest; the union-find flattened between and the
    parent comparison before Find) runs when most cells hold core points:
    dense uniform 3D where every cell holds core points and one component
    spans the lattice, plus a sparser corner. Checked against O2, and against
    the CSR path (F_NO_SPARSE)."""
    pts = datagen.uniform(400_000, 3, 20_000, 55)
    pts[:20_000] = datagen.uniform(20_000, 3, 60_000, 56)  # sparse surroundings: border and noise
    r = gpu(pts, 700, 6, flags)
    if not flags & pkg.F_NO_SPARSE:
        assert r.stats["sparse"] == 1 and r.stats["sparse_passes"] == 3, r.stats
    else:
        assert r.stats["sparse"] == 0
    want = oracle_lib.o2(pts, 700, 6)
    assert len(want.border_ids) > 0
    assert_same(np_result(r), want, f"three-pass flags={flags}")


def _star(centre, eps):
    """A non-core point at `centre` with six clusters within eps around it
    (one core point per axis direction at 0.96 eps, each joined to a blob of
    12 duplicates 0.6 eps further out): the centre is a border point of six
    clusters, more than the SP_MAXL label slots."""
    pts = [centre]
    for ax in range(3):
        for sg in (-1, 1):
            v = np.zeros(3, np.int64)
            v[ax] = sg
            pts.append(centre + v * int(0.96 * eps))
            pts.extend([centre + v * int(1.56 * eps)] * 12)
    return np.array(pts, np.int32)


@pytest.mark.parametrize("flags", [0, pkg.F_NO_BRICK])
def test_border_many_labels_vs_o2(oracle_lib, flags):
    """ClusterBorder on a c5-like lattice (0.24 points per cell, the brick
    MarkCore or the thread kernel) with planted border points in 6 clusters
    each — more than the SP_MAXL label slots: the overflowed sets are
    enumerated in ascending order — against O2."""
    pts = datagen.uniform(300_000, 3, 30_000, 61)
    eps, mp = 500, 10
    centres = [np.array([5000, 5000, 5000]), np.array([20000, 9000, 15000]), np.array([12000, 25000, 4000])]
    keep = np.ones(len(pts), bool)
    for c in centres:
        keep &= np.abs(pts.astype(np.int64) - c).max(1) > 2000
    pts = np.concatenate([pts[keep]] + [_star(c, eps) for c in centres]).astype(np.int32)
    r = gpu(pts, eps, mp, flags)
    assert r.stats["sparse"] == 1 and r.stats["brick"] == (0 if flags else 1), r.stats
    want = oracle_lib.o2(pts, eps, mp)
    rows = np.diff(want.border_off)
    assert rows.max() == 6 and (rows == 6).sum() == 3
    assert_same(np_result(r), want, f"star flags={flags}")


@pytest.mark.parametrize("d", [2, 3, 5])
def test_subcell_bounds_large_minpts_vs_o2(oracle_lib, d):
    """Row f2 for large minPts: points proved core by lower bounds from
    sub-cell counts (cells of >= 256 points subdivided, nodes inside the
    eps-ball of a query sub-cell counted without tests), the rest counted
    exactly. Seed-spreader clusters with cells of thousands of points,
    minPts around the neighbourhood sizes (some points decided by the
    bounds, some counted, some non-core), against O2 and against the path
    without the bounds."""
    L = 1e6 if d <= 3 else 1e5
    pts = datagen.seed_spreader(300_000, d, L / 10, 70 + d, 0.002, noise_frac=0.01)
    eps = 400 if d <= 3 else 1500
    for mp in (2000, 8000):
        r = gpu(pts, eps, mp)
        assert r.stats["qb_decided"] >= 0, r.stats
        want = oracle_lib.o2(pts, eps, mp)
        assert_same(np_result(r), want, f"bounds d={d} mp={mp}")
        assert_same(np_result(gpu(pts, eps, mp, pkg.F_NO_QBOUND)), want, f"no bounds d={d} mp={mp}")
    assert r.stats["qb_decided"] > 0 or d == 5


@pytest.mark.parametrize("d", [6, 7])
def test_markcore_cell_tiles_vs_o2(oracle_lib, d):
    """MarkCore's cell tiles (d >= 6: a warp per sparse cell, a lane per
    point, candidates staged 32 at a time, neighbour cells beyond eps of the
    tile's bounding box skipped) and the per-point warp kernel's point-box
    filter, on variable-density data whose sparse cells hold 1..300 points:
    minPts 40 (one 32-point slab, mixed cells) and 400 (several slabs), with
    and without the sub-cell bounds marking points core first."""
    pts = datagen.seed_spreader(150_000, d, 2e4, 20, 0.02, varden=True)
    for mp in (40, 400):
        o = oracle_lib.o2(pts, 500, mp)
        for flags in (0, pkg.F_FORCE_QBOUND):
            r = gpu(pts, 500, mp, flags=flags)
            assert_same(np_result(r), o, f"tiles d={d} mp={mp} flags={flags}")


def test_high_d_three_axis_buckets_vs_o2(oracle_lib):
    """d >= 4 with tens of thousands of clustered cells (SS-varden 7D in a
    small domain: 52K cells): the all-pairs neighbour search buckets the cells
    by three lattice axes, a run per (axis-0, axis-1) bucket over the axis-2
    window; against O2 (all-pairs cell scan, independent code)."""
    pts = datagen.seed_spreader(300_000, 7, 2e4, 27, 0.02, varden=True)
    for mp in (20, 300):
        o = oracle_lib.o2(pts, 600, mp)
        # one test pass into candidate-capacity rows + compaction (default),
        # and the counting + filling passes (the fallback for huge rows)
        for flags in (0, pkg.F_NBR_TWO_PASS):
            r = gpu(pts, 600, mp, flags=flags)
            assert r.stats["tree"] == 1 and 16384 <= r.stats["ncells"] <= 131_072, r.stats
            assert_same(np_result(r), o, f"3-axis buckets mp={mp} flags={flags}")
