"""Full-size parity on BASELINE.json's configs (10M points), in the launch
configuration bench.py times (device-resident input, default flags).

* Whole-output comparison with O2 (independent CPU grid version, pinned to O1
  in tests/test_oracle.py), bit-exact.
* Sampled O1 checks, computed one point at a time from the definition
  (P:L197-222): exact eps-neighbourhood counts decide core flags; sampled
  non-core points' border rows equal the labels of core points within eps;
  sampled core points have no eps-neighbour core point with another label.
"""
import numpy as np
import pytest

import datagen
from helpers import assert_same

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1912_06255_b200 as pkg  # noqa: E402

SAMPLES = 256
_O2 = {}


def o2_of(oracle_lib, name):
    """O2 on a BASELINE run, computed once per session (several tests compare with it)."""
    if name not in _O2:
        cfg = datagen.CONFIGS[name]
        _O2[name] = oracle_lib.o2(cfg.points(), cfg.eps, cfg.min_pts)
    return _O2[name]


def run_gpu(pts, eps, mp):
    r = pkg.dbscan(torch.from_numpy(pts).cuda(), eps, mp)
    torch.cuda.synchronize()
    class R:
        pass
    o = R()
    for f in ("core", "cluster", "border_off", "border_ids"):
        setattr(o, f, getattr(r, f).cpu().numpy())
    o.stats = r.stats
    return o


@pytest.mark.parametrize("name", ["c3", "c4_5d", "c4_7d", "c5_10", "c5_10k"])
def test_full_config(oracle_lib, name):
    cfg = datagen.CONFIGS[name]
    pts = cfg.points()
    assert datagen.sha256_prefix(pts) == cfg.sha
    g = run_gpu(pts, cfg.eps, cfg.min_pts)
    # sampled definition checks (O1, one point at a time)
    rng = np.random.default_rng(11)
    sample = rng.choice(len(pts), SAMPLES, replace=False)
    cnt = oracle_lib.counts_for(pts, cfg.eps, sample)
    assert np.array_equal(g.core[sample].astype(bool), cnt >= cfg.min_pts), "sampled core flags"
    nc = sample[~g.core[sample].astype(bool)]
    if len(nc):
        off, ids = oracle_lib.labels_near_for(pts, cfg.eps, g.core, g.cluster, nc)
        for k, i in enumerate(nc):
            assert list(g.border_ids[g.border_off[i]:g.border_off[i + 1]]) == list(ids[off[k]:off[k + 1]])
    cs = sample[g.core[sample].astype(bool)][:64]
    if len(cs):
        assert (oracle_lib.core_label_violations(pts, cfg.eps, g.core, g.cluster, cs) == 0).all()
    # whole output vs the independent grid oracle
    assert_same(g, o2_of(oracle_lib, name), name)


def test_e2e_host_path_full(oracle_lib):
    """The path bench.py's `e2e` times, at full size: every BASELINE run
    (c2, c3, c4 5D/7D, c5 at minPts 10 and 10^4) through the blocking
    host-buffer C ABI with pinned inputs and caller-owned pinned outputs,
    three host threads with one stream each taking the runs from a shared
    queue (concurrent calls, serialised input copies, side-stream output
    copies, host-written constant outputs). Two steps; every output
    byte-compared with O2."""
    import bench
    names = ["c2", "c3", "c4_5d", "c4_7d", "c5_10", "c5_10k"]
    data = [(nm, datagen.CONFIGS[nm], None, datagen.CONFIGS[nm].points()) for nm in names]
    dev = torch.device("cuda", 0)
    host = bench.e2e_host_buffers(data, torch)
    streams = [torch.cuda.Stream(dev) for _ in range(3)]
    order = bench.e2e_order(host, [float(c.n) for _, c, _, _ in data])
    for step in range(2):
        for _, _, outs in host:  # stale bytes must not survive a step
            for t in outs:
                t.fill_(0x5A if t.dtype == torch.uint8 else 0x5A5A5A5A)
        _, h2d, _, res = bench.e2e_calls(pkg, host, order, streams, dev, keep=True)
        assert h2d == sum(p.nbytes for _, _, _, p in data)
        for (nm, cfg, _, _), r in zip(data, res):
            class O:
                pass
            o = O()
            o.core, o.cluster, o.border_off = (t.numpy() for t in (r.core, r.cluster, r.border_off))
            o.border_ids = np.asarray(r.border_ids)
            assert_same(o, o2_of(oracle_lib, nm), f"e2e {nm} step {step}")


@pytest.mark.parametrize("kind", ["uniform", "spreader"])
def test_large_inputs_sampled(oracle_lib, kind):
    """Beyond the BASELINE sizes (40M points): the lattice counting sort's
    limit is passed (uniform data takes the radix sort), the hash table holds
    the seed spreader's cells. Checked by sampled O1 evaluations (core flags,
    border rows, label consistency) and global invariants of canonical ids."""
    n = 40_000_000
    if kind == "uniform":
        pts = datagen.uniform(n, 3, 200_000, 17)
        eps, mp = 500, 10
    else:
        pts = datagen.seed_spreader(n, 3, 1e6, 18, 1000 / n, noise_frac=1e-4)
        eps, mp = 1000, 100
    g = run_gpu(pts, eps, mp)
    core = g.core.astype(bool)
    # canonical ids: a core point's id is a core point of the same cluster, the smallest
    assert (g.cluster[~core] == -1).all()
    cl = g.cluster[core]
    assert core[cl].all() and (g.cluster[cl] == cl).all()
    assert (cl <= np.flatnonzero(core)).all()
    rng = np.random.default_rng(5)
    sample = rng.choice(n, SAMPLES, replace=False)
    cnt = oracle_lib.counts_for(pts, eps, sample)
    assert np.array_equal(core[sample], cnt >= mp), "sampled core flags"
    nc = sample[~core[sample]]
    if len(nc):
        off, ids = oracle_lib.labels_near_for(pts, eps, g.core, g.cluster, nc)
        for k, i in enumerate(nc):
            assert list(g.border_ids[g.border_off[i]:g.border_off[i + 1]]) == list(ids[off[k]:off[k + 1]])
    cs = sample[core[sample]][:64]
    if len(cs):
        assert (oracle_lib.core_label_violations(pts, eps, g.core, g.cluster, cs) == 0).all()
