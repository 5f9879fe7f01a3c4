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
    o = oracle_lib.o2(pts, cfg.eps, cfg.min_pts)
    assert_same(g, o, name)
