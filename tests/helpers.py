"""Shared test helpers: golden-vector loader, DBSCAN invariant checker and
clustering comparison. Pure test code; no part of either implementation."""
from __future__ import annotations

import glob
import os
from dataclasses import dataclass

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class Golden:
    name: str
    d: int
    eps: int
    min_pts: int
    pts: np.ndarray
    rows: list  # (index, kind, labels tuple)


def load_golden() -> list[Golden]:
    out = []
    for path in sorted(glob.glob(os.path.join(GOLDEN, "v*.txt"))):
        d = eps = mp = None
        pts, rows = [], []
        for line in open(path):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            tag, rest = line.split(" ", 1) if " " in line else (line, "")
            if tag == "param":
                kv = dict(t.split("=") for t in rest.split())
                d, eps, mp = int(kv["d"]), int(kv["eps"]), int(kv["min_pts"])
            elif tag == "p":
                pts.append([int(t) for t in rest.split()])
            elif tag == "e":
                i, kind, labs = rest.split(",", 2)
                rows.append((int(i), kind, tuple(int(t) for t in labs.split(";") if t != "")))
        arr = np.array(pts, dtype=np.int64).reshape(-1, d).astype(np.int32)
        out.append(Golden(os.path.basename(path), d, eps, mp, arr, rows))
    return out


def as_rows(core, cluster, off, ids):
    rows = []
    for i in range(len(core)):
        if core[i]:
            rows.append((i, "core", (int(cluster[i]),)))
        else:
            r = tuple(int(x) for x in ids[off[i]:off[i + 1]])
            rows.append((i, "border" if r else "noise", r))
    return rows


def assert_same(a, b, what=""):
    """Bit-exact comparison of two clusterings (objects with core/cluster/
    border_off/border_ids attributes, numpy or torch)."""
    def np_(x):
        return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
    for f in ("core", "cluster", "border_off", "border_ids"):
        x, y = np_(getattr(a, f)), np_(getattr(b, f))
        if x.shape != y.shape or not np.array_equal(x.astype(np.int64), y.astype(np.int64)):
            bad = None
            if x.shape == y.shape:
                bad = np.flatnonzero(x != y)[:10]
            raise AssertionError(f"{what}: field {f} differs (shapes {x.shape} vs {y.shape}; first bad {bad})")


def pairwise_d2(pts):
    p = pts.astype(np.int64)
    diff = p[:, None, :] - p[None, :, :]
    return (diff * diff).sum(-1)


def check_invariants(pts, eps, min_pts, c):
    """Check a clustering against the DBSCAN definition with an
    independent numpy brute force (small n only)."""
    n = len(pts)
    if n == 0:
        assert len(c.border_off) == 1 and c.border_off[0] == 0
        return
    adj = pairwise_d2(pts) <= eps * eps
    cnt = adj.sum(1)
    core = cnt >= min_pts
    assert np.array_equal(core, c.core.astype(bool)), "core flags"
    # core pairs within eps share a label; labels canonical (min index of component)
    for i in np.flatnonzero(core):
        nb = np.flatnonzero(adj[i] & core)
        assert (c.cluster[nb] == c.cluster[i]).all(), "eps-adjacent cores share a label"
        lab = c.cluster[i]
        assert 0 <= lab <= i and core[lab] and c.cluster[lab] == lab, "canonical label"
    assert (c.cluster[~core] == -1).all(), "non-core cluster = -1"
    # same label <=> same connected component of the core eps-graph (scipy)
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    ci = np.flatnonzero(core)
    if len(ci):
        _, comp = connected_components(csr_matrix(adj[np.ix_(ci, ci)]), directed=False)
        first = {}
        for k, i in enumerate(ci):
            first.setdefault(comp[k], i)
        exp = np.array([first[comp[k]] for k in range(len(ci))])
        assert np.array_equal(c.cluster[ci], exp), "labels = min index of core component"
    for i in np.flatnonzero(~core):
        exp = sorted(set(int(c.cluster[j]) for j in np.flatnonzero(adj[i] & core)))
        got = [int(x) for x in c.border_ids[c.border_off[i]:c.border_off[i + 1]]]
        assert got == exp, f"border set of {i}"
    for i in np.flatnonzero(core):
        assert c.border_off[i + 1] == c.border_off[i]
