"""Validity checker for rho-approximate DBSCAN — TEST INFRASTRUCTURE ONLY
(same import rules as the rest of oracle/: tests, smoke and bench only).

Definition (§2, Gan and Tao): as DBSCAN, except that core
points within (eps, eps(1+rho)] may or may not be connected; core points
within eps are connected and core points farther than eps(1+rho) are not.
Several clusterings are valid, so the parity bar for SURVEY §8(f) row f4 is
validity, checked here straight from that definition:

  1. core flags equal the exact ones (O1: |B(p, eps)| >= minPts);
  2. every exact cluster (component of the eps-graph on core points, O1's
     labels) lies inside one approximate cluster;
  3. the exact clusters inside one approximate cluster are connected by
     "relaxed" edges inside it: two of them are adjacent when some core point
     of one is within eps(1+rho) of some core point of the other (an
     approximate cluster is a connected component of the eps-graph plus some
     of the pairs within eps(1+rho), so it is connected by its own pairs);
  4. cluster ids are canonical: a core point's id is the minimum input index
     among the core points of its approximate cluster; non-core points have -1;
  5. border rows: a non-core point's row lists, ascending, the ids of the
     approximate clusters having a core point within eps of it.

The eps(1+rho) threshold is exact on integers: d^2 <= floor(eps^2 (1+rho)^2)
with rho taken as the exact rational value of the double.
Brute force O(n_core^2) pair tests (numpy, blocked): for the small and medium
instances of the tests.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

from . import o1


def relaxed_threshold(eps: int, rho: float) -> int:
    """floor(eps^2 (1 + rho)^2), exact for the double rho."""
    r = Fraction(rho)
    v = Fraction(eps) ** 2 * (1 + r) ** 2
    return v.numerator // v.denominator


def _pairs_within(P: np.ndarray, thr2: int, block: int = 2048):
    """All index pairs i < j of P (int64 rows) with squared distance <= thr2."""
    n = len(P)
    out_i, out_j = [], []
    for a in range(0, n, block):
        A = P[a:a + block]
        for b in range(a, n, block):
            B = P[b:b + block]
            d2 = ((A[:, None, :] - B[None, :, :]) ** 2).sum(-1)
            ii, jj = np.nonzero(d2 <= thr2)
            ii = ii + a
            jj = jj + b
            keep = ii < jj
            out_i.append(ii[keep])
            out_j.append(jj[keep])
    if not out_i:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(out_i), np.concatenate(out_j)


def check(pts, eps: int, min_pts: int, rho: float, core, cluster, border_off, border_ids) -> list[str]:
    """Return the list of violated conditions (empty = valid)."""
    pts = np.ascontiguousarray(pts, dtype=np.int64)
    core = np.asarray(core).astype(bool)
    cluster = np.asarray(cluster).astype(np.int64)
    border_off = np.asarray(border_off).astype(np.int64)
    border_ids = np.asarray(border_ids).astype(np.int64)
    n = len(pts)
    errs = []
    ex = o1(pts.astype(np.int32), eps, min_pts)
    # 1. core flags
    if not np.array_equal(core, ex.core.astype(bool)):
        errs.append("core flags differ from the exact ones")
        return errs
    if np.any(cluster[~core] != -1):
        errs.append("non-core point with a cluster id")
    ci = np.flatnonzero(core)
    if len(ci) == 0:
        if len(border_ids):
            errs.append("border ids without core points")
        return errs
    # 2. exact clusters inside one approximate cluster
    exl = ex.cluster[ci].astype(np.int64)
    apl = cluster[ci]
    first = {}
    for e, a in zip(exl, apl):
        if first.setdefault(int(e), int(a)) != int(a):
            errs.append(f"exact cluster {int(e)} split across approximate clusters")
            break
    # 4. canonical ids
    for a in np.unique(apl):
        members = ci[apl == a]
        if int(members.min()) != int(a):
            errs.append(f"approximate cluster {int(a)} is not named by its minimum core index")
            break
    # 3. relaxed connectivity between the exact clusters of an approximate one
    thr2 = relaxed_threshold(eps, rho)
    P = pts[ci]
    ii, jj = _pairs_within(P, thr2)
    parent = {int(e): int(e) for e in np.unique(exl)}

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x
    same = apl[ii] == apl[jj]  # only pairs inside one approximate cluster can join it
    for a, b in zip(exl[ii[same]], exl[jj[same]]):
        ra, rb = find(int(a)), find(int(b))
        if ra != rb:
            parent[max(ra, rb)] = min(ra, rb)
    comp_of_app = {}
    for e, a in zip(exl, apl):
        r = find(int(e))
        comp_of_app.setdefault(int(a), set()).add(r)
    if any(len(v) > 1 for v in comp_of_app.values()):
        errs.append("approximate cluster joins exact clusters with no chain of pairs within eps(1+rho)")
    # 5. border rows from the approximate labels (exact eps test)
    e2 = eps * eps
    for i in np.flatnonzero(~core):
        d2 = ((P - pts[i]) ** 2).sum(-1)
        want = np.unique(apl[d2 <= e2])
        got = border_ids[border_off[i]:border_off[i + 1]]
        if not np.array_equal(want, got):
            errs.append(f"border row of point {int(i)}")
            break
    if border_off[0] != 0 or border_off[-1] != len(border_ids) or n + 1 != len(border_off):
        errs.append("border CSR shape")
    return errs
