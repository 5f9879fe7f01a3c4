"""CPU oracles for exact DBSCAN — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package. The product path
(`paper_1912_06255_b200/`) never imports, links or calls it; the two share no
code (only the seeded input generators in `datagen/`, which hold none of the
method's arithmetic).

* `o1` — O1, DBSCAN straight from the definition (§2):
  O(n^2) exact counts, BFS over core points from the smallest unlabelled core
  index, border label sets. Plain C in `o1_bruteforce.c`.
* `o2` — O2, an independent sequential CPU grid DBSCAN following Alg 1-4
   with different free choices from the
  GPU path (cell side, grouping, neighbour enumeration, pair order). C++ in
  `o2_grid.cpp`. Also the "simple CPU grid version" baseline of
  BASELINE.json's north_star.
* `counts_for`, `labels_near_for`, `core_label_violations` — O1 evaluated one
  point at a time, for sampled checks at sizes where O(n^2) cannot run.

Pins: tests/test_oracle.py (golden vectors under tests/golden/, sklearn,
scipy connected components, closed forms, invariants). Nothing here is
"parity unpinned".

Result convention (DESIGN.md §"Readings"): `core` u8[n]; `cluster` i32[n] =
minimum input index of a core point of the cluster for core points, -1
otherwise; `border_off` i64[n+1] CSR over all points in input order;
`border_ids` i32[nnz] ascending distinct cluster ids (rows of core and noise
points are empty).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/liboracle.so with gcc (idempotent)."""
    if force or not os.path.exists(_LIB_PATH) or any(
            os.path.getmtime(os.path.join(_HERE, f)) > os.path.getmtime(_LIB_PATH)
            for f in ("o1_bruteforce.c", "o2_grid.cpp", "Makefile")):
        subprocess.run(["make", "-s", "-B", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB_PATH)
        P, I64, I32 = C.c_void_p, C.c_int64, C.c_int32
        lib.o1_dbscan.argtypes = [P, I64, I32, I64, I64, P, P, P, C.POINTER(C.c_void_p), C.c_int]
        lib.o1_dbscan.restype = C.c_int
        lib.o2_dbscan.argtypes = [P, I64, I32, I64, I64, P, P, P, C.POINTER(C.c_void_p)]
        lib.o2_dbscan.restype = C.c_int
        lib.o1_counts_for.argtypes = [P, I64, I32, I64, P, I64, P, C.c_int]
        lib.o1_labels_near_for.argtypes = [P, I64, I32, I64, P, P, P, I64, P, P, P, C.c_int]
        lib.o1_core_label_violations.argtypes = [P, I64, I32, I64, P, P, P, I64, P, C.c_int]
        lib.o1_free.argtypes = [P]
        lib.o2_free.argtypes = [P]
        _lib = lib
    return _lib


@dataclass
class Clustering:
    core: np.ndarray        # u8[n]
    cluster: np.ndarray     # i32[n]
    border_off: np.ndarray  # i64[n+1]
    border_ids: np.ndarray  # i32[nnz]

    def rows(self, i: int) -> np.ndarray:
        return self.border_ids[self.border_off[i]:self.border_off[i + 1]]


def _prep(pts):
    pts = np.ascontiguousarray(pts, dtype=np.int32)
    if pts.ndim != 2:
        raise ValueError("pts must be (n, d)")
    return pts, pts.shape[0], pts.shape[1]


def _run(fn, pts, eps, min_pts, *extra, free=None):
    pts, n, d = _prep(pts)
    core = np.zeros(n, np.uint8)
    cluster = np.zeros(n, np.int32)
    off = np.zeros(n + 1, np.int64)
    ids = C.c_void_p()
    rc = fn(pts.ctypes.data, n, d, int(eps), int(min_pts), core.ctypes.data,
            cluster.ctypes.data, off.ctypes.data, C.byref(ids), *extra)
    if rc != 0:
        raise RuntimeError(f"oracle returned {rc}")
    nnz = int(off[n])
    if ids.value:
        border = np.ctypeslib.as_array(C.cast(ids, C.POINTER(C.c_int32)), shape=(max(nnz, 1),))[:nnz].copy()
        free(ids)
    else:
        border = np.zeros(0, np.int32)
    return Clustering(core, cluster, off, border)


def o1(pts, eps: int, min_pts: int, threads: int = 0) -> Clustering:
    """O1: brute-force DBSCAN from the definition. O(n^2)."""
    lib = _load()
    return _run(lib.o1_dbscan, pts, eps, min_pts, int(threads), free=lib.o1_free)


def o2(pts, eps: int, min_pts: int) -> Clustering:
    """O2: independent sequential CPU grid DBSCAN (Alg 1-4)."""
    lib = _load()
    return _run(lib.o2_dbscan, pts, eps, min_pts, free=lib.o2_free)


def counts_for(pts, eps: int, sample, threads: int = 0) -> np.ndarray:
    """|B(p, eps)| (self included) for each sampled index, by brute force."""
    lib = _load()
    pts, n, d = _prep(pts)
    sample = np.ascontiguousarray(sample, dtype=np.int64)
    out = np.zeros(len(sample), np.int64)
    lib.o1_counts_for(pts.ctypes.data, n, d, int(eps), sample.ctypes.data, len(sample),
                      out.ctypes.data, int(threads))
    return out


def labels_near_for(pts, eps: int, core, label, sample, threads: int = 0):
    """For each sampled point: sorted distinct label[q] over core q within eps
    (P:L211-215 applied to a given labelling). Returns (off, ids) CSR."""
    lib = _load()
    pts, n, d = _prep(pts)
    core = np.ascontiguousarray(core, dtype=np.uint8)
    label = np.ascontiguousarray(label, dtype=np.int32)
    sample = np.ascontiguousarray(sample, dtype=np.int64)
    k = len(sample)
    cnt = np.zeros(k, np.int64)
    lib.o1_labels_near_for(pts.ctypes.data, n, d, int(eps), core.ctypes.data, label.ctypes.data,
                           sample.ctypes.data, k, cnt.ctypes.data, None, None, int(threads))
    off = np.zeros(k + 1, np.int64)
    np.cumsum(cnt, out=off[1:])
    ids = np.zeros(max(int(off[-1]), 1), np.int32)
    lib.o1_labels_near_for(pts.ctypes.data, n, d, int(eps), core.ctypes.data, label.ctypes.data,
                           sample.ctypes.data, k, cnt.ctypes.data, off.ctypes.data,
                           ids.ctypes.data, int(threads))
    return off, ids[:off[-1]]


def core_label_violations(pts, eps: int, core, label, sample, threads: int = 0) -> np.ndarray:
    """For each sampled core point: #core points within eps with another label."""
    lib = _load()
    pts, n, d = _prep(pts)
    core = np.ascontiguousarray(core, dtype=np.uint8)
    label = np.ascontiguousarray(label, dtype=np.int32)
    sample = np.ascontiguousarray(sample, dtype=np.int64)
    out = np.zeros(len(sample), np.int64)
    lib.o1_core_label_violations(pts.ctypes.data, n, d, int(eps), core.ctypes.data,
                                 label.ctypes.data, sample.ctypes.data, len(sample),
                                 out.ctypes.data, int(threads))
    return out


def serialize(c: Clustering) -> str:
    """Text form `index,core|border|noise,label[;label...]`."""
    lines = []
    for i in range(len(c.core)):
        if c.core[i]:
            lines.append(f"{i},core,{c.cluster[i]}")
        else:
            r = c.rows(i)
            lines.append(f"{i},border,{';'.join(map(str, r))}" if len(r) else f"{i},noise,")
    return "\n".join(lines)
