"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the oracle side and the CUDA side (tests, bench) and
holds NONE of the method's arithmetic: it only draws integer point sets.

Workload families follow the paper's synthetic datasets (§6
"Datasets": SS-simden / SS-varden seed spreader, UniformFill)
realised as the five `BASELINE.json` configs; the draw order is the one
SURVEY.md §8(d) fixes, and each full-size config is pinned by the SHA-256
prefix of its int32 bytes.

The paper's own datasets are not available; these seeded synthetic inputs
stand in for them (DESIGN.md §"Inputs").
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

__all__ = [
    "Config", "CONFIGS", "make", "seed_spreader", "blobs_2d", "uniform",
    "sha256_prefix", "random_small",
]


def sha256_prefix(pts: np.ndarray, k: int = 16) -> str:
    """First k hex digits of SHA-256 over the C-order int32 bytes."""
    a = np.ascontiguousarray(pts, dtype=np.int32)
    return hashlib.sha256(a.tobytes()).hexdigest()[:k]


def seed_spreader(n: int, d: int, L: float, seed: int, p_step: float,
                  noise_frac: float = 0.0, radius: float = 100.0,
                  shift: float = 50.0, per_step: int = 100,
                  varden: bool = False) -> np.ndarray:
    """Gan-Tao style seed spreader (BASELINE.json configs[1..3]).

    Draw order: restart flags, segment starts, shifts,
    ball directions, ball radii, [noise indices, noise values].
    A spreader emits `per_step` points uniform in a ball of `radius` around
    its position, then moves `shift` in a uniformly random direction; with
    probability `p_step` per step it restarts at a uniform location.

    varden=True gives SS-varden (variable-density clusters):
    each walk segment scales its ball radius and shift by 2^j, j uniform in
    {-1, 0, 1, 2}, so clusters differ 64x in density. The scales are drawn
    after every other draw (the SS-simden draws are unchanged). The paper
    names the generator (Gan and Tao's) but not its varden parameters; this
    scaling is this build's stand-in.
    """
    rng = np.random.default_rng(seed)
    S = n // per_step
    flags = rng.random(S) < p_step
    flags[0] = True
    n_seg = int(flags.sum())
    starts = rng.random((n_seg, d)) * L
    sh = rng.standard_normal((S, d))
    sh /= np.linalg.norm(sh, axis=1, keepdims=True)
    sh *= shift
    sh[flags] = 0.0
    seg = np.cumsum(flags) - 1                       # segment id per step
    csum = np.cumsum(sh, axis=0)
    first = np.flatnonzero(flags)                    # first step of each segment
    # inclusive sum within the segment: csum[t] - csum[first[seg]-1]
    base = np.where(first[:, None] > 0, csum[np.maximum(first - 1, 0)], 0.0)
    v = rng.standard_normal((n, d))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    u = rng.random(n)
    if varden:
        scale = 2.0 ** rng.integers(-1, 3, size=n_seg)
        sh = sh * scale[seg][:, None]
        csum = np.cumsum(sh, axis=0)
        base = np.where(first[:, None] > 0, csum[np.maximum(first - 1, 0)], 0.0)
        r = radius * np.repeat(scale[seg], per_step)
    else:
        r = radius
    pos = starts[seg] + (csum - base[seg])
    pts = np.repeat(pos, per_step, axis=0) + (r * u ** (1.0 / d))[:, None] * v
    if noise_frac > 0:
        k = int(round(noise_frac * n))
        idx = rng.choice(n, k, replace=False)
        pts[idx] = rng.random((k, d)) * L
    return np.clip(np.rint(pts), 0, L - 1).astype(np.int32)


def blobs_2d(seed: int = 0) -> np.ndarray:
    """BASELINE.json configs[0]: 10 Gaussian blobs + 10% uniform replacement."""
    rng = np.random.default_rng(seed)
    centres = rng.random((10, 2)) * 1e6
    pts = np.repeat(centres, 1000, axis=0) + rng.standard_normal((10000, 2)) * 2000
    idx = rng.choice(10000, 1000, replace=False)
    pts[idx] = rng.random((1000, 2)) * 1e6
    return np.rint(pts).astype(np.int32)   # no clip: negative coordinates occur


def uniform(n: int, d: int, hi: int, seed: int) -> np.ndarray:
    """UniformFill stand-in (BASELINE.json configs[4])."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, hi, size=(n, d), dtype=np.int32)


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    eps: int
    min_pts: int
    sha: str          # SHA-256 prefix of the int32 bytes
    note: str

    def points(self) -> np.ndarray:
        return make(self.name)


def make(name: str) -> np.ndarray:
    """Materialise a named config's points (int32, shape (n, d))."""
    if name == "c1":
        return blobs_2d(0)
    if name == "c2":
        return seed_spreader(1_000_000, 2, 1e6, 1, 1000 / 1_000_000)
    if name == "c3":
        return seed_spreader(10_000_000, 3, 1e6, 2, 1000 / 10_000_000, noise_frac=1e-4)
    if name == "c4_5d":
        return seed_spreader(10_000_000, 5, 1e5, 3, 1000 / 10_000_000)
    if name == "c4_7d":
        return seed_spreader(10_000_000, 7, 1e5, 3, 1000 / 10_000_000)
    if name in ("c5", "c5_10", "c5_10k"):
        return uniform(10_000_000, 3, 100_000, 4)
    raise KeyError(name)


CONFIGS = {
    "c1": Config("c1", 10_000, 2, 5000, 10, "2a9f07981dc75dde",
                 "configs[0]: 2D Gaussian blobs + 10% noise"),
    "c2": Config("c2", 1_000_000, 2, 1000, 100, "28a8a8fc1c7f5b03",
                 "configs[1]: 2D seed spreader"),
    "c3": Config("c3", 10_000_000, 3, 1000, 100, "06d8efa94b581e92",
                 "configs[2]: 3D seed spreader + 0.01% noise"),
    "c4_5d": Config("c4_5d", 10_000_000, 5, 2000, 100, "1cf7bd65de057102",
                    "configs[3]: 5D seed spreader"),
    "c4_7d": Config("c4_7d", 10_000_000, 7, 2000, 100, "85e450d468fdb43b",
                    "configs[3]: 7D seed spreader"),
    "c5_10": Config("c5_10", 10_000_000, 3, 500, 10, "191eee28296aa628",
                    "configs[4]: 3D uniform, minPts=10"),
    "c5_10k": Config("c5_10k", 10_000_000, 3, 500, 10_000, "191eee28296aa628",
                     "configs[4]: 3D uniform, minPts=10^4"),
}


def random_small(rng: np.random.Generator, n: int, d: int, span: int,
                 dup_frac: float = 0.1, negative: bool = True) -> np.ndarray:
    """Small random integer instance with duplicates and (optionally) negative
    coordinates, for oracle pins and parity sweeps. Pure input generation."""
    lo = -span // 2 if negative else 0
    pts = rng.integers(lo, lo + span, size=(n, d), dtype=np.int64)
    k = int(dup_frac * n)
    if k and n > 1:
        src = rng.integers(0, n, size=k)
        dst = rng.integers(0, n, size=k)
        pts[dst] = pts[src]
    return pts.astype(np.int32)
