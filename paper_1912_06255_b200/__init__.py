"""paper_1912_06255_b200 — exact grid DBSCAN (Wang, Gu, Shun, SIGMOD 2020,
arXiv 1912.06255) on one B200.

Thin ctypes binding over the C ABI in `include/dbscan.h`
(`libdbscan_b200.so`, built in-tree from `csrc/`). Argument marshalling only:
every step of the method runs in the library's CUDA kernels. PyTorch is used
for device memory and streams. There is no CPU fallback: importing this
package on a machine without the built library raises, and calling it without
a CUDA device returns the library's CUDA error.

    import torch, paper_1912_06255_b200 as db
    r = db.dbscan(torch.tensor(pts, dtype=torch.int32, device="cuda"), eps=1000, min_pts=100)
    r.core, r.cluster, r.border_off, r.border_ids   # torch tensors on the device

Result convention (DESIGN.md readings): `core` u8[n];
`cluster` i32[n] = minimum input index of a core point of the point's cluster
for core points, -1 otherwise; `border_off` i64[n+1] / `border_ids` i32[nnz]
= CSR of each non-core point's ascending distinct cluster ids (empty = noise).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["dbscan", "Result", "lib_path", "load", "F_DEVICE_IO", "F_TIMING", "F_CALLER_OUT",
           "F_FORCE_STENCIL", "F_FORCE_TREE", "F_FORCE_WIDE", "F_NO_WAVES", "F_NO_SPARSE",
           "F_FORCE_SPARSE", "F_RADIX_GROUP", "F_LATTICE_GROUP", "F_COUNT_WORK", "F_QUADTREE", "F_NO_BRICK", "F_NO_QBOUND", "F_FORCE_QBOUND", "F_NBR_TWO_PASS", "STAGES", "release_workspace",
           "STATS", "peak_dist",
           "DBSCANError"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# DBSCAN_B200_COUNT=1 selects the measurement build (make count): every
# distance test is counted into stats (bench.py's untimed work pass)
lib_path = os.path.join(_HERE, "libdbscan_b200_count.so" if os.environ.get("DBSCAN_B200_COUNT") == "1"
                        else "libdbscan_b200.so")

# flags (include/dbscan.h)
F_DEVICE_IO, F_TIMING, F_CALLER_OUT = 1, 2, 4
F_FORCE_STENCIL, F_FORCE_TREE, F_FORCE_WIDE, F_NO_WAVES = 8, 16, 32, 64
F_NO_SPARSE, F_FORCE_SPARSE, F_RADIX_GROUP, F_LATTICE_GROUP, F_COUNT_WORK = 128, 256, 512, 1024, 2048
F_QUADTREE, F_NO_BRICK, F_NO_QBOUND, F_FORCE_QBOUND = 4096, 8192, 16384, 32768
F_NBR_TWO_PASS = 65536
F_NO_PACKED_CORE = 131072
NSTAGES, NSTATS = 12, 32
STAGES = ["bbox", "keys+sort", "sort", "segment", "hash", "neighbors", "markcore", "compact",
          "cluster", "labels", "border", "total"]
STATS = ["ncells", "key_bits", "sort_passes", "nbr_entries", "core_cells", "pairs", "pairs_tested",
         "launches", "wide", "tree", "cell_side", "dense_dir", "sparse", "hash_group", "markcore_tests", "qt_nodes", "approx_side", "brick", "point_border",
         "sparse_passes", "bcp_tests", "border_tests", "counting_build", "qb_decided", "markcore_alg2"]


class _Result(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("core", C.c_void_p),
        ("cluster", C.c_void_p),
        ("border_off", C.c_void_p),
        ("border_ids", C.c_void_p),
        ("nnz", C.c_int64),
        ("n_core", C.c_int64),
        ("n_border", C.c_int64),
        ("n_noise", C.c_int64),
        ("n_clusters", C.c_int64),
        ("stage_ms", C.c_float * NSTAGES),
        ("stats", C.c_int64 * NSTATS),
        ("flags", C.c_uint32),
        ("priv", C.c_void_p),
    ]


class DBSCANError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"dbscan failed ({code}): {msg}")
        self.code = code


_lib = None


def load():
    """Load libdbscan_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(lib_path):
            raise ImportError(f"{lib_path} is missing: build it with `make -C {_HERE}` "
                              "or __graft_entry__.build() (no CPU fallback exists)")
        lib = C.CDLL(lib_path)
        lib.dbscan.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_uint32,
                               C.c_void_p, C.POINTER(_Result)]
        lib.dbscan.restype = C.c_int
        lib.dbscan_approx.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_double,
                                      C.c_uint32, C.c_void_p, C.POINTER(_Result)]
        lib.dbscan_approx.restype = C.c_int
        lib.dbscan_result_free.argtypes = [C.POINTER(_Result)]
        lib.dbscan_error_string.argtypes = [C.c_int]
        lib.dbscan_error_string.restype = C.c_char_p
        lib.dbscan_stage_name.argtypes = [C.c_int]
        lib.dbscan_stage_name.restype = C.c_char_p
        lib.dbscan_version.restype = C.c_int
        lib.dbscan_peak_dist.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_void_p,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.dbscan_peak_dist.restype = C.c_int
        lib.dbscan_release_workspace.argtypes = []
        lib.dbscan_release_workspace.restype = None
        _lib = lib
    return _lib


@dataclass
class Result:
    core: object         # u8[n]   (torch tensor on the device, or numpy on the host path)
    cluster: object      # i32[n]
    border_off: object   # i64[n+1]
    border_ids: object   # i32[nnz]
    n_core: int = 0
    n_border: int = 0
    n_noise: int = 0
    n_clusters: int = 0
    stage_ms: dict = field(default_factory=dict)
    stats: dict = field(default_factory=dict)


class _DeviceBuffer:
    """Owns library-allocated device memory; exposes it to torch through
    __cuda_array_interface__ and releases it with dbscan_result_free."""

    def __init__(self, res: _Result, ptr: int, n: int, typestr: str):
        self._res = res
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}

    def __del__(self):
        if _lib is not None and self._res is not None:
            _lib.dbscan_result_free(C.byref(self._res))
            self._res = None


def peak_dist(d: int, variant: int = 0, qt: int = 1, reps: int = 200, stream=None) -> dict:
    """U1 microbenchmark (dbscan_peak_dist): measured distance tests per second
    of the exact predicate on the current CUDA device. variant 0 = shipped
    uint32 path, 1 = shipped 64-bit path, 2 = fp64, 3 = the brick MarkCore's
    predicate on packed 8-byte rows (d = 3)."""
    lib = load()
    tps, ms = C.c_double(), C.c_double()
    tests, hits = C.c_int64(), C.c_int64()
    st = None
    if stream is not None:
        st = C.c_void_p(stream.cuda_stream)
    rc = lib.dbscan_peak_dist(int(d), int(variant), int(qt), int(reps), st, C.byref(tps), C.byref(ms),
                              C.byref(tests), C.byref(hits))
    _check(lib, rc)
    return {"d": d, "variant": ("u32", "i64", "f64", "brick")[variant], "qt": qt, "tests_per_s": tps.value,
            "ms": ms.value, "tests": tests.value, "hits": hits.value}


def release_workspace() -> None:
    """Free the calling thread's device workspace (dbscan_release_workspace)."""
    load().dbscan_release_workspace()


def _finish(res: _Result, flags: int) -> dict:
    info = {"stage_ms": {}, "stats": {}}
    if flags & F_TIMING:
        info["stage_ms"] = {STAGES[i]: float(res.stage_ms[i]) for i in range(NSTAGES)
                            if res.stage_ms[i] > 0}
    info["stats"] = {STATS[i]: int(res.stats[i]) for i in range(len(STATS))}
    return info


def _call(lib, ptr, n, d, eps, min_pts, rho, flags, stream, res):
    if rho is None:
        return lib.dbscan(ptr, n, d, eps, min_pts, flags, stream, res)
    return lib.dbscan_approx(ptr, n, d, eps, min_pts, float(rho), flags, stream, res)


def _check(lib, rc):
    if rc != 0:
        raise DBSCANError(rc, lib.dbscan_error_string(rc).decode())


def dbscan(points, eps: int, min_pts: int, *, flags: int = 0, timing: bool = False, stream=None,
           out=None, rho: float | None = None) -> Result:
    """Exact DBSCAN of integer points.

    points: (n, d) int32 — a CUDA torch tensor (device path: outputs are torch
    tensors on the same device, computed on `stream` or the current stream),
    or a host array / CPU tensor (host path: the library copies in and out;
    pinned memory makes those copies fast; outputs are numpy arrays).
    rho: when given, rho-approximate DBSCAN (dbscan_approx).
    out: optional (core, cluster, border_off[, border_ids]) caller buffers for
    the host path (e.g. pinned CPU tensors), passed with DBSCAN_F_CALLER_OUT;
    border_ids is used when the result fits it (returned as a prefix view).
    """
    lib = load()
    import torch
    flags = int(flags) | (F_TIMING if timing else 0)
    res = _Result()
    if isinstance(points, torch.Tensor) and points.is_cuda:
        if points.dtype != torch.int32 or points.dim() != 2:
            raise TypeError("points must be an (n, d) int32 tensor")
        pts = points.contiguous()
        n, d = pts.shape
        dev = pts.device
        cur = torch.cuda.current_stream(dev)
        st = cur if stream is None else stream
        if st != cur:  # order the call after the work that produced `points` on the current stream
            st.wait_stream(cur)
        core = torch.empty(n, dtype=torch.uint8, device=dev)
        cluster = torch.empty(n, dtype=torch.int32, device=dev)
        off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        res.core, res.cluster, res.border_off = core.data_ptr(), cluster.data_ptr(), off.data_ptr()
        with torch.cuda.device(dev):
            rc = _call(lib, C.c_void_p(pts.data_ptr()), n, d, int(eps), int(min_pts), rho,
                       flags | F_DEVICE_IO | F_CALLER_OUT, C.c_void_p(st.cuda_stream), C.byref(res))
        _check(lib, rc)
        if st != cur:  # outputs come from the current stream's allocator but are written on st
            for t in (core, cluster, off):
                t.record_stream(st)
        nnz = int(res.nnz)
        if nnz > 0:
            ids = torch.as_tensor(_DeviceBuffer(res, res.border_ids, nnz, "<i4"), device=dev)
        else:
            lib.dbscan_result_free(C.byref(res))
            ids = torch.empty(0, dtype=torch.int32, device=dev)
        info = _finish(res, flags)
        return Result(core, cluster, off, ids, int(res.n_core), int(res.n_border),
                      int(res.n_noise), int(res.n_clusters), **info)

    # host path
    if isinstance(points, torch.Tensor):
        if points.dtype != torch.int32 or points.dim() != 2:
            raise TypeError("points must be an (n, d) int32 tensor")
        host = points.contiguous()
        ptr, (n, d) = host.data_ptr(), host.shape
        keep = host
    else:
        keep = np.ascontiguousarray(points, dtype=np.int32)
        if keep.ndim != 2:
            raise TypeError("points must be (n, d)")
        ptr, (n, d) = keep.ctypes.data, keep.shape
    f = flags & ~F_DEVICE_IO
    ids_b = None
    if out is not None:
        core_b, cl_b, off_b = out[:3]
        res.core, res.cluster, res.border_off = (_hostptr(core_b), _hostptr(cl_b), _hostptr(off_b))
        if len(out) > 3 and out[3] is not None:
            ids_b = out[3]
            res.border_ids = _hostptr(ids_b)
            res.nnz = len(ids_b)
        f |= F_CALLER_OUT
    st = 0 if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    rc = _call(lib, C.c_void_p(ptr), n, d, int(eps), int(min_pts), rho, f, C.c_void_p(st), C.byref(res))
    del keep
    _check(lib, rc)
    nnz = int(res.nnz)
    if out is not None:
        core, cluster, off = out[:3]
    else:
        core = np.ctypeslib.as_array(C.cast(res.core, C.POINTER(C.c_uint8)), shape=(n,)).copy() if n else np.zeros(0, np.uint8)
        cluster = np.ctypeslib.as_array(C.cast(res.cluster, C.POINTER(C.c_int32)), shape=(n,)).copy() if n else np.zeros(0, np.int32)
        off = np.ctypeslib.as_array(C.cast(res.border_off, C.POINTER(C.c_int64)), shape=(n + 1,)).copy()
    if ids_b is not None and res.border_ids == _hostptr(ids_b):
        ids = ids_b[:nnz]
    else:
        ids = (np.ctypeslib.as_array(C.cast(res.border_ids, C.POINTER(C.c_int32)), shape=(nnz,)).copy()
               if nnz else np.zeros(0, np.int32))
    info = _finish(res, flags)
    out_res = Result(core, cluster, off, ids, int(res.n_core), int(res.n_border), int(res.n_noise),
                     int(res.n_clusters), **info)
    lib.dbscan_result_free(C.byref(res))
    return out_res


def _hostptr(b) -> int:
    if hasattr(b, "data_ptr"):
        return b.data_ptr()
    return b.ctypes.data
