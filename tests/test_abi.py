"""C-ABI checks that run without a GPU (-m "not gpu"): the library loads,
exports every symbol include/dbscan.h declares, and rejects invalid
arguments before touching CUDA."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dbscan.h")


@pytest.fixture(scope="module")
def lib():
    import paper_1912_06255_b200 as pkg
    if not os.path.exists(pkg.lib_path):
        import __graft_entry__
        __graft_entry__.build()
    return pkg.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(dbscan\w*)\s*\(", src, flags=re.M)))


def test_header_declares_entry_points():
    assert declared_functions() == ["dbscan", "dbscan_approx", "dbscan_error_string", "dbscan_peak_dist",
                                    "dbscan_release_workspace", "dbscan_result_free", "dbscan_stage_name", "dbscan_version"]


def test_exports(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.dbscan_version() >= 100
    assert lib.dbscan_stage_name(11) == b"total"
    # no workspace was created (no GPU call): releasing the idle ones is a no-op
    import paper_1912_06255_b200 as pkg
    pkg.release_workspace()


def test_struct_layout_matches_header(lib):
    """The ctypes mirror has the header's field order and size."""
    import paper_1912_06255_b200 as pkg
    names = [f[0] for f in pkg._Result._fields_]
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    body = re.search(r"typedef struct dbscan_result \{(.*?)\} dbscan_result;", src, flags=re.S).group(1)
    hdr = re.findall(r"\*?\s*(\w+)(?:\[\w+\])?\s*[,;]", body)
    assert names == [h for h in hdr if h not in ("int64_t", "uint8_t", "int32_t", "float", "uint32_t", "void")]
    assert C.sizeof(pkg._Result) == 8 * 10 + 4 * 12 + 8 * 32 + 8 + 8


@pytest.mark.parametrize("args", [
    dict(n=-1), dict(d=0), dict(d=9), dict(eps=0), dict(min_pts=0), dict(null_pts=True),
    dict(flags=8 | 16), dict(null_out=True),
])
def test_einval_before_cuda(lib, args):
    import paper_1912_06255_b200 as pkg
    pts = (C.c_int32 * 8)()
    res = pkg._Result()
    rc = lib.dbscan(None if args.get("null_pts") else C.cast(pts, C.c_void_p), args.get("n", 4),
                    args.get("d", 2), args.get("eps", 5), args.get("min_pts", 2), args.get("flags", 0),
                    None, None if args.get("null_out") else C.byref(res))
    assert rc == -1
    assert lib.dbscan_error_string(rc).startswith(b"invalid argument")
    assert not res.border_ids and not res.priv


@pytest.mark.parametrize("args", [(0, 0, 1, 1), (9, 0, 1, 1), (3, 4, 1, 1), (2, 3, 1, 1), (3, 0, 3, 1), (3, 0, 1, 0)])
def test_peak_dist_einval(lib, args):
    """U1 rejects bad arguments before touching CUDA."""
    v = C.c_double()
    assert lib.dbscan_peak_dist(*args, None, C.byref(v), None, None, None) == -1


def test_product_does_not_import_oracle():
    """The product path never references the oracle (test infrastructure)."""
    pkgdir = os.path.join(ROOT, "paper_1912_06255_b200")
    for dp, _, files in os.walk(pkgdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "o1_" not in txt and "o2_" not in txt and "liboracle" not in txt, f
