"""The C-ABI library builds for sm_100a, loads, and exports every function include/bbc.h declares
(no compute calls: this runs without a GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "bbc.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:bbc_status|void|int64_t|const char\*)\s+(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("ivf_load", "ivf_free", "bbc_search", "bbc_search_host", "bbc_workspace_size"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2604_01960_b200 import build
    lib_path = build.build()
    L = ctypes.CDLL(lib_path)
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)$", out, flags=re.M))
    assert set(_declared()) <= exported
    from paper_2604_01960_b200 import bbc
    assert set(bbc.EXPORTS) == set(_declared())


def test_sass_is_sm100a():
    from paper_2604_01960_b200 import build
    lib_path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_errors_without_gpu():
    """Argument validation happens before any device work: a null index is rejected."""
    from paper_2604_01960_b200 import bbc
    L = bbc.lib()
    size = ctypes.c_size_t()
    assert L.bbc_workspace_size(None, 1, 1, 1, 1, ctypes.byref(size), None) == 1
    assert b"null" in L.bbc_last_error()
    h = ctypes.c_void_p()
    assert L.ivf_load(b"/nonexistent/index", 0, 1, 0, ctypes.byref(h)) == 2


def test_python_constants_match_header():
    """Every mode constant the binding exposes equals the header's #define."""
    with open(os.path.join(ROOT, "include", "bbc.h")) as f:
        defs = dict(re.findall(r"^#define\s+(BBC_\w+)\s+(-?\d+)", f.read(), flags=re.M))
    from paper_2604_01960_b200.bbc import Index
    pairs = {"SCAN_SIMT": "BBC_SCAN_SIMT", "SCAN_TENSOR": "BBC_SCAN_TENSOR",
             "PROBE_SIMT": "BBC_PROBE_SIMT", "PROBE_TENSOR": "BBC_PROBE_TENSOR",
             "PROBE_AUTO": "BBC_PROBE_AUTO", "RERANK_QUERY": "BBC_RERANK_QUERY",
             "RERANK_LIST": "BBC_RERANK_LIST", "RERANK_AUTO": "BBC_RERANK_AUTO",
             "RERANK_TILE": "BBC_RERANK_TILE",
             "CODES_AUTO": "BBC_CODES_AUTO", "CODES_CACHED": "BBC_CODES_CACHED",
             "CODES_STREAM": "BBC_CODES_STREAM", "ORDER_AUTO": "BBC_ORDER_AUTO",
             "ORDER_PROBE": "BBC_ORDER_PROBE", "ORDER_SWEEP": "BBC_ORDER_SWEEP",
             "ALG3_OFF": "BBC_ALG3_OFF", "ALG3_LIST": "BBC_ALG3_LIST", "ALG3_QUERY": "BBC_ALG3_QUERY"}
    for py, c in pairs.items():
        assert c in defs, c
        assert getattr(Index, py) == int(defs[c]), py


def test_setters_reject_bad_arguments_without_gpu():
    """Mode setters validate before touching the (null) handle."""
    from paper_2604_01960_b200 import bbc
    L = bbc.lib()
    for fn, v in (("bbc_set_buckets", 0), ("bbc_set_buckets", 256), ("bbc_set_remap", -1),
                  ("bbc_set_remap", 256), ("bbc_set_rerank_order", 7), ("bbc_set_scan_mode", 9),
                  ("bbc_set_probe_mode", 5), ("bbc_set_code_loads", 3),
                  ("bbc_set_scan_order", 3)):
        assert getattr(L, fn)(None, v) == 1, fn            # null index first: BBC_ERR_ARG
    for mode, eps0 in ((1, 1.9), (3, 1.9), (1, 0.0)):
        assert L.bbc_set_bound_rerank(None, mode, eps0) == 1   # null index: BBC_ERR_ARG
