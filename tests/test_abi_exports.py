"""The C-ABI boundary: every entry point include/kvt_b200.h declares is
exported by the product library (kvt_*), and the placement half of it by the
two checkers (orc_* CPU restatement, ref_* reference library). Load-only —
no compute call, so this runs without a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kvt_b200.h")


def declared():
    src = open(HEADER).read()
    api = re.search(r"#define KVT_DECLARE_API\(P\)(.*?)\n\n", src, re.S).group(1)
    codec = re.search(r"#define KVT_DECLARE_CODEC\(P\)(.*?)\n\n", src, re.S).group(1)
    placement = re.findall(r"P##(\w+)\(", api)
    codec_fns = re.findall(r"P##(\w+)\(", codec)
    extra = re.findall(r"^(?:int|int64_t)\s+kvt_(\w+)\(", src, re.M)
    return placement, codec_fns, extra


def test_header_parses():
    placement, codec, extra = declared()
    assert "insert_joint" in placement and "rearrange" in placement and len(placement) >= 20
    assert "compress" in codec and "unpack" in codec
    assert set(extra) >= {"sync", "set_stream", "launch_count"}


def _exports(path):
    lib = C.CDLL(path)
    return lambda name: hasattr(lib, name)


def test_product_exports_every_declared_symbol():
    import paper_2512_14946_b200 as pkg
    if not os.path.exists(pkg.LIB_PATH):
        pytest.fail(f"{pkg.LIB_PATH} not built (run __graft_entry__.build())")
    has = _exports(pkg.LIB_PATH)
    placement, codec, extra = declared()
    missing = [f"kvt_{n}" for n in placement + codec + extra if not has(f"kvt_{n}")]
    assert not missing, missing


def test_checkers_export_the_placement_abi():
    placement, codec, _ = declared()
    orc = os.path.join(ROOT, "oracle", "liboracle.so")
    has = _exports(orc)
    assert not [n for n in placement + codec if not has("orc_" + n)]
    ref = os.path.join(ROOT, "oracle", "_ref", "libkvtier_ref.so")
    if os.path.exists(ref):
        has = _exports(ref)
        assert not [n for n in placement if not has("ref_" + n)]


def test_product_fails_loudly_without_library(tmp_path, monkeypatch):
    import paper_2512_14946_b200 as pkg
    monkeypatch.setattr(pkg, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(pkg, "_PRODUCT", None)
    with pytest.raises(RuntimeError, match="missing"):
        pkg.product()


def test_product_refuses_to_run_without_a_gpu():
    """No CPU fallback: on a box without a visible CUDA device the product
    handle cannot be created (KVT_ECUDA) — the caller gets an error, never a
    silently CPU-computed result."""
    import torch

    import paper_2512_14946_b200 as pkg
    from paper_2512_14946_b200 import _abi as A
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    abi = pkg.product()
    h = C.c_void_p()
    assert abi.create(0, None, C.byref(h)) == A.KVT_ECUDA
    assert b"CUDA" in abi.last_error()
