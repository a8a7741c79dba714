"""B200-native EvicPress hot path: KV codec + utility scoring + greedy
placement, hand-written sm_100a CUDA behind the C ABI in include/kvt_b200.h.

The product library is libkvt_b200.so, built in-tree by
`python -c "import __graft_entry__ as g; g.build()"` (or `make -C
paper_2512_14946_b200/csrc`). There is no CPU fallback: `product()` raises
when the library is missing, and every call fails with KVT_ECUDA when no GPU
is visible.
"""
from __future__ import annotations

import os

from . import _abi

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libkvt_b200.so")

_PRODUCT = None


def product() -> _abi.Abi:
    """Bind the CUDA implementation (kvt_* symbols). Fails loudly if unbuilt."""
    global _PRODUCT
    if _PRODUCT is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        _PRODUCT = _abi.Abi(LIB_PATH, "kvt_", codec=True, extra=True)
    return _PRODUCT


__all__ = ["product", "LIB_PATH"]
