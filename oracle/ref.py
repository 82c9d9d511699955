"""Bind the compiled reference host library (oracle/_ref/libsbref.so). Test infrastructure."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libsbref.so")


def available() -> bool:
    return os.path.exists(REF_LIB)


_api = None


def api():
    global _api
    if _api is None:
        from paper_2604_13847_b200.host import HostAPI

        if not available():
            raise FileNotFoundError(f"{REF_LIB} not built (make -C oracle ref; needs /root/reference)")
        _api = HostAPI(ctypes.CDLL(REF_LIB, mode=ctypes.RTLD_LOCAL), "sbref_")
    return _api
