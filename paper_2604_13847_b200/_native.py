"""Loader for the in-tree native library (host decision layer + sm_100a kernels).

There is no fallback: if ``lib/libsparsebalance_b200.so`` is missing the import fails
loudly and tells the caller to run ``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SB_LIB_PATH: experiment builds only (e.g. tools/ A/B timing); the product path is the in-tree lib.
LIB_PATH = os.environ.get("SB_LIB_PATH") or os.path.join(_HERE, "lib", "libsparsebalance_b200.so")

_lib = None


class NativeError(RuntimeError):
    """Runtime / CUDA failure reported by the native layer (return code 2)."""


class ConfigError(ValueError):
    """Invalid argument reported by the native layer (return code 1).

    Mirrors sparsebalance::ConfigError (reference errors.hpp:11-17)."""


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native library not built: {LIB_PATH} (run `python -c 'import __graft_entry__ as g; g.build()'`)"
            )
        _lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_LOCAL)
    return _lib


def check(rc: int, last_error) -> None:
    if rc == 0:
        return
    msg = last_error().decode() if last_error is not None else ""
    if rc == 1:
        raise ConfigError(msg)
    raise NativeError(msg or f"native call failed with code {rc}")
