"""The C-ABI shared library loads without a GPU and exports every entry point the public
headers declare (include/sb_kernels.h, include/sb_host.h). No compute calls here."""
import ctypes
import os
import re

from paper_2604_13847_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header, pattern):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(pattern, text)))


def test_kernel_abi_exported():
    lib = _native.lib()
    names = declared("sb_kernels.h", r"\b(sb_[a-z0-9_]+)\s*\(")
    assert len(names) >= 12, names
    for n in names:
        assert hasattr(lib, n), f"missing export {n}"


def test_host_abi_exported():
    lib = _native.lib()
    names = [n for n in declared("sb_host.h", r"SBH\(([a-z0-9_]+)\)") if n != "name"]
    assert len(names) >= 18, names
    for n in names:
        assert hasattr(lib, "sbh_" + n), f"missing export sbh_{n}"


def test_only_abi_symbols_exported():
    """-fvisibility=hidden: the C++ host layer's internals do not leak (no clash with a
    reference build loaded in the same process)."""
    out = os.popen(f"nm -D --defined-only {_native.LIB_PATH}").read()
    ours = [l.split()[-1] for l in out.splitlines() if " T " in l]
    assert ours and all(s.startswith(("sb_", "sbh_")) for s in ours if not s.startswith("_")), ours[:20]


def test_block_layout_host_no_gpu():
    """The one host-side helper of the kernel ABI runs without a device."""
    lib = _native.lib()
    cu = (ctypes.c_int32 * 4)(0, 300, 300, 1000)
    blk = (ctypes.c_int32 * 4)()
    tri = (ctypes.c_int64 * 4)()
    nbt, nbm = ctypes.c_int(), ctypes.c_int()
    trit = ctypes.c_int64()
    assert lib.sb_block_layout_host(cu, 3, 128, blk, tri, ctypes.byref(nbt), ctypes.byref(trit), ctypes.byref(nbm)) == 0
    assert list(blk) == [0, 3, 3, 9] and list(tri) == [0, 6, 6, 27] and nbt.value == 9 and nbm.value == 6
    assert lib.sb_block_layout_host(cu, 3, 96, blk, tri, ctypes.byref(nbt), ctypes.byref(trit), ctypes.byref(nbm)) == 1
