"""Loads the in-tree CUDA library libsphg.so.  Fails loudly when it is missing:
there is no CPU fallback for the hot path."""
import ctypes as C
import os

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, os.environ.get("SPHG_LIB", "libsphg.so"))
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"CUDA extension missing: {LIB_PATH} — run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        abi.declare(lib, "sphg_")
        lib.sphg_sizeof_params.restype = C.c_size_t
        lib.sphg_sizeof_body.restype = C.c_size_t
        lib.sphg_sizeof_soa.restype = C.c_size_t
        _lib = lib
    return _lib
