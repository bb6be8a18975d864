"""Host-side mirror of sphfsi::ParticleStore<3> (store.hpp:24-100) and the body table.

The fields, their order, dtypes and the interleaved-xyz layout of Vec<3>
fields are those of the reference container, so a C++ caller can hand its
ParticleStore vectors to the C ABI unchanged.  The
concentration fields (store.hpp:36-37,45) carry the diffusion extension (SURVEY
§8(f) f2).
"""
import ctypes as C

import numpy as np

from . import abi

VEC_FIELDS = ("pos", "vel", "vel_adv", "acc", "acc_bg", "body_frame_pos", "wall_velocity", "force")
SCALAR_FIELDS = ("density", "pressure", "mass", "temperature", "dT_dt", "wall_pressure", "concentration", "dC_dt")
TAG_FIELDS = {"kind": np.uint8, "group": np.uint32, "material": np.uint16, "dirichlet_T": np.uint8,
              "owner": np.uint32, "dirichlet_C": np.uint8}

BODY_DTYPE = np.dtype([
    ("mass", "f8"), ("com", "f8", 3), ("inertia", "f8", 6), ("q", "f8", 4),
    ("vel", "f8", 3), ("omega", "f8", 3), ("force", "f8", 3), ("torque", "f8", 3),
    ("acc", "f8", 3), ("alpha", "f8", 3),
    ("material", "i4"), ("mobile", "i4"), ("alive", "i4"), ("pad", "i4")])
assert BODY_DTYPE.itemsize == C.sizeof(abi.Body)


class ParticleStore:
    """SoA particle store in gid order (gid = index)."""

    def __init__(self, n=0):
        self.n = int(n)
        for f in VEC_FIELDS:
            setattr(self, f, np.zeros((self.n, 3), np.float64))
        for f in SCALAR_FIELDS:
            setattr(self, f, np.zeros(self.n, np.float64))
        for f, dt in TAG_FIELDS.items():
            setattr(self, f, np.zeros(self.n, dt))
        self.dirichlet_T[:] = abi.NO_DIRICHLET
        self.dirichlet_C[:] = abi.NO_DIRICHLET

    def __len__(self):
        return self.n

    def size(self):
        return self.n

    def copy(self):
        s = ParticleStore(0)
        s.n = self.n
        for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS):
            setattr(s, f, getattr(self, f).copy())
        return s

    def nbytes(self):
        return sum(getattr(self, f).nbytes for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS))

    def soa(self, fields=None):
        """ctypes SoA view (the arrays must stay alive while it is used)."""
        s = abi.SoA()
        s.n = self.n
        for f in VEC_FIELDS + SCALAR_FIELDS:
            a = getattr(self, f)
            if fields is not None and f not in fields:
                continue
            assert a.dtype == np.float64 and a.flags.c_contiguous
            setattr(s, f, a.ctypes.data_as(C.POINTER(C.c_double)))
        for f, dt in TAG_FIELDS.items():
            if fields is not None and f not in fields:
                continue
            a = getattr(self, f)
            assert a.dtype == dt and a.flags.c_contiguous
            ctype = {np.uint8: C.c_uint8, np.uint16: C.c_uint16, np.uint32: C.c_uint32}[dt]
            setattr(s, f, a.ctypes.data_as(C.POINTER(ctype)))
        return s


def empty_bodies(nb):
    b = np.zeros(nb, BODY_DTYPE)
    b["q"][:, 0] = 1.0
    b["mobile"] = 1
    b["alive"] = 1
    return b


def bodies_ptr(b):
    if b is None or len(b) == 0:
        return C.POINTER(abi.Body)()
    assert b.dtype == BODY_DTYPE and b.flags.c_contiguous
    return b.ctypes.data_as(C.POINTER(abi.Body))
