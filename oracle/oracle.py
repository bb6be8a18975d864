"""ctypes binding of the CPU oracle (oracle/_ref/libsph_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py, never by the product package.
"""
import ctypes as C
import os

import numpy as np

from paper_2103_07925_b200 import abi
from paper_2103_07925_b200.sim import Simulation

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libsph_oracle.so")
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"oracle not built: {LIB_PATH} (run `make -C oracle` where /root/reference exists)")
        lib = C.CDLL(LIB_PATH)
        abi.declare(lib, "orc_")
        dp = C.POINTER(C.c_double)
        lib.orc_get_scales.argtypes = [C.c_void_p] + [dp] * 7
        lib.orc_get_scales.restype = C.c_int
        lib.orc_get_pscales.argtypes = [C.c_void_p, dp, dp]
        lib.orc_get_pscales.restype = C.c_int
        lib.orc_get_scale_dC.argtypes = [C.c_void_p, dp]
        lib.orc_get_scale_dC.restype = C.c_int
        for f in ("orc_kernel_w", "orc_kernel_dw"):
            getattr(lib, f).argtypes = [C.c_double, C.c_double]
            getattr(lib, f).restype = C.c_double
        lib.orc_kernel_sigma.argtypes = [C.c_double]
        lib.orc_kernel_sigma.restype = C.c_double
        lib.orc_eos_pressure.argtypes = [C.c_double] * 3
        lib.orc_eos_pressure.restype = C.c_double
        lib.orc_orientation_step.argtypes = [dp, dp, C.c_double, dp]
        lib.orc_rotate.argtypes = [dp, dp, dp]
        lib.orc_kahan_sum.argtypes = [dp, C.c_size_t]
        lib.orc_kahan_sum.restype = C.c_double
        lib.orc_particle_inertia.argtypes = [C.c_double, C.c_double]
        lib.orc_particle_inertia.restype = C.c_double
        lib.orc_seed_lattice_box.argtypes = [dp, dp, C.c_double, dp, C.c_size_t]
        lib.orc_seed_lattice_box.restype = C.c_size_t
        lib.orc_seed_lattice_ball.argtypes = [dp, C.c_double, C.c_double, dp, C.c_size_t]
        lib.orc_seed_lattice_ball.restype = C.c_size_t
        for f in ("orc_sizeof_params", "orc_sizeof_body", "orc_sizeof_soa"):
            getattr(lib, f).restype = C.c_size_t
        _lib = lib
    return _lib


class Oracle(Simulation):
    """Same interface as the product's Simulation, backed by the CPU oracle."""
    prefix = "orc_"

    def __init__(self, params):
        super().__init__(params, 0, load())

    @classmethod
    def validate(cls, params, lib=None, prefix=None):
        return Simulation.validate(params, lib or load(), "orc_")

    def scales(self):
        """Per-particle sums of |pair contributions| (DESIGN.md §5 tolerance metric), plus acc_p /
        force_p: the pressure sensitivity sum |d term/d p| c^2 rho (absolute EOS allowance)."""
        n = self.n
        nb = self.num_bodies()
        out = {k: np.zeros(n) for k in ("acc", "acc_bg", "dT_dt", "force", "density")}
        bf, bt = np.zeros(max(nb, 1)), np.zeros(max(nb, 1))
        dp = C.POINTER(C.c_double)
        self._check(self.lib.orc_get_scales(self._h, *[out[k].ctypes.data_as(dp) for k in
                                                       ("acc", "acc_bg", "dT_dt", "force", "density")],
                                            bf.ctypes.data_as(dp), bt.ctypes.data_as(dp)), "scales")
        out["body_force"], out["body_torque"] = bf[:nb], bt[:nb]
        out["dC_dt"] = np.zeros(n)
        out["acc_p"], out["force_p"] = np.zeros(n), np.zeros(n)
        if n:
            self._check(self.lib.orc_get_scale_dC(self._h, out["dC_dt"].ctypes.data_as(dp)), "scales")
            self._check(self.lib.orc_get_pscales(self._h, out["acc_p"].ctypes.data_as(dp),
                                                 out["force_p"].ctypes.data_as(dp)), "scales")
        return out


def seed_lattice_box(lo, hi, dx):
    lib = load()
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    dp = C.POINTER(C.c_double)
    n = lib.orc_seed_lattice_box(lo.ctypes.data_as(dp), hi.ctypes.data_as(dp), dx, None, 0)
    out = np.zeros((n, 3))
    lib.orc_seed_lattice_box(lo.ctypes.data_as(dp), hi.ctypes.data_as(dp), dx, out.ctypes.data_as(dp), n)
    return out


def seed_lattice_ball(center, diameter, dx):
    lib = load()
    c = np.ascontiguousarray(center, np.float64)
    dp = C.POINTER(C.c_double)
    n = lib.orc_seed_lattice_ball(c.ctypes.data_as(dp), diameter, dx, None, 0)
    out = np.zeros((n, 3))
    lib.orc_seed_lattice_ball(c.ctypes.data_as(dp), diameter, dx, out.ctypes.data_as(dp), n)
    return out
