"""Host-side mirror of the reference's interaction-evaluator and rigid-body API.

`Simulation` drives one device context through the C ABI (include/sphg.h).
Method names follow SPEC's operations so callers read like the reference's
scenario driver (SPEC:525-533 `step`, SPEC:243-363 per-op evaluators,
SPEC:328-354 body reductions); each evaluator runs the corresponding bulk
stage over the whole store on the GPU.

There is no CPU fallback: constructing a Simulation without the CUDA library
(libsphg.so) raises.
"""
import ctypes as C

import numpy as np

from . import abi
from .store import ParticleStore, BODY_DTYPE, bodies_ptr


class SPHError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def dt_limits(params, u_max, m_r, lib=None):
    """compute_dt terms without a device: cfl, viscous, body force, contact, conduction."""
    if lib is None:
        from ._lib import load
        lib = load()
    out = (C.c_double * 5)()
    lib.sphg_dt_limits(C.byref(params), float(u_max), float(m_r), out)
    return list(out)


class Simulation:
    prefix = "sphg_"

    def __init__(self, params, device=0, lib=None):
        if lib is None:
            from ._lib import load
            lib = load()
        self.lib = lib
        self.params = params
        self._h = C.c_void_p()
        rc = self._fn("create")(C.byref(params), int(device), C.byref(self._h))
        if rc != 0:
            raise SPHError(rc, "create failed: " + self.validate(params, lib, self.prefix))
        self.n = 0

    # ------------------------------------------------------------ plumbing
    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc, what):
        if rc != 0:
            msg = self._fn("last_error")(self._h)
            raise SPHError(rc, f"{what}: {msg.decode() if msg else ''}")

    @classmethod
    def validate(cls, params, lib=None, prefix=None):
        """validate_config (config.hpp:110-167): '' if valid, else messages joined by newlines."""
        if lib is None:
            from ._lib import load
            lib = load()
        buf = C.create_string_buffer(4096)
        getattr(lib, (prefix or cls.prefix) + "validate")(C.byref(params), buf, len(buf))
        return buf.value.decode()

    def close(self):
        if self._h:
            self._fn("destroy")(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------ state
    def upload(self, store, bodies=None):
        soa = store.soa()
        nb = 0 if bodies is None else len(bodies)
        self._check(self._fn("upload")(self._h, C.byref(soa), bodies_ptr(bodies), nb), "upload")
        self.n = store.n

    def upload_state(self, pos, vel):
        """Warm kinematic update (positions, velocities; gid order, (n,3) float64). Either may be None."""
        dp = C.POINTER(C.c_double)
        pp = None if pos is None else np.ascontiguousarray(pos, np.float64)
        vv = None if vel is None else np.ascontiguousarray(vel, np.float64)
        self._check(self._fn("upload_state")(self._h, pp.ctypes.data_as(dp) if pp is not None else None,
                                             vv.ctypes.data_as(dp) if vv is not None else None, self.n),
                    "upload_state")

    def num_bodies(self):
        nb = C.c_size_t(0)
        self._check(self._fn("num_bodies")(self._h, C.byref(nb)), "num_bodies")
        return nb.value

    def download(self, store=None, fields=None):
        """Returns (ParticleStore, bodies) in gid order."""
        if store is None:
            store = ParticleStore(self.n)
        soa = store.soa(fields)
        nb = C.c_size_t(self.num_bodies())
        bodies = np.zeros(nb.value, BODY_DTYPE)
        self._check(self._fn("download")(self._h, C.byref(soa), bodies_ptr(bodies), C.byref(nb)), "download")
        return store, bodies

    # ------------------------------------------------------------ stepping
    def initialize(self):
        self._check(self._fn("initialize")(self._h), "initialize")

    def step(self, nsteps=1):
        """step(state, dt), nsteps times."""
        self._check(self._fn("step")(self._h, int(nsteps)), "step")

    def step_download(self, nsteps=1, store=None, fields=None):
        """nsteps steps, then download() of `fields` — one call, so the fields that are final before
        the last step's force pass (positions, density, pressure, wall state, mass, tags) are copied
        to the host while the forces run.  Returns (ParticleStore, bodies) like download()."""
        if store is None:
            store = ParticleStore(self.n)
        soa = store.soa(fields)
        nb = C.c_size_t(self.num_bodies())
        bodies = np.zeros(nb.value, BODY_DTYPE)
        rc = self._fn("step_download")(self._h, int(nsteps), C.byref(soa), bodies_ptr(bodies), C.byref(nb))
        self._check(rc, "step_download")
        if nb.value != len(bodies):  # bodies spawned during the steps
            bodies = np.zeros(nb.value, BODY_DTYPE)
            self._check(self._fn("download")(self._h, C.byref(store.soa(())), bodies_ptr(bodies), C.byref(nb)),
                        "download")
        return store, bodies

    def run_stage(self, stage):
        self._check(self._fn("run_stage")(self._h, int(stage)), abi.STAGE_NAMES[stage])

    # SPEC operation names (bulk over the store)
    def build_pairs(self):
        """partition/migrate rebin + build_pairs."""
        self.run_stage(abi.STAGE_REBUILD)

    def density_summation(self):
        """density_summation + eos_pressure."""
        self.run_stage(abi.STAGE_DENSITY)

    def conduction_rhs(self):
        """apply_thermal_dirichlet + conduction_rhs + explicit T update; with
        params.diffusion also the concentration analogue (one stage)."""
        self.run_stage(abi.STAGE_HEAT)

    def diffusion_rhs(self):
        """Dirichlet concentration + diffusion_rhs + explicit C update; shares the
        stage with conduction_rhs (both run when enabled)."""
        self.run_stage(abi.STAGE_HEAT)

    def extrapolate_wall_quantities(self):
        self.run_stage(abi.STAGE_EXTRAPOLATE)

    def momentum_rhs(self):
        """momentum_rhs + coupling_force_on_rigid + contact_force."""
        self.run_stage(abi.STAGE_FORCES)

    def reduce_force_torque(self):
        self.run_stage(abi.STAGE_BODIES)

    def reduce_mass_quantities(self):
        self.run_stage(abi.STAGE_MASS)

    def apply_transitions(self):
        """detect_transitions + apply_transitions + split_disconnected_bodies."""
        self.run_stage(abi.STAGE_TRANSITIONS)

    # ------------------------------------------------------------ inspection
    def get_cells(self):
        cell = np.zeros(self.n, np.int64)
        order = np.zeros(self.n, np.uint32)
        self._check(self._fn("get_cells")(self._h, cell.ctypes.data_as(C.POINTER(C.c_int64)),
                                          order.ctypes.data_as(C.POINTER(C.c_uint32))), "get_cells")
        return cell, order

    def get_nlist(self, offsets_only=False):
        """Verlet candidate lists (CSR by gid, rows gid-sorted); offsets_only: just the n+1 offsets."""
        off = np.zeros(self.n + 1, np.int64)
        self._check(self._fn("get_nlist")(self._h, off.ctypes.data_as(C.POINTER(C.c_int64)), None), "get_nlist")
        if offsets_only:
            return off
        nbr = np.zeros(int(off[-1]), np.uint32)
        self._check(self._fn("get_nlist")(self._h, off.ctypes.data_as(C.POINTER(C.c_int64)),
                                          nbr.ctypes.data_as(C.POINTER(C.c_uint32))), "get_nlist")
        return off, nbr

    def stats(self):
        s = abi.Stats()
        self._check(self._fn("stats")(self._h, C.byref(s)), "stats")
        return s

    def set_timing(self, enabled=True):
        self._check(self._fn("set_timing")(self._h, int(bool(enabled))), "set_timing")

    def set_wall_motion(self, n_groups, velocity, acceleration=None):
        """Moving wall groups (WallGroup<3>, config.hpp:35-51): boundary particles with group g <
        n_groups move with velocity(g, t) -> 3 floats; acceleration(g, t) defaults to the
        reference's central difference.  velocity=None fixes the walls again."""
        if velocity is None:
            self._wall_cb = None
            self._check(self._fn("set_wall_motion")(self._h, 0, abi.WALL_MOTION_FN(), None), "set_wall_motion")
            return

        def cb(g, t, vel, acc, user):
            v = velocity(int(g), float(t))
            for k in range(3):
                vel[k] = float(v[k])
            if acceleration is not None:
                a = acceleration(int(g), float(t))
                for k in range(3):
                    acc[k] = float(a[k])

        self._wall_cb = abi.WALL_MOTION_FN(cb)  # keep the thunk alive as long as the context uses it
        self._check(self._fn("set_wall_motion")(self._h, int(n_groups), self._wall_cb, None), "set_wall_motion")

    def shepard_grid(self, origin, spacing, dims, field=abi.FIELD_VELOCITY, kinds=(abi.FLUID,)):
        """shepard_interpolate on a regular grid (OutputPlan::shepard_grid,
        config.hpp:53-59).  Returns (values[dims..., ncomp] with NaN where unsupported, support)."""
        o = np.ascontiguousarray(origin, np.float64)
        sp = np.ascontiguousarray(spacing, np.float64)
        d = np.ascontiguousarray(dims, np.int32)
        nc = 3 if field == abi.FIELD_VELOCITY else 1
        out = np.zeros(int(np.prod(d)) * nc)
        sup = np.zeros(int(np.prod(d)), np.uint8)
        mask = 0
        for k in kinds:
            mask |= 1 << int(k)
        dp = C.POINTER(C.c_double)
        self._check(self._fn("shepard_grid")(self._h, o.ctypes.data_as(dp), sp.ctypes.data_as(dp),
                                             d.ctypes.data_as(C.POINTER(C.c_int32)), int(field), mask,
                                             out.ctypes.data_as(dp), sup.ctypes.data_as(C.POINTER(C.c_uint8))),
                    "shepard_grid")
        return out.reshape(tuple(d) + (nc,)), sup.reshape(tuple(d)).astype(bool)

    def set_event_log(self, enabled=True):
        """Record every applied transition (SPEC:502 event log); drained by transition_events()."""
        self._check(self._fn("set_event_log")(self._h, int(bool(enabled))), "set_event_log")

    def transition_events(self):
        """The transitions recorded since the last call: structured array (step, gid, direction 1 melt /
        2 solidify, body_from, body_to), ordered by step then gid."""
        n = C.c_size_t(0)
        self._check(self._fn("transition_events")(self._h, None, 0, C.byref(n)), "transition_events")
        buf = (abi.Event * max(n.value, 1))()
        self._check(self._fn("transition_events")(self._h, buf, n.value, C.byref(n)), "transition_events")
        dt = np.dtype([("step", "i8"), ("gid", "u4"), ("direction", "i4"), ("body_from", "i4"), ("body_to", "i4")])
        assert dt.itemsize == C.sizeof(abi.Event)
        return np.frombuffer(bytes(buf), dt, count=n.value).copy()

    def cell_occupancy(self, nbins=1024):
        """SPEC:218 cell-occupancy histogram of the last rebuild: (hist[k] = cells holding k particles, the
        last bin >= nbins - 1; the fullest cell's count)."""
        hist = np.zeros(nbins, np.int64)
        mx = C.c_int64(0)
        self._check(self._fn("cell_occupancy")(self._h, hist.ctypes.data_as(C.POINTER(C.c_int64)), nbins,
                                               C.byref(mx)), "cell_occupancy")
        return hist, mx.value

    # ------------------------------------------------ decomposed transition batches (sphg.h)
    def event_bodies(self, mask):
        """OR into `mask` (uint8, one per body) the bodies this rank's detected events can touch."""
        assert mask.dtype == np.uint8 and mask.flags.c_contiguous
        self._check(self._fn("event_bodies")(self._h, mask.ctypes.data_as(C.POINTER(C.c_uint8)), len(mask)),
                    "event_bodies")
        return mask

    def event_members(self, mask):
        """Local ids (ascending) of the owned event particles and owned members of the masked bodies."""
        mask = np.ascontiguousarray(mask, np.uint8)
        mp = mask.ctypes.data_as(C.POINTER(C.c_uint8))
        n = C.c_size_t(0)
        self._check(self._fn("event_members")(self._h, mp, len(mask), None, 0, C.byref(n)), "event_members")
        ids = np.zeros(max(n.value, 1), np.uint32)
        self._check(self._fn("event_members")(self._h, mp, len(mask), ids.ctypes.data_as(C.POINTER(C.c_uint32)),
                                              len(ids), C.byref(n)), "event_members")
        return ids[: n.value]

    def record_doubles(self):
        return int(self._fn("record_doubles")())

    @staticmethod
    def _ptr(a):
        """Address of a C-contiguous numpy array or torch tensor (host or device)."""
        return C.c_void_p(a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data)

    def record_pack(self, ids, out=None):
        """Records (sphg.h) of the particles with local ids `ids` -> (m, record_doubles) float64; ids / out
        may be numpy arrays or torch tensors (uint32 / int32 ids; device tensors stay on the device)."""
        if not hasattr(ids, "data_ptr"):
            ids = np.ascontiguousarray(ids, np.uint32)
        if out is None:
            out = np.zeros((len(ids), self.record_doubles()))
        self._check(self._fn("record_pack")(self._h, self._ptr(ids), len(ids), self._ptr(out)), "record_pack")
        return out

    def record_unpack(self, ids, recs, keep_position=True):
        if not hasattr(ids, "data_ptr"):
            ids = np.ascontiguousarray(ids, np.uint32)
            recs = np.ascontiguousarray(recs, np.float64)
            assert recs.shape == (len(ids), self.record_doubles())
        self._check(self._fn("record_unpack")(self._h, self._ptr(ids), len(ids), self._ptr(recs),
                                              int(bool(keep_position))), "record_unpack")

    def upload_records(self, recs, n_owned, bodies):
        """Replace the whole store by `recs` (the first n_owned owned, the rest ghosts) and the body table;
        recs may be a device tensor (no host round trip)."""
        n = int(recs.shape[0])
        if not hasattr(recs, "data_ptr"):
            recs = np.ascontiguousarray(recs, np.float64)
        bodies = np.ascontiguousarray(bodies, BODY_DTYPE)
        self._check(self._fn("upload_records")(self._h, n, int(n_owned), self._ptr(recs) if n else None,
                                               self._ptr(bodies) if len(bodies) else None, len(bodies)),
                    "upload_records")
        self.n = n

    def replace_bodies(self, bodies):
        bodies = np.ascontiguousarray(bodies, BODY_DTYPE)
        self._check(self._fn("replace_bodies")(self._h, bodies_ptr(bodies), len(bodies)), "replace_bodies")

    def counters(self):
        """Cheap host counters: (steps, rebuilds, host_syncs, kernel_launches)."""
        out = (C.c_int64 * 4)()
        self._check(self._fn("counters")(self._h, out), "counters")
        return tuple(out)

    def count_pairs(self):
        """(candidates, interacting, interacting with fluid i, interacting with non-fluid i)."""
        out = (C.c_int64 * 4)()
        self._check(self._fn("count_pairs")(self._h, out), "count_pairs")
        return tuple(out)

    def compute_dt(self):
        """compute_dt terms: cfl, viscous, body force, contact, conduction."""
        out = (C.c_double * 5)()
        self._check(self._fn("compute_dt")(self._h, out), "compute_dt")
        return list(out)
