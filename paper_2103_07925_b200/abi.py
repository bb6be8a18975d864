"""ctypes mirror of include/sphg.h (the C ABI of the hot path).

Struct layouts must match the header exactly; tests/test_abi.py checks the
sizes against the compiled libraries.
"""
import ctypes as C

MAX_MAT = 8
MAX_DIRICHLET = 8
MAX_PIECES = 8
NO_MATERIAL = -1
NO_DIRICHLET = 0xFF

FLUID, RIGID, BOUNDARY = 0, 1, 2  # store.hpp:11 Kind

OK, ERR_CONFIG, ERR_RUNTIME, ERR_CUDA = 0, 2, 3, 4
NEED_PARTITION = 5  # sphg_step stopped before a step its partition may not cover (not an error)
NEED_TRANSITIONS = 6  # a decomposed step detected phase transitions: the caller applies the batch (not an error)
DT_REFUSE, DT_WARN, DT_OFF = 0, 1, 2  # sphg_params.dt_check
DT_TERMS = ("cfl", "viscous", "body force", "contact", "conduction")  # compute_dt order

STAGE_REBUILD = 0
STAGE_DENSITY = 1
STAGE_HEAT = 2
STAGE_EXTRAPOLATE = 3
STAGE_FORCES = 4
STAGE_BODIES = 5
STAGE_KICK_DRIFT = 6
STAGE_FINAL_KICK = 7
STAGE_TRANSITIONS = 8
STAGE_MASS = 9

HALO_STATE, HALO_DENSITY, HALO_WALL = 0, 1, 2
XCHG_MAX, XCHG_BODIES = 3, 4  # exchange phases of the in-library decomposed step (sphg_set_exchange)
TRANSITIONS_NONE, TRANSITIONS_TEMPERATURE, TRANSITIONS_CONCENTRATION = 0, 1, 2  # config.hpp:61
FIELD_VELOCITY, FIELD_TEMPERATURE, FIELD_CONCENTRATION, FIELD_PRESSURE, FIELD_DENSITY = 0, 1, 2, 3, 4
MAX_HALO_SLOTS = 64

STAGE_NAMES = ["rebuild", "density", "heat", "extrapolate", "forces", "bodies",
               "kick_drift", "final_kick", "transitions", "mass", "forces_fluid", "forces_rigid",
               "", "", "", ""]


class Material(C.Structure):
    """sphfsi::Material (material.hpp:17-36) + per-material body force (config.hpp:79)."""
    _fields_ = [("rho0", C.c_double), ("nu", C.c_double), ("cp", C.c_double),
                ("kappa", C.c_double), ("c", C.c_double), ("pb", C.c_double),
                ("T_t", C.c_double), ("melt_target", C.c_int32),
                ("solidify_target", C.c_int32), ("body_force", C.c_double * 3),
                ("D", C.c_double), ("C_t", C.c_double)]


class Schedule(C.Structure):
    """sphfsi::Schedule (config.hpp:20-33)."""
    _fields_ = [("n", C.c_int32), ("pad", C.c_int32),
                ("t_end", C.c_double * MAX_PIECES), ("value", C.c_double * MAX_PIECES)]


MAX_BUFFERS = 4


class Buffer(C.Structure):
    """sphg_buffer: inflow / outflow buffer zone with a prescribed (parabolic) velocity [P23]."""
    _fields_ = [("axis", C.c_int32), ("profile_axis", C.c_int32), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("u_mean", C.c_double), ("t_start", C.c_double)]


class Params(C.Structure):
    """Flat POD of sphfsi::ScenarioConfig<3> (config.hpp:68-106)."""
    _fields_ = [("dx", C.c_double), ("h", C.c_double), ("dt", C.c_double), ("t0", C.c_double),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("periodic", C.c_int32 * 3), ("n_mat", C.c_int32),
                ("cell_edge_override", C.c_double),
                ("mat", Material * MAX_MAT),
                ("kc", C.c_double), ("dc", C.c_double),
                ("tvf", C.c_int32), ("thermal", C.c_int32), ("transitions", C.c_int32),
                ("n_dirichlet", C.c_int32),
                ("dirichlet_T", Schedule * MAX_DIRICHLET),
                ("default_fluid_mat", C.c_int32), ("nlist_capacity", C.c_int32),
                ("rank", C.c_int32), ("nranks", C.c_int32),
                ("diffusion", C.c_int32), ("n_dirichlet_c", C.c_int32),
                ("dirichlet_C", Schedule * MAX_DIRICHLET),
                # moving Gaussian surface heat flux (C4, [P21]; not in the reference)
                ("heat_source", C.c_int32), ("hs_material_mask", C.c_uint32),
                ("hs_power", C.c_double), ("hs_radius", C.c_double),
                ("hs_origin", C.c_double * 3), ("hs_velocity", C.c_double * 3),
                # runtime time-step assertion: DT_REFUSE / DT_WARN / DT_OFF
                ("dt_check", C.c_int32), ("n_buffers", C.c_int32), ("buffers", Buffer * MAX_BUFFERS)]


_dp = C.POINTER(C.c_double)


class SoA(C.Structure):
    """Host views of a ParticleStore<3> (store.hpp:26-46), gid order."""
    _fields_ = [("n", C.c_size_t),
                ("pos", _dp), ("vel", _dp), ("vel_adv", _dp), ("acc", _dp), ("acc_bg", _dp),
                ("density", _dp), ("pressure", _dp), ("mass", _dp), ("temperature", _dp),
                ("dT_dt", _dp),
                ("kind", C.POINTER(C.c_uint8)), ("group", C.POINTER(C.c_uint32)),
                ("material", C.POINTER(C.c_uint16)),
                ("body_frame_pos", _dp), ("wall_pressure", _dp), ("wall_velocity", _dp),
                ("dirichlet_T", C.POINTER(C.c_uint8)), ("force", _dp),
                ("owner", C.POINTER(C.c_uint32)),
                ("concentration", _dp), ("dC_dt", _dp), ("dirichlet_C", C.POINTER(C.c_uint8))]


class Body(C.Structure):
    """RigidBody."""
    _fields_ = [("mass", C.c_double), ("com", C.c_double * 3), ("inertia", C.c_double * 6),
                ("q", C.c_double * 4), ("vel", C.c_double * 3), ("omega", C.c_double * 3),
                ("force", C.c_double * 3), ("torque", C.c_double * 3),
                ("acc", C.c_double * 3), ("alpha", C.c_double * 3),
                ("material", C.c_int32), ("mobile", C.c_int32), ("alive", C.c_int32),
                ("pad", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("rebuilds", C.c_int64), ("n_pairs_candidate", C.c_int64),
                ("transitions_melt", C.c_int64), ("transitions_solidify", C.c_int64),
                ("bodies_alive", C.c_int64), ("nlist_capacity", C.c_int32),
                ("max_neighbours", C.c_int32), ("cells", C.c_int32 * 3), ("pad", C.c_int32),
                ("time", C.c_double), ("max_displacement", C.c_double), ("u_max", C.c_double),
                ("stage_ms", C.c_double * 16), ("kernel_launches", C.c_int64),
                ("last_step_call_ms", C.c_double), ("graph_captures", C.c_int64),
                ("graph_replays", C.c_int64), ("dt_violations", C.c_int64), ("host_syncs", C.c_int64),
                ("dt_term", C.c_int32),
                ("pad3", C.c_int32), ("dt_limit", C.c_double)]


class Event(C.Structure):
    """sphg_event: one applied transition (SPEC:502 event log)."""
    _fields_ = [("step", C.c_int64), ("gid", C.c_uint32), ("direction", C.c_int32),
                ("body_from", C.c_int32), ("body_to", C.c_int32)]


MELT, SOLIDIFY = 1, 2  # sphg_event.direction


# int fn(int32 phase, void* stream, void* user)  (sphg_set_exchange)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_int32, C.c_void_p, C.c_void_p)

# void fn(int32 group, double t, double vel[3], double acc[3], void* user)  (sphg_set_wall_motion)
WALL_MOTION_FN = C.CFUNCTYPE(None, C.c_int32, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double),
                             C.c_void_p)
MAX_WALL_GROUPS = 8


def declare(lib, prefix):
    """Attach argtypes/restypes for the sphg_* (or orc_*) entry points."""
    vp = C.c_void_p
    sig = {
        "create": (C.c_int, [C.POINTER(Params), C.c_int, C.POINTER(vp)]),
        "upload": (C.c_int, [vp, C.POINTER(SoA), C.POINTER(Body), C.c_size_t]),
        "initialize": (C.c_int, [vp]),
        "step": (C.c_int, [vp, C.c_int]),
        "run_stage": (C.c_int, [vp, C.c_int]),
        "download": (C.c_int, [vp, C.POINTER(SoA), C.POINTER(Body), C.POINTER(C.c_size_t)]),
        "get_cells": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_uint32)]),
        "get_nlist": (C.c_int, [vp, C.POINTER(C.c_int64), C.POINTER(C.c_uint32)]),
        "stats": (C.c_int, [vp, C.POINTER(Stats)]),
        "num_bodies": (C.c_int, [vp, C.POINTER(C.c_size_t)]),
        "last_error": (C.c_char_p, [vp]),
        "destroy": (None, [vp]),
        "validate": (C.c_int, [C.POINTER(Params), C.c_char_p, C.c_size_t]),
    }
    optional = {
        "set_timing": (C.c_int, [vp, C.c_int]),
        "compute_dt": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "dt_limits": (C.c_int, [C.POINTER(Params), C.c_double, C.c_double, C.POINTER(C.c_double)]),
        "count_pairs": (C.c_int, [vp, C.POINTER(C.c_int64)]),
        "halo_set": (C.c_int, [vp, C.c_int, C.POINTER(C.c_uint32), C.c_size_t]),
        "halo_pack": (C.c_int, [vp, C.c_int, C.c_int, C.c_void_p]),
        "halo_unpack": (C.c_int, [vp, C.c_int, C.c_int, C.c_void_p]),
        "body_partials": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "body_apply_totals": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "max_displacement": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "halo_doubles": (C.c_int, [C.c_int]),
        "upload_state": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t]),
        "set_wall_motion": (C.c_int, [vp, C.c_int32, WALL_MOTION_FN, C.c_void_p]),
        "set_event_log": (C.c_int, [vp, C.c_int]),
        "set_exchange": (C.c_int, [vp, EXCHANGE_FN, C.c_void_p]),
        "get_stream": (C.c_int, [vp, C.POINTER(C.c_void_p)]),
        "halo_bind": (C.c_int, [vp, C.c_int, C.c_int, C.c_void_p]),
        "max_bind": (C.c_int, [vp, C.c_void_p]),
        "body_bind": (C.c_int, [vp, C.c_void_p, C.c_void_p, C.c_int32]),
        "drift": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "set_partition_limit": (C.c_int, [vp, C.c_double]),
        "counters": (C.c_int, [vp, C.POINTER(C.c_int64)]),
        "transition_events": (C.c_int, [vp, C.POINTER(Event), C.c_size_t, C.POINTER(C.c_size_t)]),
        "cell_occupancy": (C.c_int, [vp, C.POINTER(C.c_int64), C.c_size_t, C.POINTER(C.c_int64)]),
        "event_bodies": (C.c_int, [vp, C.POINTER(C.c_uint8), C.c_size_t]),
        "event_members": (C.c_int, [vp, C.POINTER(C.c_uint8), C.c_size_t, C.POINTER(C.c_uint32), C.c_size_t,
                                    C.POINTER(C.c_size_t)]),
        "record_doubles": (C.c_int, []),
        "record_pack": (C.c_int, [vp, C.c_void_p, C.c_size_t, C.c_void_p]),
        "record_unpack": (C.c_int, [vp, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int]),
        "replace_bodies": (C.c_int, [vp, C.POINTER(Body), C.c_size_t]),
        "upload_records": (C.c_int, [vp, C.c_size_t, C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t]),
        "shepard_grid": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                   C.c_int32, C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_uint8)]),
    }
    for name, (res, args) in list(sig.items()) + list(optional.items()):
        fn = getattr(lib, prefix + name, None)
        if fn is None:
            if name in optional:
                continue
            raise ImportError(f"{prefix}{name} missing from {lib._name}")
        fn.restype = res
        fn.argtypes = args
    return lib
