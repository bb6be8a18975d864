"""Scenario output of the reference's `scenario_io` module, on top
of the device path: particle snapshots, body trajectories, Shepard-filtered grid dumps and the
`run` loop that writes them per an OutputPlan.

Formats (versioned, self-describing, byte-stable for fixed input — SPEC:605-610):

* snapshot (`write_snapshot`): plain columnar text.  Header lines start with `#`:
  `# sphfsi-snapshot 1`, `# dim 3`, `# time <t>`, `# step <k>`, `# particles <n>`,
  `# columns gid x y z kind material u_x u_y u_z rho p T C body`; then one row per particle in gid
  order.  Floats are written with 17 significant digits (`%.17g`, exact fp64 round trip), `body`
  is the body id of a rigid particle and -1 otherwise.  An empty store gives a header-only file.
* trajectory (`TrajectoryWriter`): CSV, header `t,body,alive,mass,r_x,r_y,r_z,u_x,u_y,u_z,
  omega_x,omega_y,omega_z`, one row per body per write.
* grid (`write_grid`): `# sphfsi-grid 1` header with time, origin, spacing, dims, field; rows
  `i j k x y z value... support` in C order of (i, j, k); unsupported points carry `nan`.

The gather that feeds them is the device download (`Simulation.download`, packed into gid order on
the GPU) and the device Shepard gather (`Simulation.shepard_grid`, f4); only the text formatting
runs on the host.  Everything here takes any object with the `Simulation` interface.
"""
import dataclasses
import os

import numpy as np

from . import abi
from .sim import SPHError
from .store import ParticleStore

FORMAT_VERSION = 1
SNAPSHOT_COLUMNS = ("gid", "x", "y", "z", "kind", "material", "u_x", "u_y", "u_z", "rho", "p", "T", "C", "body")
SNAPSHOT_FIELDS = ("pos", "vel", "density", "pressure", "temperature", "concentration", "kind", "material", "group")
TRAJECTORY_COLUMNS = ("t", "body", "alive", "mass", "r_x", "r_y", "r_z", "u_x", "u_y", "u_z",
                      "omega_x", "omega_y", "omega_z")
FIELD_NAMES = {abi.FIELD_VELOCITY: "velocity", abi.FIELD_TEMPERATURE: "temperature",
               abi.FIELD_CONCENTRATION: "concentration", abi.FIELD_PRESSURE: "pressure",
               abi.FIELD_DENSITY: "density"}


def _g(x):
    return "%.17g" % x


def _write_rows(fh, cols, fmts):
    """Columns (equal-length 1-D arrays) -> text rows, vectorised per chunk."""
    n = len(cols[0]) if cols else 0
    chunk = 1 << 16
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        parts = []
        for c, f in zip(cols, fmts):
            v = c[a:b]
            parts.append(np.char.mod(f, v))
        rows = parts[0]
        for p in parts[1:]:
            rows = np.char.add(np.char.add(rows, " "), p)
        fh.write("\n".join(rows.tolist()))
        fh.write("\n")


def write_snapshot(store, t, path, step=0):
    """write_snapshot(store, bodies, t, plan) -> file; `store` is a ParticleStore
    in gid order (e.g. from Simulation.download).  Returns the path."""
    n = store.n
    body = np.where(store.kind == abi.RIGID, store.group.astype(np.int64), -1)
    with open(path, "w", newline="\n") as fh:
        fh.write("# sphfsi-snapshot %d\n# dim 3\n# time %s\n# step %d\n# particles %d\n# columns %s\n"
                 % (FORMAT_VERSION, _g(t), int(step), n, " ".join(SNAPSHOT_COLUMNS)))
        if n:
            cols = [np.arange(n, dtype=np.int64), store.pos[:, 0], store.pos[:, 1], store.pos[:, 2],
                    store.kind.astype(np.int64), store.material.astype(np.int64),
                    store.vel[:, 0], store.vel[:, 1], store.vel[:, 2], store.density, store.pressure,
                    store.temperature, store.concentration, body]
            fmts = ["%d", "%.17g", "%.17g", "%.17g", "%d", "%d"] + ["%.17g"] * 7 + ["%d"]
            _write_rows(fh, cols, fmts)
    return path


def read_snapshot(path):
    """Inverse of write_snapshot: (header dict, {column: array})."""
    header, names = {}, None
    with open(path) as fh:
        lines = fh.read().split("\n")
    body = []
    for ln in lines:
        if ln.startswith("# "):
            k, _, v = ln[2:].partition(" ")
            header[k] = v
        elif ln:
            body.append(ln)
    names = header["columns"].split()
    data = np.array([r.split() for r in body], dtype=object).reshape(len(body), len(names))
    out = {}
    for c, name in enumerate(names):
        col = data[:, c]
        out[name] = (col.astype(np.int64) if name in ("gid", "kind", "material", "body")
                     else np.array([float(x) for x in col], np.float64))
    header["time"] = float(header["time"])
    for k in ("step", "particles", "dim"):
        header[k] = int(header[k])
    return header, out


class TrajectoryWriter:
    """Body trajectories as CSV (`run shear_migration` -> (t, r_y, u_x) of the disk)."""

    def __init__(self, path):
        self.path = path
        with open(path, "w", newline="\n") as fh:
            fh.write(",".join(TRAJECTORY_COLUMNS) + "\n")

    def write(self, t, bodies):
        with open(self.path, "a", newline="\n") as fh:
            for k, b in enumerate(bodies):
                vals = [_g(t), str(k), str(int(b["alive"])), _g(b["mass"])]
                vals += [_g(x) for x in b["com"]] + [_g(x) for x in b["vel"]] + [_g(x) for x in b["omega"]]
                fh.write(",".join(vals) + "\n")


def write_grid(path, t, origin, spacing, dims, field, values, support):
    """Shepard-filtered grid dump: values[dims..., ncomp], support[dims]."""
    dims = tuple(int(d) for d in dims)
    ncomp = values.shape[-1]
    with open(path, "w", newline="\n") as fh:
        fh.write("# sphfsi-grid %d\n# time %s\n# origin %s\n# spacing %s\n# dims %d %d %d\n# field %s\n"
                 % (FORMAT_VERSION, _g(t), " ".join(_g(x) for x in origin), " ".join(_g(x) for x in spacing),
                    dims[0], dims[1], dims[2], FIELD_NAMES.get(field, str(field))))
        comp = ["value"] if ncomp == 1 else ["value_%d" % c for c in range(ncomp)]
        fh.write("# columns i j k x y z %s support\n" % " ".join(comp))
        ii, jj, kk = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
        ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
        xyz = [origin[a] + spacing[a] * idx for a, idx in enumerate((ii, jj, kk))]
        v = values.reshape(-1, ncomp)
        cols = [ii, jj, kk] + xyz + [v[:, c] for c in range(ncomp)] + [support.ravel().astype(np.int64)]
        if len(ii):
            _write_rows(fh, cols, ["%d"] * 3 + ["%.17g"] * (3 + ncomp) + ["%d"])
    return path


def compute_reynolds(u_w, D, nu, H):
    """Re = u_w D^2 / (4 nu H) (PAPER §4.2)."""
    if D == 0.0:
        return 0.0
    if not (u_w > 0 and D > 0 and nu > 0 and H > 0):
        raise ValueError("compute_reynolds: u_w, D, nu, H must be positive")
    return u_w * D * D / (4.0 * nu * H)


@dataclasses.dataclass
class GridSpec:
    origin: tuple
    spacing: tuple
    dims: tuple
    fields: tuple = (abi.FIELD_VELOCITY,)
    kinds: tuple = (abi.FLUID,)


@dataclasses.dataclass
class OutputPlan:
    """OutputPlan (config.hpp:53-59): intervals in steps (0 = never)."""
    out_dir: str
    snapshot_interval: int = 0
    trajectory_interval: int = 0
    grid_interval: int = 0
    grid: GridSpec = None
    prefix: str = "sph"
    event_log: bool = False  # transition event log CSV: step,particle,direction,body_from,body_to
    occupancy: bool = False  # cell-occupancy histogram CSV at every snapshot point


def _wants(plan, step, traj):
    snap = bool(plan.snapshot_interval) and step % plan.snapshot_interval == 0
    tr = traj is not None and bool(plan.trajectory_interval) and step % plan.trajectory_interval == 0
    return snap, tr, (SNAPSHOT_FIELDS if snap else ("kind",)) if (snap or tr) else None


def write_occupancy(fh, step, hist, max_count):
    """SPEC:218 diagnostic dump: rows (step, particles per cell, cells); the last bin is 'or more'."""
    last = len(hist) - 1
    for k, m in enumerate(hist):
        if m:
            fh.write("%d,%s%d,%d\n" % (step, ">=" if k == last else "", k, m))
    fh.write("%d,max,%d\n" % (step, max_count))


def _write_outputs(sim, plan, step, traj, store, downloaded=None, occ=None):
    st = sim.stats()
    t = st.time
    snap, tr, fields = _wants(plan, step, traj)
    if occ is not None and snap:
        write_occupancy(occ, step, *sim.cell_occupancy())
    gr = plan.grid is not None and plan.grid_interval and step % plan.grid_interval == 0
    if snap or tr:
        if downloaded is not None:
            store, bodies = downloaded
        else:
            store, bodies = sim.download(store, fields=fields)
        if snap:
            write_snapshot(store, t, os.path.join(plan.out_dir, "%s_%08d.txt" % (plan.prefix, step)), step)
        if tr:
            traj.write(t, bodies)
    if gr:
        g = plan.grid
        for f in g.fields:
            vals, sup = sim.shepard_grid(g.origin, g.spacing, g.dims, f, g.kinds)
            write_grid(os.path.join(plan.out_dir, "%s_grid_%s_%08d.txt" % (plan.prefix, FIELD_NAMES[f], step)),
                       t, g.origin, g.spacing, g.dims, f, vals, sup)
    return store


def run(sim, nsteps, plan, log=None):
    """run(config, overrides) -> exit status + artifacts for an already uploaded and
    initialised simulation: steps it `nsteps` times, writing the plan's outputs at step 0 and every
    interval.  Between output points the steps go to the device in one sphg_step(K) call (one
    sphg_step_download(K) when the point writes a snapshot or trajectory).  Returns
    (status, message): 0 ok, 2 config violation, 3 runtime assertion (escaped / coincident
    particle, non-finite state), 4 device failure — the SPEC's exit codes."""
    os.makedirs(plan.out_dir, exist_ok=True)
    events = None
    if plan.event_log:
        sim.set_event_log(True)
        events = open(os.path.join(plan.out_dir, plan.prefix + "_transitions.csv"), "w", newline="\n")
        events.write("step,particle,direction,body_from,body_to\n")
    occ = None
    if plan.occupancy:
        occ = open(os.path.join(plan.out_dir, plan.prefix + "_occupancy.csv"), "w", newline="\n")
        occ.write("step,particles_per_cell,cells\n")
    traj = TrajectoryWriter(os.path.join(plan.out_dir, plan.prefix + "_bodies.csv")) if plan.trajectory_interval else None
    intervals = [i for i in (plan.snapshot_interval, plan.trajectory_interval,
                             plan.grid_interval if plan.grid is not None else 0) if i]
    store = ParticleStore(sim.n)
    step = 0
    try:
        store = _write_outputs(sim, plan, 0, traj, store, occ=occ)
        while step < nsteps:
            nxt = min([nsteps] + [(step // i + 1) * i for i in intervals])
            fields = _wants(plan, nxt, traj)[2]
            if fields is not None:  # snapshot step: the download overlaps the last step's forces
                got = sim.step_download(nxt - step, store=store, fields=fields)
            else:
                sim.step(nxt - step)
                got = None
            step = nxt
            store = _write_outputs(sim, plan, step, traj, store, got, occ=occ)
            if events is not None:
                _write_events(events, sim.transition_events())
            if log:
                log("step %d t=%s" % (step, _g(sim.stats().time)))
    except SPHError as e:
        if events is not None:
            _write_events(events, sim.transition_events())
        return e.code, str(e)
    finally:
        if events is not None:
            events.close()
        if occ is not None:
            occ.close()
    return 0, "ok"


def _write_events(fh, ev):
    names = {1: "melt", 2: "solidify"}
    for e in ev:
        fh.write("%d,%d,%s,%d,%d\n" % (e["step"], e["gid"], names[int(e["direction"])], e["body_from"], e["body_to"]))


def scaling_report(lines, path):
    """`run scaling_box --workers 1..8` -> CSV of (workers, wall time/step, efficiency %) in the
    paper's format (PAPER §4.6) from bench.py JSON lines (dicts with n_gpus, ms_per_step,
    scaling).  Efficiency is relative to the 1-GPU line: t1/tN for weak scaling, t1/(N tN) for
    strong scaling."""
    by_n = {int(d["n_gpus"]): d for d in lines}
    if 1 not in by_n:
        raise ValueError("scaling_report needs the 1-GPU line")
    t1 = by_n[1]["ms_per_step"]
    with open(path, "w", newline="\n") as fh:
        fh.write("workers,wall_time_per_step_s,efficiency_percent\n")
        for n in sorted(by_n):
            d = by_n[n]
            tn = d["ms_per_step"]
            eff = t1 / tn if d.get("scaling", "weak") == "weak" else t1 / (n * tn)
            fh.write("%d,%r,%r\n" % (n, tn / 1000.0, round(100.0 * eff, 12)))
    return path
