"""scenario_io outputs: snapshot / trajectory / grid formats and the
run loop.  CPU tests drive the loop with the oracle engine (same interface); the GPU test runs it
on the device and checks the files against the device download and the oracle's run."""
import os

import numpy as np
import pytest

from paper_2103_07925_b200 import abi, scenarios
from paper_2103_07925_b200.output import (OutputPlan, GridSpec, SNAPSHOT_COLUMNS, compute_reynolds,
                                          read_snapshot, run, write_snapshot)
from paper_2103_07925_b200.store import ParticleStore


def test_empty_store_snapshot_is_header_only(tmp_path):  # SPEC:608 [TRIVIAL]
    p = write_snapshot(ParticleStore(0), 0.0, str(tmp_path / "e.txt"))
    lines = open(p).read().splitlines()
    assert all(ln.startswith("#") for ln in lines)
    assert lines[0] == "# sphfsi-snapshot 1" and "# particles 0" in lines
    h, cols = read_snapshot(p)
    assert h["particles"] == 0 and all(len(v) == 0 for v in cols.values())


def test_one_particle_one_row_all_columns(tmp_path):  # SPEC:609 [TRIVIAL]
    s = ParticleStore(1)
    s.pos[0] = (0.1, -2.5e-7, 3.0)
    s.vel[0] = (1.0 / 3.0, 0.0, -7.25)
    s.density[0], s.pressure[0], s.temperature[0], s.concentration[0] = 1000.0, -3.5, 293.15, 0.25
    s.kind[0], s.group[0], s.material[0] = abi.RIGID, 4, 1
    p = write_snapshot(s, 1.25e-3, str(tmp_path / "one.txt"), step=7)
    rows = [ln for ln in open(p).read().splitlines() if not ln.startswith("#")]
    assert len(rows) == 1 and len(rows[0].split()) == len(SNAPSHOT_COLUMNS)
    h, c = read_snapshot(p)
    assert h["time"] == 1.25e-3 and h["step"] == 7 and h["dim"] == 3
    assert c["x"][0] == 0.1 and c["y"][0] == -2.5e-7 and c["u_x"][0] == 1.0 / 3.0  # exact round trip
    assert c["body"][0] == 4 and c["kind"][0] == abi.RIGID and c["material"][0] == 1
    s.kind[0] = abi.FLUID
    write_snapshot(s, 0.0, p)
    assert read_snapshot(p)[1]["body"][0] == -1


def test_compute_reynolds():  # SPEC:594-600 examples
    assert compute_reynolds(0.02, 2.5e-3, 5e-6, 1e-2) == pytest.approx(0.625, rel=1e-14)
    assert compute_reynolds(0.024, 2.5e-3, 5e-6, 1e-2) == pytest.approx(0.75, rel=1e-14)
    assert compute_reynolds(0.02, 0.0, 5e-6, 1e-2) == 0.0
    with pytest.raises(ValueError):
        compute_reynolds(-1.0, 1.0, 1.0, 1.0)


def _plan(d):
    lo = (0.0, 0.0, 0.0)
    return OutputPlan(out_dir=str(d), snapshot_interval=2, trajectory_interval=1, grid_interval=3,
                      grid=GridSpec(origin=lo, spacing=(2e-3, 2e-3, 2e-3), dims=(4, 3, 2),
                                    fields=(abi.FIELD_VELOCITY, abi.FIELD_TEMPERATURE)))


def _run(engine_cls, sc, d):
    sim = engine_cls(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    status = run(sim, 5, _plan(d))
    return sim, status


def test_run_outputs_are_deterministic(tmp_path):  # same config + seed -> byte-identical
    from oracle.oracle import Oracle
    sc = scenarios.config2(nside=10, n_grid=1, r_range=(2.0, 2.0), seed=3)
    for k in (0, 1):
        sim, status = _run(Oracle, sc, tmp_path / str(k))
        assert status == (0, "ok")
    files = sorted(os.listdir(tmp_path / "0"))
    assert files == sorted(os.listdir(tmp_path / "1"))
    # snapshots at 0, 2, 4 (+ the final step 5 is not an interval point), grids at 0, 3 for 2 fields
    assert sum(f.startswith("sph_0") for f in files) == 3
    assert sum("_grid_" in f for f in files) == 4 and "sph_bodies.csv" in files
    for f in files:
        assert open(tmp_path / "0" / f, "rb").read() == open(tmp_path / "1" / f, "rb").read(), f
    traj = open(tmp_path / "0" / "sph_bodies.csv").read().splitlines()
    assert traj[0].startswith("t,body,alive,mass") and len(traj) == 1 + 6 * len(sc.bodies)
    h, c = read_snapshot(str(tmp_path / "0" / "sph_00000004.txt"))
    st, _ = sim.download()
    assert h["step"] == 4 and h["particles"] == sc.store.n


def test_run_reports_runtime_assertion(tmp_path):  # exit status 3 with the message
    from oracle.oracle import Oracle
    sc = scenarios.config1(nside=12, n_spheres=1, r_range=(3.0, 3.0))
    sc.store.vel[9] = np.nan
    sim = Oracle(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    code, msg = run(sim, 3, OutputPlan(out_dir=str(tmp_path), snapshot_interval=1))
    assert code == 3 and "non-finite state of particle" in msg


@pytest.mark.gpu
def test_run_on_device_matches_download_and_oracle(tmp_path):
    from oracle.oracle import Oracle
    from paper_2103_07925_b200 import Simulation
    sc = scenarios.config2(nside=10, n_grid=1, r_range=(2.0, 2.0), seed=3)
    sim, status = _run(lambda p: Simulation(p, device=0), sc, tmp_path / "gpu")
    assert status == (0, "ok")
    orc, status = _run(Oracle, sc, tmp_path / "orc")
    assert status == (0, "ok")
    # the last snapshot (step 4) is a faithful dump of the device state at that step ...
    h, c = read_snapshot(str(tmp_path / "gpu" / "sph_00000004.txt"))
    ho, co = read_snapshot(str(tmp_path / "orc" / "sph_00000004.txt"))
    assert h["time"] == ho["time"]
    for k in ("gid", "kind", "material", "body"):
        assert np.array_equal(c[k], co[k]), k
    for k in ("x", "y", "z", "u_x", "u_y", "u_z", "rho", "p", "T"):
        scale = max(np.abs(co[k]).max(), 1e-300)
        assert np.abs(c[k] - co[k]).max() <= 1e-10 * scale, k
    # ... and the body trajectories agree with the oracle's
    a = np.loadtxt(tmp_path / "gpu" / "sph_bodies.csv", delimiter=",", skiprows=1)
    b = np.loadtxt(tmp_path / "orc" / "sph_bodies.csv", delimiter=",", skiprows=1)
    assert a.shape == b.shape
    assert np.allclose(a, b, rtol=1e-10, atol=1e-14)


def test_scaling_report(tmp_path):  # (workers, wall time/step, efficiency %)
    from paper_2103_07925_b200.output import scaling_report
    lines = [{"n_gpus": 1, "ms_per_step": 10.0, "scaling": "strong"},
             {"n_gpus": 2, "ms_per_step": 6.25, "scaling": "strong"},
             {"n_gpus": 4, "ms_per_step": 2.5, "scaling": "strong"}]
    p = scaling_report(lines, str(tmp_path / "s.csv"))
    rows = open(p).read().splitlines()
    assert rows[0] == "workers,wall_time_per_step_s,efficiency_percent"
    assert rows[1] == "1,0.01,100.0" and rows[2] == "2,0.00625,80.0" and rows[3] == "4,0.0025,100.0"
    weak = [{"n_gpus": 1, "ms_per_step": 10.0, "scaling": "weak"}, {"n_gpus": 8, "ms_per_step": 12.5, "scaling": "weak"}]
    assert open(scaling_report(weak, p)).read().splitlines()[2] == "8,0.0125,80.0"


def _melt_case():
    return scenarios.config2(nside=12, n_grid=2, r_range=(2.0, 3.0), seed=5, melt_forcing=True)


def test_transition_event_log(tmp_path):  # "Event log (CSV): step, particle id, direction, body ids"
    from oracle.oracle import Oracle
    sc = _melt_case()
    sim = Oracle(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    sim.set_event_log(True)
    before, _ = sim.download()
    sim.step(1)
    ev = sim.transition_events()
    after, _ = sim.download()
    st = sim.stats()
    melt, solid = ev[ev["direction"] == abi.MELT], ev[ev["direction"] == abi.SOLIDIFY]
    assert len(melt) == st.transitions_melt > 0 and len(solid) == st.transitions_solidify > 0
    assert np.all(ev["step"] == 1) and np.all(np.diff(ev["gid"].astype(np.int64)) > 0)
    assert np.all(before.kind[melt["gid"]] == abi.RIGID) and np.all(after.kind[melt["gid"]] == abi.FLUID)
    assert np.array_equal(melt["body_from"], before.group[melt["gid"]].astype(np.int32)) and np.all(melt["body_to"] == -1)
    assert np.all(after.kind[solid["gid"]] == abi.RIGID)
    assert np.array_equal(solid["body_to"], after.group[solid["gid"]].astype(np.int32)) and np.all(solid["body_from"] == -1)
    assert len(sim.transition_events()) == 0  # drained
    # through the run loop: one CSV row per event
    sim2 = Oracle(sc.params)
    sim2.upload(sc.store, sc.bodies)
    sim2.initialize()
    assert run(sim2, 3, OutputPlan(out_dir=str(tmp_path), trajectory_interval=2, event_log=True)) == (0, "ok")
    rows = open(tmp_path / "sph_transitions.csv").read().splitlines()
    st2 = sim2.stats()
    assert rows[0] == "step,particle,direction,body_from,body_to"
    assert len(rows) - 1 == st2.transitions_melt + st2.transitions_solidify
    assert rows[1].split(",")[:3] == ["1", str(int(ev["gid"][0])), "melt" if ev["direction"][0] == 1 else "solidify"]


@pytest.mark.gpu
def test_transition_event_log_device_matches_oracle():
    from oracle.oracle import Oracle
    from paper_2103_07925_b200 import Simulation
    sc = _melt_case()
    out = []
    for make in (lambda p: Simulation(p, device=0), Oracle):
        e = make(sc.params)
        e.upload(sc.store, sc.bodies)
        e.initialize()
        e.set_event_log(True)
        e.step(3)
        out.append(e.transition_events())
    assert len(out[0]) > 0 and np.array_equal(out[0], out[1])


def test_cell_occupancy_histogram_csv(tmp_path, oracle_mod):  # SPEC:218 diagnostic dump
    sc = scenarios.config1(nside=12, n_spheres=1, r_range=(2.0, 2.0), seed=3)
    sim = oracle_mod.Oracle(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    hist, mx = sim.cell_occupancy(nbins=256)
    assert hist.sum() == np.prod([int(sc.params.hi[a] / (3.1 * sc.params.dx)) for a in range(3)])
    assert (np.arange(256) * hist).sum() == sc.store.n and hist[mx] > 0 and hist[mx + 1:].sum() == 0
    plan = OutputPlan(out_dir=str(tmp_path), snapshot_interval=2, occupancy=True)
    assert run(sim, 2, plan)[0] == 0
    rows = open(tmp_path / "sph_occupancy.csv").read().splitlines()
    assert rows[0] == "step,particles_per_cell,cells"
    steps = {r.split(",")[0] for r in rows[1:]}
    assert steps == {"0", "2"}
    tot = sum(int(r.split(",")[1]) * int(r.split(",")[2]) for r in rows[1:]
              if r.startswith("2,") and r.split(",")[1] not in ("max",) and not r.split(",")[1].startswith(">="))
    assert tot == sc.store.n
