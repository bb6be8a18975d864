"""GPU (sm_100a, through the C ABI) vs the CPU oracle on identical seeded inputs.

Bars (BASELINE north_star): cells, sort order and Verlet lists bit-exact;
density / acceleration / temperature rate / body force & torque within 1e-10
(DESIGN.md §5 metric); phase flags bit-exact after step 1.
"""
import os

import numpy as np
import pytest

from paper_2103_07925_b200 import scenarios, Simulation, SPHError, abi
from tests.helpers import compare_state, run_pair, vec_err

pytestmark = pytest.mark.gpu

CASES = {
    "c1_small": lambda: scenarios.config1(nside=20, n_spheres=3, r_range=(3.0, 4.0), seed=11),
    "c1": lambda: scenarios.config1(),
    "c2_small": lambda: scenarios.config2(nside=18, n_grid=2, r_range=(2.0, 3.0), seed=5),
    "c2_melt": lambda: scenarios.config2(nside=18, n_grid=2, r_range=(2.0, 3.0), seed=5, melt_forcing=True),
    # two phases (multi-EOS / harmonic-mean viscosity / dominant-material wall state), cubes + spheres
    "c3_small": lambda: scenarios.config3(nside=20, n_bodies=4, r_range=(2.0, 3.0), seed=7),
    # concentration diffusion + Dirichlet-C fluid bath + concentration-mode dissolution at step 1
    "dissolve": lambda: scenarios.dissolving_bodies(nside=16, n_bodies=3, r_range=(2.0, 3.0), seed=13, forcing=True),
    # powder bed (periodic x, y; substrate + lid walls; gas; log-normal grains) under the moving
    # Gaussian surface heat flux [P21]: exposed grain surfaces melt at step 1
    # the paper's strong-scaling case at a small size (closed box, 8 spheres D = 2.5 on a grid, lattice
    # without jitter: many pairs exactly at r_c / r_v)
    "paper46_small": lambda: scenarios.paper_strong_scaling(nside=30, n_grid=2),
    "c4_small": lambda: scenarios.config4(nx=24, ny=24, nz=40, n_grains=12, r0_dx=6.0, T0=1698.0, seed=3),
}


@pytest.fixture(scope="module")
def Oracle():
    from oracle.oracle import Oracle as O
    return O


# below the melting point (no transitions, so graphs replay) with a fast scan: the spot moves ~1.4 dx
# per step, so a replay that kept a stale t^{n+1} for the source kernel would differ
GRAPH_CASES = {"c4_scan": lambda: scenarios.config4(nx=24, ny=24, nz=40, n_grains=12, r0_dx=6.0, T0=1500.0,
                                                    scan_speed=1e4, seed=3)}


def sim_factory(params):
    return Simulation(params, device=0)


@pytest.mark.parametrize("case", list(CASES))
def test_cells_and_nlist_bitexact(case, Oracle):
    sc = CASES[case]()
    sim, orc = run_pair(sc, sim_factory, Oracle, init=False)
    for e in (sim, orc):
        e.build_pairs()
    cg, og = sim.get_cells()
    co, oo = orc.get_cells()
    assert np.array_equal(cg, co), "cell ids differ"
    assert np.array_equal(og, oo), "(cell, gid) order differs"
    offg, nbg = sim.get_nlist()
    offo, nbo = orc.get_nlist()
    assert np.array_equal(offg, offo), "neighbour counts differ"
    assert np.array_equal(nbg, nbo), "neighbour lists differ"


@pytest.mark.parametrize("case", list(CASES))
def test_initialize_parity(case, Oracle):
    sc = CASES[case]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    compare_state(sim, orc, sc.params, what=f"{case} init")


@pytest.mark.parametrize("case", list(CASES))
def test_step1_parity(case, Oracle):
    sc = CASES[case]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    sim.step(1)
    orc.step(1)
    compare_state(sim, orc, sc.params, what=f"{case} step1")


def test_phase_flags_bitexact_step1(Oracle):
    sc = CASES["c2_melt"]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    sim.step(1)
    orc.step(1)
    g, gb = sim.download()
    o, ob = orc.download()
    assert orc.stats().transitions_melt > 0 and orc.stats().transitions_solidify > 0
    assert np.array_equal(g.kind, o.kind)
    assert np.array_equal(g.group, o.group)
    assert np.array_equal(g.material, o.material)
    assert len(gb) == len(ob)
    assert np.array_equal(gb["alive"], ob["alive"])
    assert sim.stats().transitions_melt == orc.stats().transitions_melt
    assert sim.stats().transitions_solidify == orc.stats().transitions_solidify
    # mass and particle count conserved exactly
    assert g.mass.sum() == sc.store.mass.sum()


def test_multistep_c1_small(Oracle):
    sc = CASES["c1_small"]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    sim.step(10)
    orc.step(10)
    # chaotic growth of round-off over 10 steps: 1e-7 of the pair-sum scale
    compare_state(sim, orc, sc.params, tol=1e-7, what="c1_small 10 steps")
    assert sim.stats().rebuilds == orc.stats().rebuilds


def test_multistep_transitions(Oracle):
    """Melting and solidification over several steps: flags bit-exact every step, fields within
    the multistep tolerance, rebuild count equal (transitions force a rebuild)."""
    sc = CASES["c2_melt"]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    for k in range(6):
        sim.step(1)
        orc.step(1)
        g, gb = sim.download()
        o, ob = orc.download()
        assert np.array_equal(g.kind, o.kind), f"kind differs after step {k + 1}"
        assert np.array_equal(g.group, o.group), f"group differs after step {k + 1}"
        assert np.array_equal(gb["alive"], ob["alive"])
    assert sim.stats().transitions_melt == orc.stats().transitions_melt
    assert sim.stats().transitions_solidify == orc.stats().transitions_solidify
    assert sim.stats().rebuilds == orc.stats().rebuilds
    compare_state(sim, orc, sc.params, tol=1e-7, what="c2_melt 6 steps")


def test_multistep_dissolve(Oracle):
    """Diffusion + concentration transitions over several steps: flags exact, fields at the
    multistep bar."""
    sc = CASES["dissolve"]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    for k in range(5):
        sim.step(1)
        orc.step(1)
        g, _ = sim.download()
        o, _ = orc.download()
        assert np.array_equal(g.kind, o.kind), f"kind differs after step {k + 1}"
    assert sim.stats().transitions_melt == orc.stats().transitions_melt > 0
    compare_state(sim, orc, sc.params, tol=1e-7, what="dissolve 5 steps")


def test_multistep_powder_bed(Oracle):
    """C4 at a small size: the moving surface heat flux melts exposed grain surfaces every step; the
    grains lose particles (bodies shrink / split), flags bit-exact every step, fields at the
    multistep bar, and the source rate itself matches (dT/dt of the exposed particles)."""
    sc = CASES["c4_small"]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    for k in range(5):
        sim.step(1)
        orc.step(1)
        g, gb = sim.download()
        o, ob = orc.download()
        assert np.array_equal(g.kind, o.kind), f"kind differs after step {k + 1}"
        assert np.array_equal(g.group, o.group), f"group differs after step {k + 1}"
        assert np.array_equal(gb["alive"], ob["alive"])
    assert sim.stats().transitions_melt == orc.stats().transitions_melt > 0
    assert sim.stats().rebuilds == orc.stats().rebuilds
    compare_state(sim, orc, sc.params, tol=1e-7, what="c4_small 5 steps")


def test_moving_heat_flux_parity(Oracle):
    """Fast scan (the spot moves ~1.4 dx per step) below the melting point: the source term follows
    the spot on the device exactly as in the oracle (periodic wrap of the centre included)."""
    sc = GRAPH_CASES["c4_scan"]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    for k in range(4):
        sim.step(1)
        orc.step(1)
        g, _ = sim.download()
        o, _ = orc.download()
        assert np.count_nonzero(o.dT_dt > 1e6) > 0  # exposed particles under the spot
        assert vec_err(g.dT_dt, o.dT_dt, orc.scales()["dT_dt"], tol=1e-7) <= 1.0, f"dT/dt after step {k + 1}"
    compare_state(sim, orc, sc.params, tol=1e-7, what="c4_scan 4 steps")


def test_multistep_c3_small(Oracle):
    sc = CASES["c3_small"]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    sim.step(8)
    orc.step(8)
    compare_state(sim, orc, sc.params, tol=1e-7, what="c3_small 8 steps")


def test_stage_by_stage(Oracle):
    sc = CASES["c2_small"]()
    sim, orc = run_pair(sc, sim_factory, Oracle, init=False)
    for st in (abi.STAGE_REBUILD, abi.STAGE_DENSITY, abi.STAGE_EXTRAPOLATE, abi.STAGE_FORCES, abi.STAGE_BODIES,
               abi.STAGE_KICK_DRIFT):
        sim.run_stage(st)
        orc.run_stage(st)
    compare_state(sim, orc, sc.params, what="stages")
    for st in (abi.STAGE_DENSITY, abi.STAGE_HEAT, abi.STAGE_EXTRAPOLATE, abi.STAGE_FORCES, abi.STAGE_BODIES,
               abi.STAGE_FINAL_KICK, abi.STAGE_MASS):
        sim.run_stage(st)
        orc.run_stage(st)
    compare_state(sim, orc, sc.params, what="stages2")


def test_isolated_particle_density():
    from paper_2103_07925_b200.store import ParticleStore
    sc = scenarios.config1(nside=16, n_spheres=0)
    s = ParticleStore(1)
    s.pos[0] = [0.008, 0.008, 0.008]
    s.mass[0] = 1e-6
    s.density[0] = 1000.0
    sim = Simulation(sc.params)
    sim.upload(s, None)
    sim.density_summation()
    g, _ = sim.download()
    h = sc.params.dx
    w0 = 66.0 / (120.0 * np.pi * h ** 3)
    assert abs(g.density[0] - 1e-6 * w0) <= 1e-14 * g.density[0]


def test_empty_store():
    from paper_2103_07925_b200.store import ParticleStore
    sc = scenarios.config1(nside=16, n_spheres=0)
    sim = Simulation(sc.params)
    sim.upload(ParticleStore(0), None)
    sim.initialize()
    sim.step(3)
    assert sim.stats().steps == 3


def test_coincident_particles_fail():  # fatal, names the particle
    sc = scenarios.config1(nside=16, n_spheres=0)
    sc.store.pos[5] = sc.store.pos[6]
    sim = Simulation(sc.params)
    sim.upload(sc.store, sc.bodies)
    with pytest.raises(SPHError) as e:
        sim.initialize()
    assert e.value.code == 3 and "coincident particles at particle 5 " in str(e.value)


def test_escaped_particle_fail():  # fatal, names the particle and the step
    sc = scenarios.config2(nside=12, n_grid=1, r_range=(2.0, 2.0))
    sc.store.pos[7, 2] = sc.params.hi[2] + 1e-3
    sim = Simulation(sc.params)
    sim.upload(sc.store, sc.bodies)
    with pytest.raises(SPHError) as e:
        sim.initialize()
    assert e.value.code == 3 and "escaped particle 7 " in str(e.value)


def test_non_finite_state_fail(Oracle):  # SPEC:625 runtime assertion on a blown-up state
    """A NaN velocity spreads through the initial forces to the particle's neighbours; both engines
    stop at step 1 naming the same (smallest) gid of the non-finite set."""
    sc = scenarios.config1(nside=16, n_spheres=1, r_range=(3.0, 3.0))
    sc.store.vel[9] = np.nan
    msgs = []
    for eng in (Simulation(sc.params), Oracle(sc.params)):
        eng.upload(sc.store, sc.bodies)
        eng.initialize()
        with pytest.raises(SPHError) as e:
            eng.step(1)
        assert e.value.code == 3 and "non-finite state of particle" in str(e.value), str(e.value)
        msgs.append(str(e.value).split("non-finite")[1])
    assert msgs[0] == msgs[1]


def test_nlist_capacity_growth(Oracle):
    sc = scenarios.config1(nside=16, n_spheres=1, r_range=(3.0, 3.0))
    sc.params.nlist_capacity = 8
    sim, orc = run_pair(sc, sim_factory, Oracle, init=False)
    sim.build_pairs()
    orc.build_pairs()
    assert sim.stats().nlist_capacity >= sim.stats().max_neighbours > 8
    assert np.array_equal(sim.get_nlist()[1], orc.get_nlist()[1])


def test_warm_upload_roundtrip(Oracle):
    sc = CASES["c1_small"]()
    sim = Simulation(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    sim.step(2)
    s, b = sim.download()
    sim.upload(s, b)  # warm: same size, list kept
    s2, b2 = sim.download()
    for f in ("pos", "vel", "acc", "density", "temperature", "mass"):
        assert np.array_equal(getattr(s, f), getattr(s2, f)), f
    sim.step(1)
    orc = Oracle(sc.params)
    orc.upload(sc.store, sc.bodies)
    orc.initialize()
    orc.step(3)
    compare_state(sim, orc, sc.params, tol=1e-7, what="warm upload")


def test_cpp_dropin_on_device():
    """The C++ adapter over sphfsi::ParticleStore<3> (tests/cpp/test_dropin.cpp) runs the GPU path."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_dropin")
    assert os.path.exists(exe), "build() compiles tests/cpp/test_dropin"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("cell_build", ["0", "1"])
def test_nlist_both_builders_bitexact(cell_build, Oracle, monkeypatch):
    """Per-particle and cell-cooperative Verlet builders give the pinned list."""
    monkeypatch.setenv("SPHG_CELL_BUILD", cell_build)
    for sc in (CASES["c1_small"](), CASES["c2_small"]()):
        sim, orc = run_pair(sc, sim_factory, Oracle, init=False)
        sim.build_pairs()
        orc.build_pairs()
        assert np.array_equal(sim.get_nlist()[1], orc.get_nlist()[1])


def test_nlist_dense_cells_fallback(Oracle):
    """Cells denser than the cooperative builder takes (cell edge override 8.5 dx, ~600 particles
    per cell) fall back to the per-particle builder; the list is unchanged."""
    sc = scenarios.config1(nside=32, n_spheres=2, r_range=(3.0, 3.0), seed=5)
    sc.params.cell_edge_override = 8.5e-3
    sim, orc = run_pair(sc, sim_factory, Oracle, init=False)
    sim.build_pairs()
    orc.build_pairs()
    assert np.array_equal(sim.get_cells()[0], orc.get_cells()[0])
    assert np.array_equal(sim.get_nlist()[1], orc.get_nlist()[1])


def test_upload_state_warm_update(Oracle):
    """sphg_upload_state (kinematic host update between steps) == a full upload of the same state."""
    sc = CASES["c1_small"]()
    a = Simulation(sc.params)
    a.upload(sc.store, sc.bodies)
    a.initialize()
    a.step(2)
    s, b = a.download()
    s.vel[:] *= 0.5  # host-side intervention on the velocities
    a.upload_state(s.pos, s.vel)
    a.step(1)
    ref = Simulation(sc.params)
    ref.upload(s, b)
    ref.step(1)  # cold path: full upload of the same state (a^n carried in the store)
    ga, _ = a.download()
    gr, _ = ref.download()
    from tests.helpers import vec_err
    assert vec_err(ga.pos, gr.pos, 0.016, 1e-14) <= 1
    assert vec_err(ga.vel, gr.vel, 1e-3, 1e-9) <= 1


def test_upload_state_matches_oracle(Oracle):
    """sphg_upload_state on both engines (kinematic update, one particle pushed past half the skin
    so both drop their Verlet lists), then two steps: fields within the multistep bar."""
    sc = CASES["c1_small"]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    sim.step(2)
    orc.step(2)
    s, _ = orc.download()
    s.vel[:] *= 0.5
    s.pos[0] += 0.2 * sc.params.h
    for e in (sim, orc):
        e.upload_state(s.pos, s.vel)
        e.step(2)
    compare_state(sim, orc, sc.params, tol=1e-8, what="upload_state + 2 steps")
    assert sim.stats().rebuilds == orc.stats().rebuilds


@pytest.mark.parametrize("name", ["c1_small", "c2_melt", "c4_small"])
@pytest.mark.parametrize("pinned", [False, True])
def test_step_download_equals_step_then_download(name, pinned):
    """sphg_step_download (early fields copied during the last step's forces when transitions are
    off; c2_melt / c4_small take the plain path) returns exactly what sphg_step + sphg_download do."""
    import torch
    from paper_2103_07925_b200.store import ParticleStore, SCALAR_FIELDS, TAG_FIELDS, VEC_FIELDS
    sc = CASES[name]()
    a, b = sim_factory(sc.params), sim_factory(sc.params)
    for e in (a, b):
        e.upload(sc.store, sc.bodies)
        e.initialize()
    fields = VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS)
    out = ParticleStore(sc.store.n)
    if pinned:
        for f in fields:
            arr = getattr(out, f)
            t = torch.empty(arr.shape, dtype=getattr(torch, str(arr.dtype)), pin_memory=True)
            setattr(out, f, t.numpy())
    for k in (1, 3):
        ga, ba = a.step_download(k, store=out, fields=fields)
        b.step(k)
        gb, bb = b.download()
        for f in fields:
            assert np.array_equal(getattr(ga, f), getattr(gb, f)), f"{f} after {k} steps"
        assert np.array_equal(ba, bb)


def test_download_into_pinned_and_pageable(Oracle):
    """The gid-order device pack lands identically in pinned and pageable host arrays."""
    import torch
    sc = CASES["c2_small"]()
    sim = sim_factory(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    sim.step(1)
    a, _ = sim.download()
    b = a.copy()
    for f in ("pos", "vel", "density", "pressure", "temperature"):
        arr = getattr(b, f)
        pinned = torch.empty(arr.shape, dtype=torch.float64, pin_memory=True).numpy()
        setattr(b, f, pinned)
    sim.download(b, fields=("pos", "vel", "density", "pressure", "temperature"))
    for f in ("pos", "vel", "density", "pressure", "temperature"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("case", ["c1_small", "c2_small", "dissolve"])
def test_shepard_grid_parity(case, Oracle):
    """shepard_interpolate on a grid, device vs oracle, every field, after two steps
    (particles off their rebuild positions); points outside the domain have no support on both."""
    sc = CASES[case]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    sim.step(2)
    orc.step(2)
    p = sc.params
    lo = np.array([p.lo[a] for a in range(3)])
    hi = np.array([p.hi[a] for a in range(3)])
    dims = (9, 7, 8)
    sp = (hi - lo) / (np.array(dims) - 1) * 1.15  # the last points fall outside the domain
    org = lo - 0.05 * (hi - lo)
    kinds = (abi.FLUID,) if case != "c2_small" else (abi.FLUID, abi.RIGID)
    fields = [abi.FIELD_VELOCITY, abi.FIELD_TEMPERATURE, abi.FIELD_PRESSURE, abi.FIELD_DENSITY]
    if p.diffusion:
        fields.append(abi.FIELD_CONCENTRATION)
    for f in fields:
        g, gs = sim.shepard_grid(org, sp, dims, f, kinds)
        o, os_ = orc.shepard_grid(org, sp, dims, f, kinds)
        assert np.array_equal(gs, os_), f"support differs (field {f})"
        scale = max(float(np.nanmax(np.abs(o))), 1e-30)
        assert np.allclose(g[gs], o[os_], rtol=1e-12, atol=1e-12 * scale), f"field {f}"
        assert np.all(np.isnan(g[~gs]))


@pytest.mark.parametrize("omega", [0.0, 3000.0])
def test_moving_walls_parity(omega, Oracle):
    """Prescribed wall motion (WallGroup, config.hpp:35-51): drift with u_w(t^{n+1/2}), wall state
    u_w, a_w (central difference) at t^{n+1}; device vs oracle after 1 and 6 steps."""
    sc = scenarios.couette_channel(nside=16, nz=12)
    sim, orc = sim_factory(sc.params), Oracle(sc.params)
    for e in (sim, orc):
        e.upload(sc.store, sc.bodies)
        e.set_wall_motion(2, scenarios.wall_velocity(0.01, omega=omega))
        e.initialize()
    compare_state(sim, orc, sc.params, what=f"couette omega={omega} init")
    sim.step(1)
    orc.step(1)
    compare_state(sim, orc, sc.params, what=f"couette omega={omega} step1")
    sim.step(5)
    orc.step(5)
    compare_state(sim, orc, sc.params, tol=1e-7, what=f"couette omega={omega} 6 steps")
    g, _ = sim.download()
    o, _ = orc.download()
    w = g.kind == abi.BOUNDARY
    assert np.array_equal(g.pos[w], o.pos[w]) and np.array_equal(g.vel[w], o.vel[w])


def _momentum(sim):
    s, b = sim.download()
    fl = s.kind == abi.FLUID
    al = b["alive"] == 1
    p = (s.mass[fl, None] * s.vel[fl]).sum(0) + (b["mass"][al, None] * b["vel"][al]).sum(0)
    scale = (s.mass[fl, None] * np.abs(s.vel[fl])).sum(0) + (b["mass"][al, None] * np.abs(b["vel"][al])).sum(0)
    return p, scale, s.mass.sum()


def test_full_size_c5_momentum_conservation():
    """BASELINE's full C5 size (400^3 = 64M particles, 20,000 spheres) on the device: total linear
    momentum of fluid + bodies is conserved by the antisymmetric pair forces and contact to
    round-off (the oracle holds it to 1e-16 at small sizes; FMA-ordered pair sums to ~1e-13),
    total mass exactly, across Verlet rebuilds."""
    sc = scenarios.config5()
    sim = sim_factory(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    p0, s0, m0 = _momentum(sim)
    r0 = sim.stats().rebuilds
    sim.step(30)
    p1, s1, m1 = _momentum(sim)
    assert sim.stats().rebuilds > r0  # the run crossed at least one Verlet rebuild
    assert np.all(np.abs(p1 - p0) <= 1e-12 * np.maximum(s0, s1)), (p1 - p0) / s0
    assert m1 == m0


def test_minimum_image_entry_mode(Oracle):
    """Stores with >= 2^26 particles keep plain indices in the rows and take the minimum image in
    the pair kernels (kImgMin); forced here at a small size: lists and step-1 fields unchanged."""
    import subprocess, sys, os
    code = (
        "import numpy as np\n"
        "from paper_2103_07925_b200 import scenarios, Simulation\n"
        "from oracle.oracle import Oracle\n"
        "from tests.helpers import compare_state, run_pair\n"
        "sc = scenarios.config1(nside=20, n_spheres=3, r_range=(3.0, 4.0), seed=11)\n"
        "sim, orc = run_pair(sc, lambda p: Simulation(p, device=0), Oracle, init=False)\n"
        "sim.build_pairs(); orc.build_pairs()\n"
        "assert np.array_equal(sim.get_nlist()[1], orc.get_nlist()[1])\n"
        "sim.initialize(); orc.initialize(); sim.step(1); orc.step(1)\n"
        "compare_state(sim, orc, sc.params, what='imgmin step1')\n"
        "s, b = orc.download(); sim.upload(s, b); o2 = Oracle(sc.params); o2.upload(s, b)\n"
        "sim.step(1); o2.step(1)\n"
        "compare_state(sim, o2, sc.params, what='imgmin step2')\n"
        "print('ok')\n")
    env = dict(os.environ, SPHG_IMG_MIN="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_cell_occupancy_matches_oracle(Oracle):  # SPEC:218 histogram from the device cell ranges
    sc = CASES["c2_small"]()
    sim, orc = Simulation(sc.params), Oracle(sc.params)
    for e in (sim, orc):
        e.upload(sc.store, sc.bodies)
        e.initialize()
    hg, mg = sim.cell_occupancy(nbins=48)
    ho, mo = orc.cell_occupancy(nbins=48)
    assert np.array_equal(hg, ho) and mg == mo and hg.sum() > 0


def test_count_pairs(Oracle):
    """sphg_count_pairs (the bench's flop model input) against the oracle's lists and positions."""
    sc = CASES["c2_small"]()
    sim, orc = run_pair(sc, sim_factory, Oracle, init=False)
    sim.build_pairs()
    orc.build_pairs()
    cand, inter, inter_f, inter_o = sim.count_pairs()
    off, nbr = orc.get_nlist()
    o, _ = orc.download()
    p = sc.params
    L = np.array([p.hi[a] - p.lo[a] for a in range(3)])
    i = np.repeat(np.arange(len(off) - 1), np.diff(off))
    d = o.pos[i] - o.pos[nbr]
    for a in range(3):
        if p.periodic[a]:
            d[:, a] = np.where(d[:, a] > 0.5 * L[a], d[:, a] - L[a], np.where(d[:, a] < -0.5 * L[a], d[:, a] + L[a], d[:, a]))
    r2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
    rc = 3.0 * (p.h if p.h > 0 else p.dx)
    hit = r2 <= rc * rc
    assert cand == len(nbr)
    assert inter == int(hit.sum())
    assert inter_f == int(hit[o.kind[i] == abi.FLUID].sum())
    assert inter_o == inter - inter_f


def test_contact_parity(Oracle):
    """Two bodies inside each other's contact range, approaching: spring-dashpot contact
     on the device vs the oracle, initial forces and 5 steps (the contact candidates
    are ordered first in each rigid row by k_contact_order)."""
    sc = scenarios.colliding_spheres()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    _, ob = orc.download()
    p0 = scenarios.colliding_spheres().params
    p0.kc = p0.dc = 0.0
    nocontact = Oracle(p0)
    nocontact.upload(sc.store, sc.bodies)
    nocontact.initialize()
    _, nb = nocontact.download()
    assert np.all(np.abs(ob["force"][:, 0] - nb["force"][:, 0]) > 1e-3 * np.abs(nb["force"][:, 0]))  # contact acts
    compare_state(sim, orc, sc.params, what="contact init")
    sim.step(5)
    orc.step(5)
    compare_state(sim, orc, sc.params, tol=1e-7, what="contact 5 steps")


@pytest.mark.parametrize("case", ["c1_small", "c2_small"])
def test_without_transport_velocity(case, Oracle):
    """transport_velocity = false (config.hpp:90): the kTvf = false kernel variants (no A-tensor,
    no background pressure, drift with u)."""
    sc = CASES[case]()
    sc.params.tvf = 0
    sim, orc = run_pair(sc, sim_factory, Oracle)
    sim.step(1)
    orc.step(1)
    compare_state(sim, orc, sc.params, what=f"{case} tvf=0 step1")
    step_from_identical_inputs(sim, orc, Oracle, sc.params, f"{case} tvf=0 step2")


def test_heat_with_distinct_conductivities(Oracle):
    """Materials with different conductivities: the harmonic-mean kappa~ path of k_heat (the
    single-kappa shortcut is off), with melting at step 1."""
    sc = CASES["c2_melt"]()
    p = sc.params
    p.mat[1].kappa = 35.0   # solid conducts better than the liquids
    p.mat[3].kappa = 5.0    # walls
    sim, orc = run_pair(sc, sim_factory, Oracle)
    sim.step(1)
    orc.step(1)
    compare_state(sim, orc, p, what="multi-kappa heat step1")
    step_from_identical_inputs(sim, orc, Oracle, p, "multi-kappa heat step2")


def test_compute_dt_uses_device_u_max(Oracle):
    """compute_dt on the device: the CFL term from the kick's u_max (max |u^{n+1/2}|
    of the fluid) agrees with the oracle's; the other terms are the host formula."""
    from paper_2103_07925_b200.sim import dt_limits
    sc = CASES["c1_small"]()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    sim.step(3)
    orc.step(3)
    assert abs(sim.stats().u_max - orc.stats().u_max) <= 1e-9 * orc.stats().u_max
    lim = sim.compute_dt()
    m_r = sc.params.mat[1].rho0 * sc.params.dx ** 3
    want = dt_limits(sc.params, orc.stats().u_max, m_r)
    assert np.allclose(lim, want, rtol=1e-9, atol=0.0, equal_nan=True)


def test_fused_kick_is_bit_identical():
    """Inside one sphg_step(K) call the particle final kick is folded into the next kick-drift;
    K steps in one call and K single-step calls give bit-identical states."""
    sc = CASES["c1_small"]()
    a, b = sim_factory(sc.params), sim_factory(sc.params)
    for e in (a, b):
        e.upload(sc.store, sc.bodies)
        e.initialize()
    a.step(6)
    for _ in range(6):
        b.step(1)
    ga, ba = a.download()
    gb, bb = b.download()
    for f in ("pos", "vel", "vel_adv", "acc", "acc_bg", "density", "pressure", "force"):
        assert np.array_equal(getattr(ga, f), getattr(gb, f)), f
    assert np.array_equal(ba, bb)


def test_fused_heat_is_bit_identical():
    """sphg_step folds fluid conduction into the forces pass; with stage timing on it runs the
    separate heat kernel.  Both give bit-identical temperatures and rates (C2 with melting)."""
    sc = CASES["c2_melt"]()
    a, b = sim_factory(sc.params), sim_factory(sc.params)
    for e in (a, b):
        e.upload(sc.store, sc.bodies)
        e.initialize()
    b.set_timing(True)
    a.step(3)
    b.step(3)
    ga, _ = a.download()
    gb, _ = b.download()
    for f in ("temperature", "dT_dt", "pos", "vel", "acc", "density"):
        assert np.array_equal(getattr(ga, f), getattr(gb, f)), f
    assert np.array_equal(ga.kind, gb.kind)


def test_fused_diffusion_is_bit_identical():
    """Without the heat equation, sphg_step folds the fluid concentration sums into the forces pass
    (same terms, same order as k_diffusion); with stage timing on they run in k_diffusion.  Same
    concentrations, rates and transition flags bit for bit (dissolution with concentration-mode
    transitions)."""
    sc = CASES["dissolve"]()
    a, b = sim_factory(sc.params), sim_factory(sc.params)
    for e in (a, b):
        e.upload(sc.store, sc.bodies)
        e.initialize()
    b.set_timing(True)
    a.step(4)
    b.step(4)
    ga, _ = a.download()
    gb, _ = b.download()
    for f in ("concentration", "dC_dt", "pos", "vel", "acc", "density", "kind", "group"):
        assert np.array_equal(getattr(ga, f), getattr(gb, f)), f


@pytest.mark.parametrize("name,steps", [("c1_small", 40), ("c2_melt", 6), ("c3_small", 12), ("dissolve", 6),
                                        ("c4_scan", 6)])
def test_graph_replay_is_bit_identical(monkeypatch, name, steps):
    """sphg_step captures its two launch chains as CUDA graphs and replays them; a context created
    with SPHG_GRAPHS=0 launches eagerly.  Same state bit for bit, across rebuilds (new buffer sets)
    and transitions (new kind lists), and the graphs are actually replayed."""
    sc = {**CASES, **GRAPH_CASES}[name]()
    a = sim_factory(sc.params)
    monkeypatch.setenv("SPHG_GRAPHS", "0")
    b = sim_factory(sc.params)
    monkeypatch.delenv("SPHG_GRAPHS")
    for e in (a, b):
        e.upload(sc.store, sc.bodies)
        e.initialize()
    for k in (1, steps - 1):
        a.step(k)
        b.step(k)
    sa, sb = a.stats(), b.stats()
    assert sb.graph_captures == 0 and sb.graph_replays == 0
    assert sa.graph_captures > 0 and sa.graph_replays > 0
    assert sa.rebuilds == sb.rebuilds and sa.kernel_launches == sb.kernel_launches
    ga, ba = a.download()
    gb, bb = b.download()
    from paper_2103_07925_b200.store import SCALAR_FIELDS, TAG_FIELDS, VEC_FIELDS
    for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS):
        assert np.array_equal(getattr(ga, f), getattr(gb, f)), f
    assert np.array_equal(ba, bb)


def test_periodic_face_crossing_between_rebuilds(Oracle):
    """Particles that cross a periodic face between Verlet rebuilds: the image codes stored in the rows
    (fixed at build time) are patched for them and for the entries referencing them, so every step
    matches the oracle (minimum image throughout) and no rebuild is triggered by the crossing."""
    from tests.test_decomposition import crossing_case
    sc = crossing_case()
    sim, orc = run_pair(sc, sim_factory, Oracle)
    for k in range(4):
        sim.step(1)
        orc.step(1)
        compare_state(sim, orc, sc.params, tol=1e-10 if k == 0 else 1e-8, what=f"crossing step {k + 1}")
    assert sim.stats().rebuilds == orc.stats().rebuilds == 1
    g, _ = sim.download()
    L = sc.params.hi[0] - sc.params.lo[0]
    moved = np.abs(g.pos - sc.store.pos) > 0.5 * L
    assert moved.sum() >= 30  # most planted particles crossed their face (pressure turns a few back)
    sim.step(6)  # graph-replayed steps carry the patch as well
    orc.step(6)
    compare_state(sim, orc, sc.params, tol=1e-7, what="crossing 10 steps")


def _fast(sc, u):
    """Fluid velocities raised to |u_i| ~ u so Verlet rebuilds happen within a few steps."""
    fl = sc.store.kind == abi.FLUID
    rng = np.random.default_rng(17)
    sc.store.vel[fl] = rng.uniform(-u, u, (int(fl.sum()), 3))
    sc.store.vel_adv[fl] = sc.store.vel[fl]
    return sc


SPEC_CASES = {"c2_melt_fast": lambda: _fast(CASES["c2_melt"](), 2.0),
              "dissolve_fast": lambda: _fast(CASES["dissolve"](), 1.0)}


@pytest.mark.parametrize("name", list(SPEC_CASES))
def test_speculation_is_bit_identical(monkeypatch, name):
    """sphg_step queues the force chain before it reads the kick chain's flags (speculation); when the
    step needs a Verlet rebuild the queued chain voids itself and the host restores the state it
    changed (buffer swaps, deferred final kick) before rebuilding.  A context created with
    SPHG_SPECULATE=0 never speculates.  Same state bit for bit across rebuilds and phase transitions
    (ADVICE r1)."""
    sc = SPEC_CASES[name]()
    a = sim_factory(sc.params)
    monkeypatch.setenv("SPHG_SPECULATE", "0")
    b = sim_factory(sc.params)
    monkeypatch.delenv("SPHG_SPECULATE")
    for e in (a, b):
        e.upload(sc.store, sc.bodies)
        e.initialize()
    for k in (1, 5, 9):
        a.step(k)
        b.step(k)
    sa, sb = a.stats(), b.stats()
    assert sa.rebuilds == sb.rebuilds and sa.rebuilds >= 3, (sa.rebuilds, sb.rebuilds)
    assert sa.transitions_melt + sa.transitions_solidify > 0
    assert (sa.transitions_melt, sa.transitions_solidify) == (sb.transitions_melt, sb.transitions_solidify)
    ga, ba = a.download()
    gb, bb = b.download()
    from paper_2103_07925_b200.store import SCALAR_FIELDS, TAG_FIELDS, VEC_FIELDS
    for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS):
        assert np.array_equal(getattr(ga, f), getattr(gb, f)), f
    assert np.array_equal(ba, bb)


# BASELINE sizes that the oracle still steps in seconds: C2 (343k, heat + forced melting), C3 (2.41M,
# two phases, 200 bodies), the paper's own strong-scaling case (3.80M, 216 spheres, exact lattice) and
# C5 at one GPU's weak-scaling share (200^3 = 8M particles, 2500 spheres R ~ U[3, 6] dx: the headline
# sphere density, three radix passes, 4-lane rigid groups)
FULL = {
    "c2_full_melt": lambda: scenarios.config2(melt_forcing=True),
    "c3_full": lambda: scenarios.config3(),
    "paper46_full": lambda: scenarios.paper_strong_scaling(),
    "c5_200": lambda: scenarios.config5(nside=200, n_spheres=2500),
}


def step_from_identical_inputs(sim, orc, Oracle, params, what, steps=1, compare_lists=True):
    """One step of both engines from the SAME state: the oracle's state at t^n (store + body table,
    bit for bit) is uploaded into the device (a warm upload: device order and Verlet rows kept) and
    into a fresh oracle context, both step, and every field is compared at the 1e-10 bar.  (Stepping
    each engine from its own previous step would compare two trajectories that already differ by the
    1e-10 of the step before.)"""
    o_state, o_bodies = orc.download()
    orc.close()  # at the headline size two oracle contexts would not fit the host's RAM
    sim.upload(o_state, o_bodies)
    orc2 = Oracle(params)
    orc2.upload(o_state, o_bodies)
    del o_state
    sim.step(steps)
    orc2.step(steps)
    orc2.last_errors = compare_state(sim, orc2, params, what=what)
    return orc2


def _host_ram_gb():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
    except (ValueError, OSError):
        return 0.0


def test_headline_c5_parity(Oracle):
    """The headline workload itself (BASELINE configs[4], C5: 400^3 = 64M particles, 20,000 spheres, one
    GPU): cell ids and (cell, gid) order bit-exact, every particle's Verlet candidate count equal (the
    lists themselves are compared entry by entry at 8M, c5_200), initialize() and one step from identical
    inputs within 1e-10.  Needs ~150 GB of host RAM for the oracle (the B200 box has 196 GB)."""
    if _host_ram_gb() < 150:
        pytest.skip(f"host RAM {_host_ram_gb():.0f} GB < 150 GB for the 64M oracle")
    sc = scenarios.config5()
    sim, orc = run_pair(sc, sim_factory, Oracle, init=False)
    sc.store = None
    for e in (sim, orc):
        e.build_pairs()
    cg, og = sim.get_cells()
    co, oo = orc.get_cells()
    assert np.array_equal(cg, co) and np.array_equal(og, oo), "cells / order differ"
    del cg, og, co, oo
    assert np.array_equal(sim.get_nlist(offsets_only=True), orc.get_nlist(offsets_only=True)), "counts differ"
    for e in (sim, orc):
        e.initialize()
    e0 = compare_state(sim, orc, sc.params, what="c5 64M init")
    print("c5 64M init: max error / tolerance per field", e0)
    o2 = step_from_identical_inputs(sim, orc, Oracle, sc.params, "c5 64M step1")
    print("c5 64M step 1 (identical inputs): max error / tolerance per field", o2.last_errors)


@pytest.mark.parametrize("case", list(FULL))
def test_full_size_parity(case, Oracle):
    """Cells, (cell, gid) order and Verlet lists bit-exact, then initialize() and one full step from
    identical inputs (flags bit-exact, fields within 1e-10) at the BASELINE size, device vs oracle."""
    sc = FULL[case]()
    sim, orc = run_pair(sc, sim_factory, Oracle, init=False)
    for e in (sim, orc):
        e.build_pairs()
    cg, og = sim.get_cells()
    co, oo = orc.get_cells()
    assert np.array_equal(cg, co) and np.array_equal(og, oo), "cells / order differ"
    del cg, og, co, oo
    offg, nbg = sim.get_nlist()
    offo, nbo = orc.get_nlist()
    assert np.array_equal(offg, offo) and np.array_equal(nbg, nbo), "neighbour lists differ"
    del nbg, nbo, offg, offo
    for e in (sim, orc):
        e.initialize()
    compare_state(sim, orc, sc.params, what=f"{case} init")
    step_from_identical_inputs(sim, orc, Oracle, sc.params, f"{case} step1")


@pytest.mark.parametrize("name,steps", [("c1", 30), ("c1_small", 12), ("c3_small", 8), ("c2_melt", 6), ("c4_small", 5)])
def test_sm_local_grids_bit_identical(monkeypatch, name, steps):
    """The 4-lane pair passes of long lists run as SM-local persistent grids (per-SM tile queues over the
    brick-ordered lists; density, fluid forces with and without the fused conduction, extrapolation, rigid
    forces and conduction); a context created with SPHG_SM_LOCAL=0 uses flat grids.
    Every particle is summed by the same lanes in the same order, so the states are identical bit for bit,
    across rebuilds, transitions and CUDA-graph replay.  Forced here for short lists (SPHG_SM_LOCAL_MIN=0)
    and 4 lanes per particle."""
    sc = CASES[name]()
    if name == "c1":
        _fast(sc, 0.5)
    monkeypatch.setenv("SPHG_GROUP_DENSITY", "4")
    monkeypatch.setenv("SPHG_GROUP_FORCES", "4")
    monkeypatch.setenv("SPHG_SM_LOCAL_MIN", "0")
    monkeypatch.setenv("SPHG_FILL_GROUPS", "0")  # 4 lanes per particle for the short wall / rigid lists too
    monkeypatch.setenv("SPHG_SM_LOCAL", "31")
    a = sim_factory(sc.params)
    monkeypatch.setenv("SPHG_SM_LOCAL", "0")
    b = sim_factory(sc.params)
    for e in (a, b):
        e.upload(sc.store, sc.bodies)
        e.initialize()
    for k in (1, steps - 1):
        a.step(k)
        b.step(k)
    sa, sb = a.stats(), b.stats()
    assert sa.rebuilds == sb.rebuilds
    if name == "c1":
        assert sa.rebuilds >= 2
    ga, ba = a.download()
    gb, bb = b.download()
    from paper_2103_07925_b200.store import SCALAR_FIELDS, TAG_FIELDS, VEC_FIELDS
    for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS):
        assert np.array_equal(getattr(ga, f), getattr(gb, f)), f
    assert np.array_equal(ba, bb)
