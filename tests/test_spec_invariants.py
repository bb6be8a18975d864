"""The reference's physical known-answer examples and invariants that pin the wall extrapolation, the
fluid-rigid coupling, conduction and the integrator (SPEC.md lines cited per test), run on the CPU
oracle (no GPU) and, as device twins under -m gpu, on the sm_100a path through the C ABI.

These are analytic oracles, not oracle-vs-device comparisons: a sign or formula error shared by the
oracle and the device (e.g. the sign of the rho (g - a_w).(r_w - r_f) correction, DESIGN.md [P6])
fails here.
"""
import numpy as np
import pytest

from paper_2103_07925_b200 import abi, scenarios
from paper_2103_07925_b200.sim import SPHError
from paper_2103_07925_b200.store import ParticleStore, empty_bodies


@pytest.fixture(params=["oracle", pytest.param("device", marks=pytest.mark.gpu)])
def make(request):
    if request.param == "oracle":
        from oracle.oracle import Oracle
        return Oracle
    from paper_2103_07925_b200 import Simulation
    return lambda p: Simulation(p, device=0)


def loaded(make, sc, store=None, bodies=None):
    e = make(sc.params)
    e.upload(sc.store if store is None else store, sc.bodies if bodies is None else bodies)
    return e


G = 9.81


# ------------------------------------------------------------- wall extrapolation
def test_still_fluid_zero_gravity_wall_state(make):  # wall pressure = 0, interaction velocity = 0
    sc = scenarios.hydrostatic_tank(g=0.0, hydrostatic=False)
    e = loaded(make, sc)
    e.extrapolate_wall_quantities()
    s, _ = e.download()
    wl = s.kind == abi.BOUNDARY
    assert np.all(s.wall_pressure[wl] == 0.0)
    assert np.all(s.wall_velocity[wl] == 0.0)


def test_hydrostatic_wall_pressure(make):  # wall at depth H -> p_w ~ rho0 g H within 5%
    sc = scenarios.hydrostatic_tank(nz=20)
    H = sc.info["H"]
    e = loaded(make, sc)
    e.extrapolate_wall_quantities()
    s, _ = e.download()
    dx = sc.params.dx
    bottom = (s.kind == abi.BOUNDARY) & (s.pos[:, 2] < 0.0)
    first = bottom & (s.pos[:, 2] > -dx)
    # the first wall layer sits dx/2 below the fluid: rho0 g H within 5% (SPEC's bar) ...
    assert np.all(np.abs(s.wall_pressure[first] / (1000.0 * G * H) - 1.0) < 0.05)
    # ... and every supported layer follows the analytic rho0 g (H - z_w) to 0.5 %.  The opposite sign
    # of the correction, rho (g - a_w).(r_f - r_w), would put the first layer ~4 dx shallower (-17 %).
    sup = bottom & (s.wall_pressure != 0.0)
    assert sup.sum() >= 2 * first.sum()
    want = 1000.0 * G * (H - s.pos[sup, 2])
    assert np.all(np.abs(s.wall_pressure[sup] / want - 1.0) < 5e-3)
    assert np.all(s.wall_velocity[bottom] == 0.0)


def test_hydrostatic_column_settles_linear(make):  # after settling, p linear in depth within 5%
    sc = scenarios.hydrostatic_tank(nz=20, nu=1e-2, hydrostatic=False)  # starts at rho0 everywhere
    e = loaded(make, sc)
    e.initialize()
    e.step(4000)
    s, _ = e.download()
    fl = s.kind == abi.FLUID
    depth = sc.info["H"] - s.pos[fl, 2]
    A = np.vstack([depth, np.ones_like(depth)]).T
    (slope, icpt), *_ = np.linalg.lstsq(A, s.pressure[fl], rcond=None)
    assert abs(slope / (1000.0 * G) - 1.0) < 0.05
    resid = np.abs(A @ [slope, icpt] - s.pressure[fl]).max()
    assert resid < 0.05 * 1000.0 * G * sc.info["H"]


# ----------------------------------------------------------------------- coupling
def test_coupling_zero_pressure_field(make):  # fluid at rest, zero pressure field -> f_ri = 0
    sc = scenarios.hydrostatic_tank(nxy=16, nz=16, g=0.0, hydrostatic=False, sphere_radius=3.0)
    e = loaded(make, sc)
    e.extrapolate_wall_quantities()
    e.momentum_rhs()
    s, _ = e.download()
    assert np.all(s.force[s.kind == abi.RIGID] == 0.0)


def _pair_store(fluid_pos, rigid_pos, dx=1e-3):
    p = scenarios._params(dx, 1e-5, (0.0, 0.0, 0.0), (0.02, 0.02, 0.02), (0, 0, 0),
                          [scenarios.material(1000.0, nu=1e-3, c=10.0, pb=1e5), scenarios.material(1200.0, c=0.0)])
    nf, nr = len(fluid_pos), len(rigid_pos)
    s = ParticleStore(nf + nr)
    s.pos[:nf] = fluid_pos
    s.pos[nf:] = rigid_pos
    s.kind[nf:] = abi.RIGID
    s.material[nf:] = 1
    s.mass[:nf] = 1000.0 * dx ** 3
    s.mass[nf:] = 1200.0 * dx ** 3
    s.density[:] = 1000.0
    rng = np.random.default_rng(5)
    s.vel[:nf] = rng.uniform(-0.01, 0.01, (nf, 3))
    s.vel_adv[:nf] = s.vel[:nf] + rng.uniform(-1e-3, 1e-3, (nf, 3))
    b = empty_bodies(1)
    b["material"] = 1
    scenarios.body_quantities(s, b, p)
    rig = s.kind == abi.RIGID
    s.vel[rig] = 0.0
    s.vel_adv[rig] = 0.0
    return p, s, b


def test_coupling_single_pair_action_reaction(make):  # any pair -> m_i a_ir + f_ri = 0 exactly
    p, s, b = _pair_store([[0.010, 0.010, 0.010]], [[0.0115, 0.0102, 0.0097]])
    e = make(p)
    e.upload(s, b)
    e.density_summation()
    e.extrapolate_wall_quantities()
    e.momentum_rhs()
    g, _ = e.download()
    f_i = g.mass[0] * g.acc[0]  # no body force: a_i = a_ir
    f_r = g.force[1]
    assert np.linalg.norm(f_r) > 0.0
    assert np.all(np.abs(f_i + f_r) <= 4e-16 * np.abs(f_r).max())


def test_coupling_momentum_balance_cluster(make):  # SPEC:286 summed: sum_i m_i a_i + sum_r f_r = 0
    rng = np.random.default_rng(9)
    fl = rng.uniform(0.006, 0.014, (60, 3))
    rg = 0.010 + 1e-3 * np.array([[a, b_, c] for a in (-1, 0, 1) for b_ in (-1, 0, 1) for c in (-1, 0, 1)], float)
    keep = np.min(np.linalg.norm(fl[:, None, :] - rg[None, :, :], axis=2), axis=1) > 0.7e-3
    p, s, b = _pair_store(fl[keep], rg)
    e = make(p)
    e.upload(s, b)
    e.density_summation()
    e.extrapolate_wall_quantities()
    e.momentum_rhs()
    g, _ = e.download()
    fl = g.kind == abi.FLUID
    mf = g.mass[fl][:, None] * g.acc[fl]
    tot = mf.sum(axis=0) + g.force[g.kind == abi.RIGID].sum(axis=0)
    assert np.all(np.abs(tot) <= 1e-13 * np.abs(mf).sum(axis=0))


def test_archimedes_buoyancy(make):  # submerged body -> net upward coupling force ~ rho0 g V within 10%
    for R in (3.0, 4.0):
        sc = scenarios.hydrostatic_tank(nxy=20, nz=24, sphere_radius=R)
        e = loaded(make, sc)
        e.extrapolate_wall_quantities()
        e.momentum_rhs()
        e.reduce_force_torque()
        _, b = e.download()
        V = sc.info["n_rigid"] * sc.params.dx ** 3
        buoy = 1000.0 * G * V
        f = b["force"][0]
        assert abs(f[2] / buoy - 1.0) < 0.10, (R, f[2] / buoy)
        assert np.hypot(f[0], f[1]) < 1e-6 * buoy  # symmetric field: no lateral force


# ----------------------------------------------------------------------- conduction
def test_steady_conduction_rod(make):  # ends at T=0 and T=1 -> steady linear profile within 2%
    sc = scenarios.conduction_rod(nx=20)
    e = loaded(make, sc)
    e.initialize()
    for _ in range(1200):
        e.conduction_rhs()  # dt = 0.5 x the conduction limit
    s, _ = e.download()
    bar = s.kind == abi.RIGID
    x = s.pos[bar, 0]
    dx = sc.params.dx
    # analytic steady state between the held end layers (the innermost wall layers at -dx/2, L + dx/2)
    lin = (x + 0.5 * dx) / (sc.info["Lx"] + dx)
    assert np.abs(s.temperature[bar] - lin).max() < 0.02
    assert np.all(np.diff(s.temperature[bar][np.argsort(x)][::100]) >= -1e-12)


# ---------------------------------------------------------------- rigid integration
def _min_image(d, L):
    return d - L * np.round(d / L)


def test_rigidity_invariant(make):  # |r_r - r_k| constant over time to 1e-9 h
    sc = scenarios.config1(nside=16, n_spheres=3, r_range=(3.0, 3.5), seed=19, u0=0.05)
    L = sc.params.hi[0] - sc.params.lo[0]
    e = loaded(make, sc)
    e.initialize()
    rig = sc.store.kind == abi.RIGID
    grp = sc.store.group[rig]

    def radii():
        s, b = e.download()
        d = _min_image(s.pos[rig] - b["com"][grp], L)
        return np.linalg.norm(d, axis=1), b

    r0, b0 = radii()
    for _ in range(4):
        e.step(25)
        r, b = radii()
        assert np.abs(r - r0).max() <= 1e-9 * sc.params.h
    assert np.abs(b["com"] - b0["com"]).max() > 0.0  # the bodies did move


# --------------------------------------------------------------------- integrator
def _reverse(e, make, params, K):
    s, b = e.download()
    s.vel[:] *= -1.0
    s.vel_adv[:] *= -1.0
    b["vel"] *= -1.0
    b["omega"] *= -1.0
    r = make(params)
    r.upload(s, b)  # keeps a^K (acc, body acc / alpha): positions alone determine the forces here
    r.step(K)
    return r.download()


def test_reversibility_fluid_and_walls(make):  # K steps forward, K back with -u -> r^0 within 1e-8 h
    sc = scenarios.hydrostatic_tank(nxy=10, nz=12, nu=0.0, jitter=0.05, hydrostatic=False)
    p = sc.params
    p.tvf = 0  # dissipation-free: no viscosity, no transport-velocity correction
    st = sc.store
    fl = st.kind == abi.FLUID
    st.vel[fl] = np.random.default_rng(3).uniform(-0.05, 0.05, (int(fl.sum()), 3))
    st.vel_adv[:] = st.vel
    e = make(p)
    e.upload(st, sc.bodies)
    e.initialize()
    K = 50
    e.step(K)
    s2, _ = _reverse(e, make, p, K)
    d = s2.pos - st.pos
    d[:, :2] = _min_image(d[:, :2], p.hi[0] - p.lo[0])
    assert np.abs(d).max() <= 1e-8 * p.h


def test_reversibility_dry_bodies(make):  # SPEC:554 with bodies: a dry spring contact, no damping
    sc = scenarios.colliding_spheres(nside=20, R=3.0, gap=-0.3, u=0.05)
    p = sc.params
    p.dc = 0.0
    rig = sc.store.kind == abi.RIGID
    st = ParticleStore(int(rig.sum()))
    for f in ("pos", "vel", "vel_adv", "mass", "density", "kind", "group", "material", "body_frame_pos"):
        getattr(st, f)[:] = getattr(sc.store, f)[rig]
    e = make(p)
    e.upload(st, sc.bodies)
    e.initialize()
    K = 40
    e.step(K)
    _, bK = e.download()
    assert np.any(bK["force"] != 0.0)  # in contact
    s2, b2 = _reverse(e, make, p, K)
    L = p.hi[0] - p.lo[0]
    assert np.abs(_min_image(s2.pos - st.pos, L)).max() <= 1e-8 * p.h
    assert np.abs(b2["vel"] + sc.bodies["vel"]).max() <= 1e-9 * 0.05


# ------------------------------------------------------------ time-step assertion
def _rod_dt(factor, policy=abi.DT_REFUSE):
    sc = scenarios.conduction_rod(nx=12)
    lim = 0.1 * 1.0 * 1.0 * sc.params.dx ** 2 / 1.0  # 0.1 rho c_p h^2 / kappa
    sc.params.dt = factor * lim
    sc.params.dt_check = policy
    return sc


def test_dt_assertion_refuses_conduction_limit(make):
    sc = _rod_dt(1.01)
    e = loaded(make, sc)
    e.initialize()
    with pytest.raises(SPHError) as ei:
        e.step(3)
    assert ei.value.code == abi.ERR_RUNTIME
    msg = str(ei.value)
    assert "time-step condition violated at step 1" in msg and "conduction" in msg
    st = e.stats()
    assert st.steps == 1 and st.dt_term == 4


def test_dt_assertion_accepts_and_maximum_principle(make):  # 0.9 x the limit runs, T stays bounded
    sc = _rod_dt(0.9)
    rng = np.random.default_rng(4)
    bar = sc.store.kind == abi.RIGID
    sc.store.temperature[bar] = rng.uniform(0.0, 1.0, int(bar.sum()))
    e = loaded(make, sc)
    e.initialize()
    for _ in range(5):
        e.step(20)
        s, _ = e.download()
        assert s.temperature.min() >= 0.0 and s.temperature.max() <= 1.0  # discrete maximum principle
    st = e.stats()
    assert st.dt_violations == 0 and st.dt_term == 4
    assert abs(st.dt_limit - 0.1) < 1e-15


def test_dt_assertion_warn_policy_counts(make):  # C1's dt exceeds the contact limit
    sc = scenarios.config1(nside=12, n_spheres=1, r_range=(3.0, 3.0), seed=3)
    assert sc.params.dt_check == abi.DT_WARN
    e = loaded(make, sc)
    e.initialize()
    e.step(3)
    st = e.stats()
    assert st.dt_violations == 3 and st.dt_term == 3  # contact
    assert abs(st.dt_limit - 0.22 * np.sqrt(2000.0 * 1e-9 / 1e3)) < 1e-18
