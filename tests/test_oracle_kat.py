"""Pins the CPU oracle (test infrastructure) against the reference itself:
the known-answer examples SPEC.md attaches to each hot-path operation, run through
the oracle, which is compiled from the reference's own headers.

SPEC line numbers are cited per test.  No GPU needed.
"""
import math

import numpy as np
import pytest
from scipy import integrate

from paper_2103_07925_b200 import abi, scenarios
from paper_2103_07925_b200.store import ParticleStore, empty_bodies


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


def lib(O):
    return O.load()


# ------------------------------------------------------------------ kernel
def test_kernel_compact_support_and_peak(O):
    L = lib(O)
    h = 1e-3
    assert L.orc_kernel_w(h, 3 * h) == 0.0
    assert L.orc_kernel_w(h, 3.5 * h) == 0.0
    assert L.orc_kernel_w(h, 0.0) == 66.0 * L.orc_kernel_sigma(h)
    assert L.orc_kernel_dw(h, 0.0) == 0.0
    assert L.orc_kernel_dw(h, 3 * h) == 0.0


def test_kernel_normalisation_3d(O):  # SPEC:113, 639 (quadrature oracle, 1e-6)
    L = lib(O)
    h = 1.0
    val, _ = integrate.quad(lambda r: 4 * math.pi * r * r * L.orc_kernel_w(h, r), 0, 3 * h,
                            points=[1.0, 2.0], epsabs=1e-13, epsrel=1e-13)
    assert abs(val - 1.0) < 1e-6


def test_kernel_derivative_matches_fd(O):  # SPEC:122 (finite differences, 1e-8)
    L = lib(O)
    h = 1e-3
    for q in (0.3, 0.9, 1.4, 1.99, 2.5, 2.9):
        r = q * h
        e = 1e-6 * h
        fd = (L.orc_kernel_w(h, r + e) - L.orc_kernel_w(h, r - e)) / (2 * e)
        dw = L.orc_kernel_dw(h, r)
        assert dw <= 0.0
        assert abs(fd - dw) <= 1e-8 * abs(dw)


# --------------------------------------------------------------------- EOS
def test_eos_known_answers(O):
    L = lib(O)
    assert L.orc_eos_pressure(1000.0, 1000.0, 0.25) == 0.0
    assert abs(1000.0 * 0.25 ** 2 - 62.5) == 0.0
    assert abs(L.orc_eos_pressure(1010.0, 1000.0, 0.25) - 0.625) < 1e-12


# ----------------------------------------------------------------- lattice
@pytest.mark.parametrize("lo,hi,dx", [((0, 0, 0), (0.032, 0.032, 0.032), 1e-3),
                                      ((-0.003, -0.003, -0.003), (0.021, 0.021, 0.021), 1e-3),
                                      ((0.0, 0.0, 0.0), (1.0, 0.5, 0.25), 0.05)])
def test_generator_matches_seed_lattice(O, lo, hi, dx):  # lattice.hpp:38-82
    ref = O.seed_lattice_box(lo, hi, dx)
    mine = scenarios.lattice_box(lo, hi, dx)
    assert ref.shape == mine.shape
    assert np.array_equal(ref, mine)  # bit-identical


def test_seed_lattice_mass_convention():  # SPEC:63 (unit square analogue in 3D), lattice.hpp:75
    sc = scenarios.config1(nside=8, n_spheres=0)
    assert np.all(sc.store.mass == 1000.0 * (1e-3) ** 3)
    assert sc.store.n == 512


def test_ball_membership_matches_ball_region(O):  # lattice.hpp:28-36, SPEC:65 (brute-force lattice count)
    c = np.array([0.0105, 0.0102, 0.0099])
    R = 4e-3
    dx = 1e-3
    ref = O.seed_lattice_ball(c, 2 * R, dx)
    pts = scenarios.lattice_box(c - R, c + R, dx)  # the ball's own bounding-box lattice
    d = pts - c
    inside = ((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]) <= R * R  # norm_sq (vec.hpp:80)
    assert np.array_equal(ref, pts[inside])


# -------------------------------------------------------------- density
def _single_material_params(n=12, dx=1e-3, periodic=True, c=10.0, pb=0.0, g=(0, 0, 0)):
    p = abi.Params()
    L = n * dx
    p.dx = dx
    p.h = dx
    p.dt = 1e-5
    for a in range(3):
        p.lo[a], p.hi[a], p.periodic[a] = 0.0, L, int(periodic)
    p.n_mat = 2
    p.mat[0] = scenarios.material(1000.0, nu=1e-6, c=c, pb=pb, g=g)
    p.mat[1] = scenarios.material(2000.0, c=0.0)
    p.tvf = 1 if pb > 0 else 0
    p.nranks = 1
    return p


def test_isolated_particle_density(O):
    p = _single_material_params(periodic=False)
    s = ParticleStore(1)
    s.pos[0] = [0.006, 0.006, 0.006]
    s.mass[0] = 1e-6
    o = O.Oracle(p)
    o.upload(s, None)
    o.density_summation()
    g, _ = o.download()
    assert g.density[0] == 1e-6 * lib(O).orc_kernel_w(1e-3, 0.0)


def test_lattice_interior_density(O):  # SPEC:134, 250 (direct lattice summation, within 1%)
    p = _single_material_params(n=12)
    pts = scenarios.lattice_box((0, 0, 0), (0.012,) * 3, 1e-3)
    s = ParticleStore(len(pts))
    s.pos[:] = pts
    s.mass[:] = 1e-6
    o = O.Oracle(p)
    o.upload(s, None)
    o.density_summation()
    g, _ = o.download()
    assert np.all(np.abs(g.density / 1000.0 - 1.0) < 0.01)


# ------------------------------------------------------------- neighbours
def test_pairs_match_all_pairs_oracle(O):  # SPEC:195, 208 (O(N^2) oracle, periodic)
    rng = np.random.default_rng(1)
    p = _single_material_params(n=10)
    L = 0.010
    pos = rng.uniform(0, L, (500, 3))
    s = ParticleStore(500)
    s.pos[:] = pos
    s.mass[:] = 1e-6
    o = O.Oracle(p)
    o.upload(s, None)
    o.build_pairs()
    off, nbr = o.get_nlist()
    rv = 3.1e-3
    d = pos[:, None, :] - pos[None, :, :]
    d = np.where(d > L / 2, d - L, np.where(d < -L / 2, d + L, d))
    r2 = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
    for i in range(500):
        want = np.nonzero((r2[i] <= rv * rv) & (np.arange(500) != i))[0]
        assert np.array_equal(nbr[off[i]:off[i + 1]], want)


def test_pair_inclusive_at_cutoff(O):  # distance exactly r_v included, r_v + eps excluded
    p = _single_material_params(n=12, periodic=False)
    s = ParticleStore(3)
    rv = 3 * 1e-3 + 0.1 * 1e-3
    s.pos[0] = [0.005, 0.005, 0.005]
    s.pos[1] = [0.005 + rv, 0.005, 0.005]
    s.pos[2] = [0.005 - np.nextafter(rv, 1.0), 0.005, 0.005]
    s.mass[:] = 1e-6
    o = O.Oracle(p)
    o.upload(s, None)
    o.build_pairs()
    off, nbr = o.get_nlist()
    d1 = (s.pos[0, 0] - s.pos[1, 0])
    included = d1 * d1 <= rv * rv
    assert (1 in nbr[off[0]:off[1]]) == included
    assert 2 not in nbr[off[0]:off[1]]


# ---------------------------------------------------------------- momentum
def test_pairwise_antisymmetry(O):  # SPEC:267, 291, 636(d)
    p = _single_material_params(periodic=False)
    p.mat[0].nu = 0.0
    s = ParticleStore(2)
    s.pos[0] = [0.005, 0.005, 0.005]
    s.pos[1] = [0.0065, 0.0052, 0.0049]
    s.mass[:] = [1e-6, 1.3e-6]
    o = O.Oracle(p)
    o.upload(s, None)
    o.density_summation()
    o.momentum_rhs()
    g, _ = o.download()
    f0, f1 = g.mass[0] * g.acc[0], g.mass[1] * g.acc[1]
    assert np.all(np.abs(f0 + f1) <= 1e-15 * np.abs(f0).max())
    # along e_ij
    e = (s.pos[0] - s.pos[1]) / np.linalg.norm(s.pos[0] - s.pos[1])
    assert np.linalg.norm(np.cross(f0, e)) <= 1e-12 * np.linalg.norm(f0)


# ---------------------------------------------------------------- contact
def _two_rigid(O, r, kc=1.0, dc=0.0, v=(0, 0, 0), dx=1.0):
    p = abi.Params()
    p.dx = dx
    p.h = dx
    p.dt = 1e-3
    for a in range(3):
        p.lo[a], p.hi[a] = 0.0, 20.0
    p.n_mat = 2
    p.mat[0] = scenarios.material(1.0, c=1.0)
    p.mat[1] = scenarios.material(1.0)
    p.kc, p.dc = kc, dc
    p.nranks = 1
    s = ParticleStore(2)
    s.kind[:] = abi.RIGID
    s.material[:] = 1
    s.group[:] = [0, 1]
    s.mass[:] = 1.0
    s.density[:] = 1.0
    s.pos[0] = [10.0, 10.0, 10.0]
    s.pos[1] = [10.0 + r, 10.0, 10.0]
    s.vel[0] = v
    b = empty_bodies(2)
    b["material"] = 1
    b["mass"] = 1.0
    b["com"][0] = s.pos[0]
    b["com"][1] = s.pos[1]
    o = O.Oracle(p)
    o.upload(s, b)
    o.momentum_rhs()
    g, _ = o.download()
    return g.force


def test_contact_known_answers(O):
    f = _two_rigid(O, 0.5)  # k_c=1, d_c=0, dx=1, r=0.5 -> |f| = 0.5, repulsive
    assert abs(np.linalg.norm(f[0]) - 0.5) < 1e-15
    assert f[0][0] < 0 and f[1][0] > 0
    assert np.allclose(f[0], -f[1], atol=0)
    assert np.all(_two_rigid(O, 1.0) == 0.0)  # r >= dx -> 0
    # separating fast with large damping: tension cut-off -> 0
    assert np.all(_two_rigid(O, 0.5, dc=100.0, v=(-1.0, 0, 0)) == 0.0)


# ------------------------------------------------------------ rigid bodies
def test_particle_inertia_kat(O):
    dx = (math.pi / 0.75) ** (1.0 / 3.0)
    assert abs(lib(O).orc_particle_inertia(1.0, dx) - 0.4) < 1e-15


def _body_store(O, pos, masses=None, forces=None, dx=1.0):
    n = len(pos)
    p = abi.Params()
    p.dx, p.h, p.dt = dx, dx, 1e-3
    for a in range(3):
        p.lo[a], p.hi[a] = -50.0, 50.0
    p.n_mat = 2
    p.mat[0] = scenarios.material(1.0, c=1.0)
    p.mat[1] = scenarios.material(1.0)
    p.nranks = 1
    s = ParticleStore(n)
    s.kind[:] = abi.RIGID
    s.material[:] = 1
    s.group[:] = 0
    s.mass[:] = 1.0 if masses is None else masses
    s.density[:] = 1.0
    s.pos[:] = pos
    if forces is not None:
        s.force[:] = forces
    b = empty_bodies(1)
    b["material"] = 1
    o = O.Oracle(p)
    o.upload(s, b)
    return o


def test_single_particle_body(O):
    o = _body_store(O, [[1.0, 2.0, 3.0]], masses=[2.0])
    o.reduce_mass_quantities()
    _, b = o.download()
    Ir = lib(O).orc_particle_inertia(2.0, 1.0)
    assert b["mass"][0] == 2.0
    assert np.array_equal(b["com"][0], [1.0, 2.0, 3.0])
    assert np.allclose(b["inertia"][0], [Ir, Ir, Ir, 0, 0, 0], rtol=1e-15, atol=0)


def test_two_particle_parallel_axis(O):
    d = 0.7
    o = _body_store(O, [[-d, 0, 0], [d, 0, 0]])
    o.reduce_mass_quantities()
    _, b = o.download()
    Ir = lib(O).orc_particle_inertia(1.0, 1.0)
    assert abs(b["inertia"][0][2] - 2 * (Ir + d * d)) < 1e-14


def test_force_torque_known_answers(O):
    pos = np.array([[1.0, 0, 0], [-1.0, 0, 0], [0, 1.0, 0], [0, -1.0, 0]])
    o = _body_store(O, pos, forces=np.tile([0.0, 0.0, 2.0], (4, 1)))
    o.reduce_mass_quantities()
    o.reduce_force_torque()
    _, b = o.download()
    assert np.allclose(b["force"][0], [0, 0, 8.0]) and np.allclose(b["torque"][0], 0.0, atol=1e-15)
    F = np.zeros((4, 3))
    F[0] = [0.0, 3.0, 0.0]
    o = _body_store(O, pos, forces=F)
    o.reduce_mass_quantities()
    o.reduce_force_torque()
    _, b = o.download()
    assert np.allclose(b["torque"][0], np.cross([1.0, 0, 0], [0.0, 3.0, 0.0]))


def test_kahan(O):
    x = np.array([1e16, 1.0, -1e16])
    assert lib(O).orc_kahan_sum(x.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)), 3) == 1.0


# --------------------------------------------------------------- quaternion
def test_orientation_step_known_answers(O):
    import ctypes as C
    L = lib(O)
    dp = C.POINTER(C.c_double)
    q = np.array([1.0, 0, 0, 0])
    w = np.array([0, 0, math.pi / 2])
    out = np.zeros(4)
    L.orc_orientation_step(q.ctypes.data_as(dp), w.ctypes.data_as(dp), 1.0, out.ctypes.data_as(dp))
    assert np.allclose(out, [math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)], atol=1e-15)
    v = np.array([1.0, 0, 0])
    r = np.zeros(3)
    L.orc_rotate(out.ctypes.data_as(dp), v.ctypes.data_as(dp), r.ctypes.data_as(dp))
    assert np.allclose(r, [0, 1, 0], atol=1e-15)
    q2 = np.array([0.5, 0.5, -0.5, 0.5])
    L.orc_orientation_step(q2.ctypes.data_as(dp), np.zeros(3).ctypes.data_as(dp), 0.3, out.ctypes.data_as(dp))
    assert np.array_equal(out, q2)  # omega = 0 -> q unchanged exactly


# -------------------------------------------------------------- integrator
def test_free_particle_constant_force(O):
    b = (0.0, -9.81, 0.0)
    p = _single_material_params(periodic=False, g=b)
    p.dt = 1e-3
    p.dt_check = abi.DT_OFF  # an isolated particle: the KAT is the integrator, not the CFL bound
    s = ParticleStore(1)
    s.pos[0] = [0.006, 0.006, 0.006]
    s.vel[0] = [0.1, 0.0, 0.0]
    s.vel_adv[0] = s.vel[0]
    s.mass[0] = 1e-6
    s.density[0] = 1000.0
    o = O.Oracle(p)
    o.upload(s, None)
    o.initialize()
    o.step(1)
    g, _ = o.download()
    dt = p.dt
    assert np.allclose(g.vel[0], s.vel[0] + dt * np.array(b), rtol=0, atol=1e-15)
    assert np.allclose(g.pos[0], s.pos[0] + dt * s.vel[0] + 0.5 * dt * dt * np.array(b), rtol=0, atol=1e-15)


def test_dt_limits_known_answers():  # SPEC:540-542 (product host function, no device)
    from paper_2103_07925_b200.sim import dt_limits
    p = abi.Params()
    p.dx, p.h = 2e-4, 2e-4
    p.n_mat = 1
    p.mat[0] = scenarios.material(1000.0, nu=5e-6, c=0.25)
    p.kc = 1e3
    lim = dt_limits(p, 0.01, 1e-3)
    assert abs(lim[0] - 0.25 * 2e-4 / 0.26) < 1e-18
    assert abs(lim[1] - 1.0e-3) < 1e-15
    assert math.isinf(lim[2])
    assert abs(lim[3] - 0.22 * math.sqrt(1e-6)) < 1e-15
    assert math.isinf(lim[4])


# ------------------------------------------------------------------ thermal
def test_uniform_temperature_no_rate(O):
    sc = scenarios.config2(nside=10, n_grid=1, r_range=(2.0, 2.0), T0=300.0, T_hot=300.0)
    o = O.Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    o.conduction_rhs()
    g, _ = o.download()
    assert np.all(g.dT_dt == 0.0)


def test_dirichlet_schedule(O):
    sc = scenarios.config2(nside=10, n_grid=1, r_range=(2.0, 2.0))
    sch = sc.params.dirichlet_T[0]
    sch.n = 2
    sch.t_end[0], sch.value[0] = 0.5, 100.0
    sch.t_end[1], sch.value[1] = 1e30, 0.0
    bottom = sc.store.dirichlet_T == 0
    for t0, want in ((0.4, 100.0), (0.6, 0.0)):
        sc.params.t0 = t0 - sc.params.dt  # the schedule is applied at t^{n+1} [P9]
        o = O.Oracle(sc.params)
        o.upload(sc.store, sc.bodies)
        o.initialize()
        o.conduction_rhs()
        g, _ = o.download()
        assert np.all(g.temperature[bottom] == want)


# --------------------------------------------------------------- diffusion
def _dissolve(**kw):
    kw.setdefault("nside", 12)
    kw.setdefault("n_bodies", 1)
    kw.setdefault("r_range", (3.0, 3.0))
    return scenarios.dissolving_bodies(**kw)


def test_uniform_concentration_no_rate(O):
    sc = _dissolve()
    sc.store.concentration[:] = 1.0
    o = O.Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    o.diffusion_rhs()
    g, _ = o.download()
    assert np.all(g.dC_dt == 0.0)
    assert np.all(g.concentration == 1.0)


def test_two_particle_diffusion_conserves_mC(O):  # sum m_a C_a conserved to round-off
    sc = _dissolve()
    p = sc.params
    p.transitions = 0
    st = ParticleStore(2)
    c0 = np.array([0.5 * (p.lo[a] + p.hi[a]) for a in range(3)])
    st.pos[0] = c0
    st.pos[1] = c0 + [1.5 * p.dx, 0.0, 0.0]
    st.kind[:] = abi.FLUID
    st.material[0], st.material[1] = 0, 2  # different diffusivities (harmonic mean)
    st.mass[:] = 1000.0 * p.dx ** 3
    st.density[:] = 1000.0
    st.concentration[:] = (0.0, 1.0)
    o = O.Oracle(p)
    o.upload(st, empty_bodies(0))
    o.initialize()
    o.diffusion_rhs()
    g, _ = o.download()
    assert g.dC_dt[0] > 0.0 > g.dC_dt[1]
    mC = g.mass * g.dC_dt
    assert abs(mC.sum()) <= 1e-14 * np.abs(mC).max()


def test_bath_maximum_principle(O):  # body C non-decreasing and bounded by the bath's 1
    sc = _dissolve()
    o = O.Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    rig = sc.store.kind == abi.RIGID
    prev = sc.store.concentration[rig].copy()
    for _ in range(5):
        o.step(2)
        g, _ = o.download()
        cur = g.concentration[rig]
        assert np.all(cur >= prev) and np.all(cur <= 1.0)
        prev = cur
    juice = sc.store.dirichlet_C == 0
    assert np.all(g.concentration[juice] == 1.0)  # [P18] Dirichlet fluid keeps C^


def _bolus_at(O, C):
    sc = _dissolve()
    rig = sc.store.kind == abi.RIGID
    sc.store.concentration[rig] = C
    o = O.Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    o.apply_transitions()
    return sc, o


def test_concentration_transition_strict_inequality(O):  # SPEC:461-463 in concentration mode
    sc, o = _bolus_at(O, 0.8)
    assert o.stats().transitions_melt == 0
    sc, o = _bolus_at(O, 0.81)  # C_r = 0.81, C_t = 0.8 -> melt
    g, b = o.download()
    rig = sc.store.kind == abi.RIGID
    assert o.stats().transitions_melt == int(rig.sum())
    assert np.all(g.kind[rig] == abi.FLUID) and np.all(g.material[rig] == 2)  # dissolved into chyme
    assert b["alive"][0] == 0


# -------------------------------------------------------------- transitions
def _one_body_melt(O, T, u=(0.01, 0.0, 0.0)):
    sc = scenarios.config2(nside=10, n_grid=1, r_range=(2.0, 2.0), T_hot=300.0)
    s = sc.store
    rig = s.kind == abi.RIGID
    s.temperature[:] = 300.0
    s.temperature[rig] = T
    sc.bodies["vel"][0] = u
    s.vel[rig] = u
    o = O.Oracle(sc.params)
    o.upload(s, sc.bodies)
    o.initialize()
    o.apply_transitions()
    return sc, o


def test_transition_strict_inequality(O):
    sc, o = _one_body_melt(O, 1700.0)
    assert o.stats().transitions_melt == 0
    sc, o = _one_body_melt(O, np.nextafter(1700.0, 2000.0))
    g, b = o.download()
    assert o.stats().transitions_melt == int((sc.store.kind == abi.RIGID).sum())
    assert b["alive"][0] == 0  # body deleted
    melted = sc.store.kind == abi.RIGID
    assert np.all(g.kind[melted] == abi.FLUID)
    assert np.allclose(g.vel[melted], [0.01, 0.0, 0.0], atol=1e-15)  # u = u_k
    assert g.mass.sum() == sc.store.mass.sum()


def test_solidify_spawns_single_particle_body(O):
    sc = scenarios.config2(nside=10, n_grid=1, r_range=(2.0, 2.0), T_hot=300.0)
    s = sc.store
    s.temperature[:] = 300.0
    fl = np.nonzero(s.kind == abi.FLUID)[0]
    # a melt-liquid particle far from the sphere, below T_t
    far = fl[np.argmax(np.linalg.norm(s.pos[fl] - sc.bodies["com"][0], axis=1))]
    s.material[far] = 2
    s.temperature[far] = 1600.0
    o = O.Oracle(sc.params)
    o.upload(s, sc.bodies)
    o.initialize()
    o.apply_transitions()
    g, b = o.download()
    assert len(b) == 2 and b["alive"][1] == 1
    assert g.kind[far] == abi.RIGID and g.group[far] == 1
    assert b["mass"][1] == s.mass[far]
    assert np.array_equal(b["com"][1], g.pos[far])


def test_melt_solidify_roundtrip_mass(O):
    sc = scenarios.config2(nside=10, n_grid=1, r_range=(2.5, 2.5), T_hot=300.0)
    s = sc.store
    s.temperature[:] = 300.0
    rig = s.kind == abi.RIGID
    s.temperature[rig] = 1750.0
    o = O.Oracle(sc.params)
    o.upload(s, sc.bodies)
    o.initialize()
    o.apply_transitions()  # melt all
    g, b = o.download()
    assert not np.any(g.kind == abi.RIGID)
    g.temperature[rig] = 1600.0  # cool -> solidify
    o2 = O.Oracle(sc.params)
    o2.upload(g, b)
    o2.initialize()
    o2.apply_transitions()
    g2, b2 = o2.download()
    assert np.array_equal(g2.kind == abi.RIGID, rig)
    alive = b2["alive"] == 1
    assert abs(b2["mass"][alive].sum() - sc.bodies["mass"][0]) <= 1e-12 * sc.bodies["mass"][0]
    assert g2.mass.sum() == s.mass.sum()


def test_post_transition_velocity_sign(O):  # w=(0,0,1), COM shift (1,0,0), u'=0 -> correction (0,1,0)
    w = np.array([0.0, 0.0, 1.0])
    shift = np.array([1.0, 0.0, 0.0])
    assert np.array_equal(np.cross(w, shift), [0.0, 1.0, 0.0])


# -------------------------------------------------------------- conservation
def test_conservation_periodic_c1(O):  # SPEC:290, 636(a)(b)
    sc = scenarios.config1(nside=16, n_spheres=2, r_range=(3.0, 3.0), seed=3)
    o = O.Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()

    def momentum():
        g, b = o.download()
        fl = g.kind == abi.FLUID
        P = (g.mass[fl, None] * g.vel[fl]).sum(0) + (b["mass"][:, None] * b["vel"]).sum(0)
        S = np.abs(g.mass[fl, None] * g.vel[fl]).sum(0).sum()
        return P, S, g.mass.sum()

    P0, S0, M0 = momentum()
    o.step(10)
    P1, S1, M1 = momentum()
    assert M1 == M0
    assert np.all(np.abs(P1 - P0) <= 1e-10 * S0)


# ----------------------------------------------------------- Shepard grid
def _grid_over(sc, n=6):
    p = sc.params
    lo = np.array([p.lo[a] for a in range(3)])
    hi = np.array([p.hi[a] for a in range(3)])
    sp = (hi - lo) / (n + 1)
    return lo + sp, sp, (n, n, n)


def test_shepard_constant_field(O):  # constant field -> the constant (to summation round-off:
    # "exactly" holds in exact arithmetic; the two ~100-term fp64 sums round independently)
    sc = scenarios.config1(nside=12, n_spheres=1, r_range=(2.0, 2.0), seed=3)
    sc.store.temperature[:] = 7.0
    o = O.Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    org, sp, dims = _grid_over(sc)
    v, sup = o.shepard_grid(org, sp, dims, abi.FIELD_TEMPERATURE, kinds=(abi.FLUID, abi.RIGID))
    assert sup.all()
    assert np.max(np.abs(v - 7.0)) <= 7.0 * 1e-13


def test_shepard_single_neighbour_and_no_support(O):
    sc = scenarios.config1(nside=12, n_spheres=1, r_range=(2.0, 2.0), seed=3)
    p = sc.params
    st = ParticleStore(1)
    c0 = np.array([0.5 * (p.lo[a] + p.hi[a]) for a in range(3)])
    st.pos[0] = c0
    st.kind[0] = abi.FLUID
    st.mass[0] = 1000.0 * p.dx ** 3
    st.density[0] = 1000.0
    st.temperature[0] = 321.5
    o = O.Oracle(p)
    o.upload(st, empty_bodies(0))
    v, sup = o.shepard_grid(c0 + [0.7 * p.dx, 0.0, 0.0], [5 * p.dx] * 3, (2, 1, 1), abi.FIELD_TEMPERATURE)
    assert sup[0, 0, 0] and abs(v[0, 0, 0, 0] - 321.5) <= 321.5 * 2e-16
    assert not sup[1, 0, 0] and np.isnan(v[1, 0, 0, 0])  # 5 dx away: no particle within r_c


def test_shepard_linear_field_interior(O):  # linear field, interior point, within 1 %
    sc = scenarios.config1(nside=16, n_spheres=1, r_range=(2.0, 2.0), seed=3)
    s = sc.store
    s.kind[:] = abi.FLUID
    s.pos[:] = scenarios.lattice_box((0.0,) * 3, (16 * sc.params.dx,) * 3, sc.params.dx)  # no jitter
    s.temperature[:] = 300.0 + 1e4 * s.pos[:, 0]
    o = O.Oracle(sc.params)
    o.upload(s, empty_bodies(0))
    o.initialize()
    x = np.array([7.3, 8.1, 6.6]) * sc.params.dx
    v, sup = o.shepard_grid(x, [sc.params.dx] * 3, (1, 1, 1), abi.FIELD_TEMPERATURE)
    exact = 300.0 + 1e4 * x[0]
    assert abs(v[0, 0, 0, 0] - exact) <= 0.01 * abs(exact)


# ------------------------------------------------------------- moving walls
def test_moving_wall_pulls_fluid(O):  # u_wall = (0.01, 0), fluid at rest -> pulled along
    sc = scenarios.couette_channel(nside=12, nz=10, jitter=0.0)
    o = O.Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.set_wall_motion(2, scenarios.wall_velocity(0.01))
    o.initialize()
    g, _ = o.download()
    fl = g.kind == abi.FLUID
    H = 10 * sc.params.dx
    near_top = fl & (g.pos[:, 2] > H - 2 * sc.params.dx)
    near_bottom = fl & (g.pos[:, 2] < 2 * sc.params.dx)
    assert np.all(g.acc[near_top, 0] > 0.0)
    assert np.max(np.abs(g.acc[near_bottom, 0])) < 1e-8  # the fixed wall exerts no x force on fluid at rest
    top = g.kind == abi.BOUNDARY
    top &= g.group == 1
    wv = g.wall_velocity[top, 0]  # u~_w = 2 u_w - <u_f>_W = 0.02 with fluid support, u_w without
    assert np.all((wv == 0.02) | (wv == 0.01)) and np.any(wv == 0.02)


def test_moving_wall_drift_and_central_difference(O):  # config.hpp:42-50
    sc = scenarios.couette_channel(nside=12, nz=10, jitter=0.0)
    o = O.Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    om = 2000.0
    o.set_wall_motion(2, scenarios.wall_velocity(0.01, omega=om))
    o.initialize()
    o.step(3)
    g, _ = o.download()
    top = (sc.store.kind == abi.BOUNDARY) & (sc.store.group == 1)
    dt = sc.params.dt
    want = sum(dt * 0.01 * np.sin(om * (k + 0.5) * dt) for k in range(3))  # drift with u(t^{n+1/2})
    L = sc.params.hi[0] - sc.params.lo[0]
    dxs = np.mod(g.pos[top, 0] - sc.store.pos[top, 0] + 0.5 * L, L) - 0.5 * L
    assert np.allclose(dxs, want, rtol=0.0, atol=2e-17)  # a few ulps of |x| ~ 1e-2
    assert np.allclose(g.vel[top, 0], 0.01 * np.sin(om * 3 * dt), rtol=1e-14)  # u_w(t^{n+1})
    bottom = (sc.store.kind == abi.BOUNDARY) & (sc.store.group == 0)
    assert np.array_equal(g.pos[bottom], sc.store.pos[bottom])


# ---------------------------------------------------- surface heat flux [P21]
# The moving Gaussian surface flux of BASELINE C4 is an extension (the reference has no heat
# sources); these known answers pin the oracle to the formula in sphg.h.
def _flux_params(P=200.0, r0=5e-3, origin=(0.006, 0.006), vel=(0.0, 0.0), t0=0.0):
    p = _single_material_params(periodic=True)
    p.n_mat = 2
    p.mat[0] = scenarios.material(1.6, nu=1e-5, cp=520.0, kappa=0.0, c=10.0)   # gas: not in the mask
    p.mat[1] = scenarios.material(7900.0, nu=1e-6, cp=700.0, kappa=0.0, c=10.0)  # metal
    p.thermal = 1
    p.t0 = t0
    p.heat_source = 1
    p.hs_material_mask = 1 << 1
    p.hs_power, p.hs_radius = P, r0
    p.hs_origin[0], p.hs_origin[1] = origin
    p.hs_velocity[0], p.hs_velocity[1] = vel
    return p


def _flux_rates(O, p, pos, mats):
    s = ParticleStore(len(pos))
    s.pos[:] = pos
    s.material[:] = mats
    s.mass[:] = np.where(np.asarray(mats) == 1, 7900.0, 1.6) * p.dx ** 3
    s.density[:] = np.where(np.asarray(mats) == 1, 7900.0, 1.6)
    s.temperature[:] = 300.0
    o = O.Oracle(p)
    o.upload(s, None)
    o.initialize()
    o.conduction_rhs()
    g, _ = o.download()
    return g.dT_dt


def _peak_rate(p):
    q0 = 2.0 * p.hs_power / (math.pi * p.hs_radius ** 2)
    return q0 * p.dx ** 2 / (7900.0 * p.dx ** 3 * 700.0)


def test_heat_flux_isolated_particle_at_spot_centre(O):
    p = _flux_params()
    r = _flux_rates(O, p, [[0.006, 0.006, 0.006]], [1])
    assert r[0] == pytest.approx(_peak_rate(p), rel=1e-15)


def test_heat_flux_gaussian_profile_and_truncation(O):
    p = _flux_params(r0=1e-3)
    x = 0.006 + np.array([0.0, 1e-3, 2e-3, 3.99e-3, 4.01e-3])  # 0, r0, 2 r0, just inside / outside 4 r0
    # one particle per run, so none shadows another
    got = [_flux_rates(O, p, [[xi, 0.006, 0.006]], [1])[0] for xi in x]
    want = [_peak_rate(p) * math.exp(-2.0 * ((xi - 0.006) / 1e-3) ** 2) for xi in x[:4]] + [0.0]
    assert got[:4] == pytest.approx(want[:4], rel=1e-14)
    assert got[4] == 0.0


def test_heat_flux_shadowing(O):
    p = _flux_params()
    c = [0.006, 0.006, 0.006]
    above = [0.006, 0.006, 0.007]              # dz = dx, lateral 0: shadows the lower particle
    beside = [0.006 + 8e-4, 0.006, 0.007]      # lateral 0.8 dx > 3/4 dx: does not shadow
    half = [0.006, 0.006, 0.006 + 4e-4]        # dz = 0.4 dx <= dx/2: does not shadow
    r = _flux_rates(O, p, [c, above], [1, 1])
    assert r[0] == 0.0 and r[1] > 0.0
    assert _flux_rates(O, p, [c, beside], [1, 1])[0] == pytest.approx(_peak_rate(p), rel=1e-15)
    assert _flux_rates(O, p, [c, half], [1, 1])[0] == pytest.approx(_peak_rate(p), rel=1e-15)
    # a gas particle (material not in the mask) neither absorbs nor shadows
    r = _flux_rates(O, p, [c, above], [1, 0])
    assert r[0] == pytest.approx(_peak_rate(p), rel=1e-15) and r[1] == 0.0


def test_heat_flux_spot_moves_and_wraps(O):
    # spot centre at t^{n+1} = t0 + dt: origin + v t^{n+1}, wrapped on the periodic x axis (L = 12 mm)
    v = 100.0
    t1 = 1.0e-4
    p = _flux_params(r0=1e-3, origin=(0.011, 0.006), vel=(v, 0.0), t0=t1 - 1e-5)
    xc = 0.011 + v * t1 - 0.012  # 0.009 after the wrap
    r = _flux_rates(O, p, [[xc, 0.006, 0.006]], [1])
    assert r[0] == pytest.approx(_peak_rate(p), rel=1e-12)


def test_heat_flux_config_refused_without_heat_equation():
    from paper_2103_07925_b200 import _lib
    import ctypes as C
    lib = _lib.load()
    p = _flux_params()
    p.thermal = 0
    buf = C.create_string_buffer(4096)
    assert lib.sphg_validate(C.byref(p), buf, 4096) == abi.ERR_CONFIG
    assert b"heat source needs the heat equation" in buf.value
