"""Seeded synthetic scenarios for the BASELINE.json configs (inputs only; untimed).

The reference publishes no dataset: BASELINE.json's configs *are* the inputs.
Positions follow the lattice convention of the reference's seed_lattice /
for_each_lattice_point (lattice.hpp:38-82: points at lo + (k + 1/2) dx, last
axis fastest, mass rho0 dx^3); tests/test_oracle_kat.py checks the generator
against the reference's own seed_lattice bit for bit.  Random numbers come from
a counter-based SplitMix64 (53-bit mantissa mapping), so the same arrays are
produced on any host and are uploaded identically to the GPU and the oracle
(SURVEY App. A13).  Streams: 0 jitter, 1 velocities, 2 body placement,
3 temperatures.

Pinned choices for under-specified configs are listed in DESIGN.md §6.
"""
from dataclasses import dataclass, field
import math

import numpy as np

from . import abi
from .store import ParticleStore, empty_bodies

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_STREAM = np.uint64(0xD1B54A32D192ED03)


def splitmix_u01(seed, stream, idx):
    """Counter-based SplitMix64 -> uniform [0,1) with 53-bit mantissa."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = np.array([seed], np.uint64) ^ (np.array([stream], np.uint64) * _STREAM)
        z = base + (idx + np.uint64(1)) * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def lattice_counts(lo, hi, dx):
    """Points per axis, restating for_each_lattice_point (lattice.hpp:43-52)."""
    n = []
    for a in range(3):
        ext = hi[a] - lo[a]
        if ext < 0.0:
            return [0, 0, 0]
        k = int(math.floor(ext / dx + 1e-12))
        if lo[a] + (0.5 + float(k)) * dx > hi[a] + 1e-9 * dx:
            k -= 1
        k += 1
        if k <= 0:
            return [0, 0, 0]
        n.append(k)
    return n


def lattice_box(lo, hi, dx):
    """All lattice points of a box, lexicographic (last axis fastest) — lattice.hpp:53-65."""
    n = lattice_counts(lo, hi, dx)
    if min(n) <= 0:
        return np.zeros((0, 3))
    axes = [lo[a] + (0.5 + np.arange(n[a], dtype=np.float64)) * dx for a in range(3)]
    g = np.meshgrid(*axes, indexing="ij")
    return np.stack([g[0].ravel(), g[1].ravel(), g[2].ravel()], axis=1)


def material(rho0, nu=0.0, cp=0.0, kappa=0.0, c=0.0, pb=0.0, T_t=float("nan"),
             melt=-1, solidify=-1, g=(0.0, 0.0, 0.0), D=0.0, C_t=float("nan")):
    m = abi.Material()
    m.rho0, m.nu, m.cp, m.kappa, m.c, m.pb, m.T_t = rho0, nu, cp, kappa, c, pb, T_t
    m.D, m.C_t = D, C_t
    m.melt_target, m.solidify_target = melt, solidify
    for a in range(3):
        m.body_force[a] = g[a]
    return m


@dataclass
class Scenario:
    name: str
    params: abi.Params
    store: ParticleStore
    bodies: np.ndarray
    steps: int
    info: dict = field(default_factory=dict)


def _params(dx, dt, lo, hi, periodic, mats, kc=0.0, dc=0.0, tvf=1, thermal=0, transitions=0):
    p = abi.Params()
    p.dx, p.h, p.dt, p.t0 = dx, dx, dt, 0.0
    for a in range(3):
        p.lo[a], p.hi[a], p.periodic[a] = lo[a], hi[a], int(periodic[a])
    p.n_mat = len(mats)
    for i, m in enumerate(mats):
        p.mat[i] = m
    p.kc, p.dc, p.tvf, p.thermal, p.transitions = kc, dc, tvf, thermal, transitions
    p.default_fluid_mat = 0
    p.nranks = 1
    return p


def dt_limits_host(params, u_max, m_r):
    """compute_dt terms in plain Python (scenario setup; the product check runs in the
    library): cfl, viscous, body force, contact, conduction (+inf = absent)."""
    inf = float("inf")
    lim = [inf] * 5
    h = params.h if params.h > 0 else params.dx
    bmax = 0.0
    for m in range(params.n_mat):
        M = params.mat[m]
        if M.c > 0:
            lim[0] = min(lim[0], 0.25 * h / (M.c + u_max))
        if M.nu > 0:
            lim[1] = min(lim[1], 0.125 * h * h / M.nu)
        bmax = max(bmax, math.sqrt(sum(M.body_force[a] ** 2 for a in range(3))))
        if params.thermal and M.kappa > 0 and M.cp > 0:
            lim[4] = min(lim[4], 0.1 * M.rho0 * M.cp * h * h / M.kappa)
    if bmax > 0:
        lim[2] = 0.25 * math.sqrt(h / bmax)
    if params.kc > 0 and m_r > 0:
        lim[3] = 0.22 * math.sqrt(m_r / params.kc)
    return lim


def damping_from_ratio(zeta, kc, m_r):
    """d_c = 2 zeta sqrt(k_c m_eff), m_eff = m_r/2 for equal rigid particles."""
    return 2.0 * zeta * math.sqrt(kc * 0.5 * m_r)


def place_spheres(seed, n_spheres, lo, L, r_lo, r_hi, dx, periodic=True, max_tries=None):
    """Rejection-sampled non-overlapping spheres: (periodic) centre distance > R1+R2+dx.

    Candidates are consumed in order from stream 2 (4 draws each: x, y, z, radius).
    """
    lo = np.asarray(lo, float)
    L = np.asarray(L, float)
    rmax = r_hi * dx
    cell = 2.0 * rmax + dx
    ng = np.maximum(1, np.floor(L / cell).astype(int))
    grid = {}
    centers, radii = [], []
    tries = 0
    max_tries = max_tries or 50 * n_spheres + 1000
    batch = 8192
    while len(centers) < n_spheres and tries < max_tries:
        u = splitmix_u01(seed, 2, np.arange(4 * tries, 4 * (tries + batch), dtype=np.uint64)).reshape(batch, 4)
        for k in range(batch):
            tries += 1
            c = lo + u[k, :3] * L
            R = (r_lo + u[k, 3] * (r_hi - r_lo)) * dx
            if not periodic:
                if np.any(c - R < lo + dx) or np.any(c + R > lo + L - dx):
                    continue
            gi = np.floor((c - lo) / L * ng).astype(int) % ng
            ok = True
            for ox in (-1, 0, 1):
                for oy in (-1, 0, 1):
                    for oz in (-1, 0, 1):
                        key = tuple((gi + (ox, oy, oz)) % ng)
                        for s in grid.get(key, ()):
                            d = c - centers[s]
                            if periodic:
                                d = d - L * np.round(d / L)
                            if d @ d <= (R + radii[s] + dx) ** 2:
                                ok = False
                                break
                        if not ok:
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if ok:
                grid.setdefault(tuple(gi), []).append(len(centers))
                centers.append(c)
                radii.append(R)
                if len(centers) == n_spheres:
                    break
    return np.array(centers).reshape(-1, 3), np.array(radii)


def mark_spheres(nlat, lo, dx, L, centers, radii, periodic):
    """Body id (or -1) per lattice point (lattice order) for points inside a sphere.

    Membership is tested on the unjittered lattice point with the minimum-image
    distance, |d|^2 = (dx^2 + dy^2) + dz^2 <= R^2 (ball_region, lattice.hpp:28-36).
    """
    nx, ny, nz = nlat
    owner = np.full(nx * ny * nz, -1, np.int64)
    for k, (c, R) in enumerate(zip(centers, radii)):
        idx = []
        for a, na in enumerate(nlat):
            i0 = int(math.floor((c[a] - R - lo[a]) / dx - 0.5)) - 1
            i1 = int(math.ceil((c[a] + R - lo[a]) / dx - 0.5)) + 1
            ii = np.arange(i0, i1 + 1)
            if periodic[a]:
                ii = np.unique(ii % na)
            else:
                ii = ii[(ii >= 0) & (ii < na)]
            idx.append(ii)
        gx, gy, gz = np.meshgrid(*idx, indexing="ij")
        gx, gy, gz = gx.ravel(), gy.ravel(), gz.ravel()
        p = np.stack([lo[a] + (0.5 + g.astype(np.float64)) * dx for a, g in enumerate((gx, gy, gz))], 1)
        d = p - c
        for a in range(3):
            if periodic[a]:
                d[:, a] -= L[a] * np.round(d[:, a] / L[a])
        inside = ((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]) <= R * R
        lin = ((gx * ny + gy) * nz + gz)[inside]
        owner[lin] = k
    return owner


def particle_inertia(m, dx):
    reff = (0.75 / math.pi) ** (1.0 / 3.0) * dx
    return 0.4 * m * reff * reff


def body_quantities(store, bodies, params):
    """reduce_mass_quantities on the host for the initial state; sets chi (Remark 3.7)."""
    L = np.array([params.hi[a] - params.lo[a] for a in range(3)])
    per = np.array([params.periodic[a] for a in range(3)], bool)
    rig = np.nonzero(store.kind == abi.RIGID)[0]
    if len(rig) == 0:
        return
    order = rig[np.lexsort((rig, store.group[rig]))]
    grp = store.group[order].astype(np.int64)
    starts = np.r_[0, np.nonzero(np.diff(grp))[0] + 1]
    anchor = np.repeat(store.pos[order[starts]], np.diff(np.r_[starts, len(order)]), axis=0)

    def mimg(d):
        d = d.copy()
        for a in range(3):
            if per[a]:
                d[:, a] -= L[a] * np.round(d[:, a] / L[a])
        return d

    m = store.mass[order]
    rel = mimg(store.pos[order] - anchor)
    M = np.add.reduceat(m, starts)
    com = store.pos[order[starts]] + np.add.reduceat(m[:, None] * rel, starts, axis=0) / M[:, None]
    for a in range(3):
        if per[a]:
            lo, hi = params.lo[a], params.hi[a]
            com[:, a] = np.where(com[:, a] < lo, com[:, a] + L[a], np.where(com[:, a] >= hi, com[:, a] - L[a], com[:, a]))
    comp = np.repeat(com, np.diff(np.r_[starts, len(order)]), axis=0)
    d = mimg(store.pos[order] - comp)
    Ir = particle_inertia(m, params.dx)
    d2 = (d[:, 0] ** 2 + d[:, 1] ** 2) + d[:, 2] ** 2
    I6 = np.stack([Ir + m * (d2 - d[:, 0] ** 2), Ir + m * (d2 - d[:, 1] ** 2), Ir + m * (d2 - d[:, 2] ** 2),
                   -m * d[:, 0] * d[:, 1], -m * d[:, 0] * d[:, 2], -m * d[:, 1] * d[:, 2]], 1)
    ids = grp[starts]
    bodies["mass"][ids] = M
    bodies["com"][ids] = com
    bodies["inertia"][ids] = np.add.reduceat(I6, starts, axis=0)
    store.body_frame_pos[order] = d  # q = identity at setup


def _finish(store, bodies):
    rig = store.kind == abi.RIGID
    store.vel[rig] = 0.0
    store.vel_adv[:] = store.vel
    return store, bodies


def periodic_spheres(nside=32, n_spheres=4, r_range=(4.0, 4.0), dx=1e-3, dt=1e-5, seed=2103,
                     rho_f=1000.0, c=10.0, eta=1e-3, rho_s=2000.0, kc=1e3, zeta=0.1, u0=0.01,
                     jitter=0.05, name="c1", steps=100, centers=None, radii=None):
    """BASELINE configs[0] (C1: 32^3, 4 spheres R=4dx) and configs[4] (C5: 400^3, ~20k spheres R~U[3,6]dx).

    Periodic cube, lattice + uniform jitter, fluid u ~ U(-u0, u0), spheres
    relabelled rigid (mass rho_s dx^3), linear EOS (material.hpp:59-62; BASELINE
    says 'Tait'), p_b = p0 = rho0 c^2.
    """
    L = nside * dx
    lo, hi = (0.0, 0.0, 0.0), (L, L, L)
    p0 = rho_f * c * c
    mats = [material(rho_f, nu=eta / rho_f, c=c, pb=p0),   # 0 fluid
            material(rho_s, c=0.0)]                          # 1 solid
    m_r = rho_s * dx ** 3
    params = _params(dx, dt, lo, hi, (1, 1, 1), mats, kc=kc, dc=damping_from_ratio(zeta, kc, m_r))
    # BASELINE prescribes dt = 1e-5 s, above the contact limit 0.22 sqrt(m_r/k_c) = 9.84e-6 s (SURVEY
    # App. B1): the runtime assertion warns instead of refusing (App. A15)
    params.dt_check = abi.DT_WARN if dt > dt_limits_host(params, 0.0, m_r if kc > 0 else 0.0)[3] else abi.DT_REFUSE
    pos = lattice_box(lo, hi, dx)
    n = len(pos)
    if centers is None:
        centers, radii = place_spheres(seed, n_spheres, lo, (L, L, L), r_range[0], r_range[1], dx, True)
    centers, radii = np.asarray(centers, np.float64), np.asarray(radii, np.float64)
    owner = mark_spheres((nside,) * 3, lo, dx, (L, L, L), centers, radii, (True, True, True))
    s = ParticleStore(n)
    u = splitmix_u01(seed, 0, np.arange(3 * n, dtype=np.uint64)).reshape(n, 3)
    pos = pos + (2.0 * u - 1.0) * (jitter * dx)
    pos = np.where(pos < 0.0, pos + L, np.where(pos >= L, pos - L, pos))
    s.pos[:] = pos
    v = splitmix_u01(seed, 1, np.arange(3 * n, dtype=np.uint64)).reshape(n, 3)
    s.vel[:] = (2.0 * v - 1.0) * u0
    rig = owner >= 0
    s.kind[:] = abi.FLUID
    s.kind[rig] = abi.RIGID
    s.group[rig] = owner[rig].astype(np.uint32)
    s.material[rig] = 1
    s.mass[:] = rho_f * dx ** 3
    s.mass[rig] = rho_s * dx ** 3
    s.density[:] = rho_f
    s.density[rig] = rho_s
    bodies = empty_bodies(len(centers))
    bodies["material"] = 1
    body_quantities(s, bodies, params)
    _finish(s, bodies)
    info = dict(n=n, n_fluid=int((~rig).sum()), n_rigid=int(rig.sum()), n_boundary=0,
                n_bodies=len(centers), rigid_fraction=float(rig.mean()))
    return Scenario(name, params, s, bodies, steps, info)


def colliding_spheres(nside=20, R=3.0, gap=-0.3, u=0.05, dx=1e-3, **kw):
    """Two spheres of radius R dx, centres 2R + gap + 1 dx apart along x (the default puts three
    particle pairs of the two bodies within the contact range dx), approaching each other
    at +-u: spring-dashpot contact is active from the first force evaluation."""
    L = nside * dx
    c0 = 0.5 * L
    off = (R + 0.5 * gap + 0.5) * dx  # +0.5: lattice points sit at half spacings
    centers = [(c0 - off, c0, c0), (c0 + off, c0, c0)]
    sc = periodic_spheres(nside=nside, dx=dx, centers=centers, radii=[R * dx, R * dx], name="collide", **kw)
    s, b = sc.store, sc.bodies
    for k, sgn in ((0, 1.0), (1, -1.0)):
        b["vel"][k] = (sgn * u, 0.0, 0.0)
        s.vel[(s.kind == abi.RIGID) & (s.group == k)] = (sgn * u, 0.0, 0.0)
    s.vel_adv[:] = s.vel
    return sc


def config1(**kw):
    """BASELINE configs[0]: 32^3 periodic, 4 spheres R=4dx, dt=1e-5, 100 steps."""
    kw.setdefault("name", "c1")
    return periodic_spheres(**kw)


def config5(nside=400, n_spheres=20000, **kw):
    """BASELINE configs[4]: 400^3 = 64M periodic, ~20k spheres R~U[3,6]dx (App. B8: sphere count kept)."""
    kw.setdefault("name", "c5")
    kw.setdefault("steps", 100)
    return periodic_spheres(nside=nside, n_spheres=n_spheres, r_range=(3.0, 6.0), **kw)


def closed_box_melting(nside=64, dx=1e-3, dt=5e-6, seed=2107, n_grid=3, r_range=(3.0, 6.0),
                       T0=300.0, T_hot=1800.0, T_t=1700.0, rho=7900.0, c=20.0, nu=1e-6, cp=700.0,
                       kappa=20.0, g=-9.81, kc=10.0, zeta=0.1, jitter=0.05, melt_forcing=False,
                       name="c2", steps=500):
    """BASELINE configs[1] (C2): closed box, 3-layer walls, 27 spheres on a jittered 3x3x3 grid.

    Materials: 0 carrier liquid (no transition),
    1 solid metal (T_t, melts into 2), 2 melt liquid (T_t, solidifies into 1),
    3 wall.  Bottom wall = Dirichlet group 0 at T_hot.  melt_forcing=True is
    the parity variant of App. B5: sphere temperatures ~ U[T_t-5, T_t+5] and a
    melt-liquid layer at the same temperatures, so flags flip at step 1.
    """
    L = nside * dx
    nl = 3  # wall_layers = floor(r_c/dx) (config.hpp:105)
    lo = (-nl * dx,) * 3
    hi = (L + nl * dx,) * 3
    p0 = rho * c * c
    grav = (0.0, 0.0, g)
    mats = [material(rho, nu=nu, cp=cp, kappa=kappa, c=c, pb=p0, g=grav),                        # 0 carrier
            material(rho, cp=cp, kappa=kappa, c=c, T_t=T_t, melt=2, g=grav),                     # 1 solid
            material(rho, nu=nu, cp=cp, kappa=kappa, c=c, pb=p0, T_t=T_t, solidify=1, g=grav),  # 2 melt
            material(rho, cp=cp, kappa=kappa, c=c)]                                               # 3 wall
    m_r = rho * dx ** 3
    params = _params(dx, dt, lo, hi, (0, 0, 0), mats, kc=kc, dc=damping_from_ratio(zeta, kc, m_r),
                     thermal=1, transitions=1)
    params.n_dirichlet = 1
    params.dirichlet_T[0].n = 1
    params.dirichlet_T[0].t_end[0] = 1e30
    params.dirichlet_T[0].value[0] = T_hot
    fl = lattice_box((0.0,) * 3, (L,) * 3, dx)
    wl = lattice_box(lo, hi, dx)
    outside = np.any((wl < 0.0) | (wl > L), axis=1)
    wl = wl[outside]
    nf, nw = len(fl), len(wl)
    # spheres on a jittered grid
    ug = splitmix_u01(seed, 2, np.arange(4 * n_grid ** 3, dtype=np.uint64)).reshape(-1, 4)
    centers, radii = [], []
    sp = L / n_grid
    k = 0
    for i in range(n_grid):
        for j in range(n_grid):
            for l in range(n_grid):
                c0 = np.array([(i + 0.5) * sp, (j + 0.5) * sp, (l + 0.5) * sp])
                centers.append(c0 + (2.0 * ug[k, :3] - 1.0) * 2.0 * dx)
                radii.append((r_range[0] + ug[k, 3] * (r_range[1] - r_range[0])) * dx)
                k += 1
    centers, radii = np.array(centers), np.array(radii)
    owner = mark_spheres((nside,) * 3, (0.0,) * 3, dx, (L,) * 3, centers, radii, (False,) * 3)
    n = nf + nw
    s = ParticleStore(n)
    u = splitmix_u01(seed, 0, np.arange(3 * nf, dtype=np.uint64)).reshape(nf, 3)
    s.pos[:nf] = fl + (2.0 * u - 1.0) * (jitter * dx)
    s.pos[nf:] = wl
    rig = np.zeros(n, bool)
    rig[:nf] = owner >= 0
    s.kind[:nf] = abi.FLUID
    s.kind[nf:] = abi.BOUNDARY
    s.kind[rig] = abi.RIGID
    s.group[rig] = owner[owner >= 0].astype(np.uint32)
    s.material[:nf] = 0
    s.material[rig] = 1
    s.material[nf:] = 3
    s.mass[:] = rho * dx ** 3
    s.density[:] = rho
    s.temperature[:] = T0
    bottom = np.zeros(n, bool)
    bottom[nf:] = wl[:, 2] < 0.0
    s.dirichlet_T[bottom] = 0
    s.temperature[bottom] = T_hot
    if melt_forcing:
        tu = splitmix_u01(seed, 3, np.arange(n, dtype=np.uint64))
        Tf = (T_t - 5.0) + 10.0 * tu
        s.temperature[rig] = Tf[rig]
        band = np.zeros(n, bool)
        band[:nf] = (fl[:, 2] > 0.35 * L) & (fl[:, 2] < 0.65 * L)
        band &= s.kind == abi.FLUID
        s.material[band] = 2
        s.temperature[band] = Tf[band]
        s.temperature[(s.kind == abi.FLUID) & ~band] = T_t
    bodies = empty_bodies(len(centers))
    bodies["material"] = 1
    body_quantities(s, bodies, params)
    _finish(s, bodies)
    info = dict(n=n, n_fluid=int((s.kind == abi.FLUID).sum()), n_rigid=int(rig.sum()), n_boundary=nw,
                n_bodies=len(centers), rigid_fraction=float(rig.mean()))
    return Scenario(name, params, s, bodies, steps, info)


def two_phase_with_bodies(nside=128, dx=1e-3, dt=None, seed=2111, n_bodies=200, r_range=(2.0, 4.0),
                          liquid_frac=0.6, rho_l=1000.0, rho_g=1.0, eta_l=1e-3, eta_g=1e-5, c=20.0,
                          rho_s=1200.0, g=-9.81, kc=10.0, zeta=0.1, jitter=0.05, name="c3", steps=200):
    """BASELINE configs[2] (C3): closed box, lower liquid_frac liquid (rho 1000, eta 1e-3), upper gas
    (rho 1, eta 1e-5), shared background pressure, rigid cubes and spheres (50/50 by seed, edge or
    diameter 4-8 dx -> half-size r_range) of density 1200 placed in the liquid, gravity, isothermal.
    Pinned: equal reference pressures p0 = rho c^2 in both phases (c_liquid = c,
    c_gas = c sqrt(rho_l / rho_g)), shared p_b = p0, dt = 0.2 h / c_gas, 3-layer walls, k_c = 10.
    Exercises the multi-viscosity (eta~ harmonic mean) and multi-EOS (dominant wall material) paths."""
    c_g = c * math.sqrt(rho_l / rho_g)
    if dt is None:
        dt = 0.2 * dx / c_g
    L = nside * dx
    nl = 3
    lo = (-nl * dx,) * 3
    hi = (L + nl * dx,) * 3
    pb = rho_l * c * c
    grav = (0.0, 0.0, g)
    mats = [material(rho_l, nu=eta_l / rho_l, c=c, pb=pb, g=grav),   # 0 liquid
            material(rho_g, nu=eta_g / rho_g, c=c_g, pb=pb, g=grav), # 1 gas
            material(rho_s, c=0.0, g=grav),                            # 2 solid
            material(rho_l, c=c)]                                       # 3 wall
    m_r = rho_s * dx ** 3
    params = _params(dx, dt, lo, hi, (0, 0, 0), mats, kc=kc, dc=damping_from_ratio(zeta, kc, m_r))
    fl = lattice_box((0.0,) * 3, (L,) * 3, dx)
    wl = lattice_box(lo, hi, dx)
    wl = wl[np.any((wl < 0.0) | (wl > L), axis=1)]
    nf, nw = len(fl), len(wl)
    # bodies: centres in the liquid, non-overlapping; even ids spheres, odd ids cubes
    zmax = liquid_frac * L
    centers, radii = place_spheres(seed, n_bodies, (0.0, 0.0, 0.0), (L, L, zmax), r_range[0], r_range[1], dx,
                                   periodic=False)
    owner = np.full(nf, -1, np.int64)
    n1 = nside
    for k, (cc, R) in enumerate(zip(centers, radii)):
        d = fl - cc
        if k % 2 == 0:
            inside = ((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]) <= R * R
        else:
            inside = np.all(np.abs(d) <= R, axis=1)  # axis-aligned cube (box_region, lattice.hpp:22-25)
        owner[inside & (owner < 0)] = k
    n = nf + nw
    s = ParticleStore(n)
    u = splitmix_u01(seed, 0, np.arange(3 * nf, dtype=np.uint64)).reshape(nf, 3)
    s.pos[:nf] = fl + (2.0 * u - 1.0) * (jitter * dx)
    s.pos[nf:] = wl
    rig = np.zeros(n, bool)
    rig[:nf] = owner >= 0
    gas = np.zeros(n, bool)
    gas[:nf] = fl[:, 2] >= zmax
    s.kind[:nf] = abi.FLUID
    s.kind[nf:] = abi.BOUNDARY
    s.kind[rig] = abi.RIGID
    s.group[rig] = owner[owner >= 0].astype(np.uint32)
    s.material[:nf] = 0
    s.material[gas & ~rig] = 1
    s.material[rig] = 2
    s.material[nf:] = 3
    rho = np.where(gas, rho_g, rho_l)
    rho[rig] = rho_s
    rho[nf:] = rho_l
    s.mass[:] = rho * dx ** 3
    s.density[:] = rho
    bodies = empty_bodies(len(centers))
    bodies["material"] = 2
    body_quantities(s, bodies, params)
    _finish(s, bodies)
    info = dict(n=n, n_fluid=int((s.kind == abi.FLUID).sum()), n_rigid=int(rig.sum()), n_boundary=nw,
                n_bodies=len(centers), rigid_fraction=float(rig.mean()), n_gas=int((gas & ~rig).sum()))
    return Scenario(name, params, s, bodies, steps, info)


def dissolving_bodies(nside=32, dx=1e-3, dt=1e-5, seed=2113, n_bodies=4, r_range=(3.0, 5.0), rho=1000.0,
                      c=10.0, nu_g=1e-5, nu_c=2e-5, D_g=8e-3, D_s=2e-3, D_c=2e-3, C_t=0.8, kc=10.0, zeta=0.1,
                      jitter=0.05, forcing=False, name="dissolve", steps=200):
    """Concentration-driven dissolution (PAPER:936 gastric example in 3D SI units):
    closed box of "gastric juice" held at C = 1 by a Dirichlet concentration group on every juice
    particle (PAPER: "fixed to C^ = 1.0 at all times"), rigid boluses with C0 = 0 and diffusivity
    D_s that dissolve into "chyme" (fluid, D_c) when C > C_t = 0.8; juice diffusivity D_g = 4 D_s
    (the paper's 1.0 : 0.25), equal densities, no gravity, isothermal; concentration transitions
    (TransitionMode::Concentration).  forcing=True: body concentrations ~ U[C_t - 0.05, C_t + 0.05]
    so dissolution starts at step 1 (the parity variant)."""
    L = nside * dx
    nl = 3
    lo = (-nl * dx,) * 3
    hi = (L + nl * dx,) * 3
    p0 = rho * c * c
    mats = [material(rho, nu=nu_g, c=c, pb=p0, D=D_g),                 # 0 gastric juice
            material(rho, c=c, D=D_s, C_t=C_t, melt=2),                 # 1 bolus (solid)
            material(rho, nu=nu_c, c=c, pb=p0, D=D_c),                  # 2 chyme
            material(rho, c=c)]                                          # 3 wall (no diffusion)
    m_r = rho * dx ** 3
    params = _params(dx, dt, lo, hi, (0, 0, 0), mats, kc=kc, dc=damping_from_ratio(zeta, kc, m_r),
                     transitions=abi.TRANSITIONS_CONCENTRATION)
    params.diffusion = 1
    params.n_dirichlet_c = 1
    params.dirichlet_C[0].n = 1
    params.dirichlet_C[0].t_end[0] = 1e30
    params.dirichlet_C[0].value[0] = 1.0
    fl = lattice_box((0.0,) * 3, (L,) * 3, dx)
    wl = lattice_box(lo, hi, dx)
    wl = wl[np.any((wl < 0.0) | (wl > L), axis=1)]
    nf, nw = len(fl), len(wl)
    centers, radii = place_spheres(seed, n_bodies, (0.0,) * 3, (L,) * 3, r_range[0], r_range[1], dx,
                                   periodic=False)
    owner = mark_spheres((nside,) * 3, (0.0,) * 3, dx, (L,) * 3, centers, radii, (False,) * 3)
    n = nf + nw
    st = ParticleStore(n)
    u = splitmix_u01(seed, 0, np.arange(3 * nf, dtype=np.uint64)).reshape(nf, 3)
    st.pos[:nf] = fl + (2.0 * u - 1.0) * (jitter * dx)
    st.pos[nf:] = wl
    rig = np.zeros(n, bool)
    rig[:nf] = owner >= 0
    st.kind[:nf] = abi.FLUID
    st.kind[nf:] = abi.BOUNDARY
    st.kind[rig] = abi.RIGID
    st.group[rig] = owner[owner >= 0].astype(np.uint32)
    st.material[:nf] = 0
    st.material[rig] = 1
    st.material[nf:] = 3
    st.mass[:] = m_r
    st.density[:] = rho
    juice = st.kind == abi.FLUID
    st.concentration[juice] = 1.0
    st.dirichlet_C[juice] = 0
    if forcing:
        cu = splitmix_u01(seed, 3, np.arange(n, dtype=np.uint64))
        st.concentration[rig] = (C_t - 0.05) + 0.1 * cu[rig]
    bodies = empty_bodies(len(centers))
    bodies["material"] = 1
    body_quantities(st, bodies, params)
    _finish(st, bodies)
    info = dict(n=n, n_fluid=int(juice.sum()), n_rigid=int(rig.sum()), n_boundary=nw, n_bodies=len(centers),
                rigid_fraction=float(rig.mean()))
    return Scenario(name, params, st, bodies, steps, info)


def couette_channel(nside=16, nz=None, dx=1e-3, dt=1e-5, seed=2117, rho=1000.0, c=10.0, nu=1e-5, u_wall=0.01,
                    jitter=0.05, name="couette", steps=200):
    """Moving wall groups (PAPER §4.2): channel periodic in x and y,
    3-layer walls below z = 0 (wall group 0, fixed) and above z = H (wall group 1, moving along x
    with u_wall; see `wall_velocity`).  Fluid at rest initially, no gravity, no bodies."""
    nz = nz or nside
    L = nside * dx
    H = nz * dx
    nl = 3
    lo = (0.0, 0.0, -nl * dx)
    hi = (L, L, H + nl * dx)
    p0 = rho * c * c
    mats = [material(rho, nu=nu, c=c, pb=p0), material(rho, c=c)]  # 0 fluid, 1 wall
    params = _params(dx, dt, lo, hi, (1, 1, 0), mats)
    fl = lattice_box((0.0, 0.0, 0.0), (L, L, H), dx)
    wl = lattice_box(lo, hi, dx)
    wl = wl[(wl[:, 2] < 0.0) | (wl[:, 2] > H)]
    nf, nw = len(fl), len(wl)
    n = nf + nw
    st = ParticleStore(n)
    u = splitmix_u01(seed, 0, np.arange(3 * nf, dtype=np.uint64)).reshape(nf, 3)
    pos = fl + (2.0 * u - 1.0) * (jitter * dx)
    for a in range(2):  # periodic axes: wrap the jitter
        pos[:, a] = np.mod(pos[:, a], L)
    st.pos[:nf] = pos
    st.pos[nf:] = wl
    st.kind[:nf] = abi.FLUID
    st.kind[nf:] = abi.BOUNDARY
    st.material[nf:] = 1
    st.group[nf:] = (wl[:, 2] > H).astype(np.uint32)  # wall group: 0 bottom, 1 top
    st.mass[:] = rho * dx ** 3
    st.density[:] = rho
    bodies = empty_bodies(0)
    _finish(st, bodies)
    info = dict(n=n, n_fluid=nf, n_rigid=0, n_boundary=nw, n_bodies=0, rigid_fraction=0.0, u_wall=u_wall)
    return Scenario(name, params, st, bodies, steps, info)


def wall_velocity(u_wall, omega=0.0):
    """velocity(g, t) of couette_channel's wall groups: group 1 moves along x with
    u_wall (omega = 0) or u_wall sin(omega t); group 0 is fixed."""
    def v(g, t):
        if g != 1:
            return (0.0, 0.0, 0.0)
        return (u_wall * (math.sin(omega * t) if omega else 1.0), 0.0, 0.0)
    return v


def deposit_grains(seed, n_grains, Lx, Ly, z0, dx, median=4.0, sigma=0.3, r_clip=(2.0, 8.0), gap=1.0, trials=32):
    """Seeded sequential deposition of log-normal spheres onto a plane (C4 powder layer).

    Radii R = median exp(sigma N(0,1)) dx (Box-Muller on stream 4), clipped to r_clip.  Grain k is
    dropped vertically at `trials` positions (x, y) ~ U(periodic footprint) (stream 2); at each it
    rests at the first contact, with the substrate at z0 (centre z0 + R + gap dx) or with an earlier
    grain j (centre distance R + R_j + gap dx, minimum image in x and y), and it is placed at the
    lowest of these rests (first on ties).  The lowest-of-several drops stands in for the settling of
    a DEM random close packing, which is not run.  Returns centres (n, 3)
    and radii (n,)."""
    u = splitmix_u01(seed, 4, np.arange(2 * n_grains, dtype=np.uint64)).reshape(n_grains, 2)
    z = np.sqrt(-2.0 * np.log1p(-u[:, 0])) * np.cos(2.0 * math.pi * u[:, 1])
    radii = np.clip(median * np.exp(sigma * z), r_clip[0], r_clip[1]) * dx
    xy_all = splitmix_u01(seed, 2, np.arange(2 * trials * n_grains, dtype=np.uint64)).reshape(n_grains, trials, 2)
    xy_all = xy_all * (Lx, Ly)
    xy = np.zeros((n_grains, 2))
    cz = np.zeros(n_grains)
    g = gap * dx
    for k in range(n_grains):
        R = radii[k]
        t = xy_all[k]                                  # (trials, 2)
        zk = np.full(trials, z0 + R + g)
        if k:
            d = xy[None, :k, :] - t[:, None, :]        # (trials, k, 2)
            d[..., 0] -= Lx * np.round(d[..., 0] / Lx)
            d[..., 1] -= Ly * np.round(d[..., 1] / Ly)
            rho2 = d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]
            s2 = (R + radii[:k] + g) ** 2
            zc = np.where(rho2 < s2, cz[:k] + np.sqrt(np.maximum(s2 - rho2, 0.0)), -np.inf)
            zk = np.maximum(zk, zc.max(axis=1))
        b = int(np.argmin(zk))
        xy[k] = t[b]
        cz[k] = zk[b]
    return np.column_stack([xy, cz]), radii


def powder_bed(nx=400, ny=200, nz=194, dx=5e-6, dt=None, seed=2119, n_grains=5000, median=4.0, sigma=0.3,
               T0=1550.0, T_t=1700.0, rho=7900.0, c=20.0, nu=1e-6, cp=700.0, kappa=20.0,
               rho_gas=1.6, eta_gas=2.2e-5, cp_gas=520.0, kappa_gas=0.018, power=200.0, r0_dx=20.0,
               scan_speed=1.0, g=-9.81, kc=1e3, zeta=0.1, jitter=0.05, name="c4", steps=1000):
    """BASELINE configs[3] (C4): powder-bed-fusion-like melt, ~16M particles at dx = 5e-6 m.

    Periodic in x and y; a 3-layer substrate slab (boundary particles, Dirichlet at T0) at the bottom
    and a 3-layer lid on top; n_grains rigid metal grains (log-normal radii, median 4 dx, sigma 0.3)
    deposited on the substrate by deposit_grains; argon-like gas everywhere else (rho 1.6).  Metal as
    C2 (rho 7900, c 20, c_p 700, kappa 20, T_t 1700: solid 1 melts into liquid 2, which solidifies
    into 1).  A Gaussian surface heat flux of `power` W, 1/e^2 radius r0_dx dx, scans along x at
    `scan_speed` m/s from x = L_x/4 on the centre line [P21] (an extension: the reference has no heat
    sources).  Pinned: gas c = c sqrt(rho / rho_gas) with one shared
    p_b = rho c^2 (as C3), dt = 0.2 h / c_gas, bed preheated to T0 = 1550 K so the exposed grain
    surface reaches T_t within the run (the flux heats it by ~330 K over 1000 steps).
    nz counts the interior lattice layers (200 with the two 3-layer walls)."""
    c_g = c * math.sqrt(rho / rho_gas)
    if dt is None:
        dt = 0.2 * dx / c_g
    Lx, Ly, Lz = nx * dx, ny * dx, nz * dx
    nl = 3
    lo = (0.0, 0.0, -nl * dx)
    hi = (Lx, Ly, Lz + nl * dx)
    pb = rho * c * c
    grav = (0.0, 0.0, g)
    mats = [material(rho_gas, nu=eta_gas / rho_gas, cp=cp_gas, kappa=kappa_gas, c=c_g, pb=pb, g=grav),  # 0 gas
            material(rho, cp=cp, kappa=kappa, c=c, T_t=T_t, melt=2, g=grav),                          # 1 solid
            material(rho, nu=nu, cp=cp, kappa=kappa, c=c, pb=pb, T_t=T_t, solidify=1, g=grav),       # 2 melt
            material(rho, cp=cp, kappa=kappa, c=c),                                                    # 3 substrate
            material(rho_gas, c=c_g)]                                                                  # 4 lid
    m_r = rho * dx ** 3
    params = _params(dx, dt, lo, hi, (1, 1, 0), mats, kc=kc, dc=damping_from_ratio(zeta, kc, m_r),
                     thermal=1, transitions=1)
    params.n_dirichlet = 1
    params.dirichlet_T[0].n = 1
    params.dirichlet_T[0].t_end[0] = 1e30
    params.dirichlet_T[0].value[0] = T0
    params.heat_source = 1
    params.hs_material_mask = (1 << 1) | (1 << 2) | (1 << 3)
    params.hs_power = power
    params.hs_radius = r0_dx * dx
    params.hs_origin[0], params.hs_origin[1] = 0.25 * Lx, 0.5 * Ly
    params.hs_velocity[0] = scan_speed
    fl = lattice_box((0.0, 0.0, 0.0), (Lx, Ly, Lz), dx)
    wl = lattice_box(lo, hi, dx)
    wl = wl[(wl[:, 2] < 0.0) | (wl[:, 2] > Lz)]
    nf, nw = len(fl), len(wl)
    centers, radii = deposit_grains(seed, n_grains, Lx, Ly, 0.0, dx, median, sigma)
    keep = centers[:, 2] + radii < Lz - 3.0 * dx  # grains must fit under the lid
    centers, radii = centers[keep], radii[keep]
    owner = mark_spheres((nx, ny, nz), (0.0, 0.0, 0.0), dx, (Lx, Ly, Lz), centers, radii, (True, True, False))
    n = nf + nw
    st = ParticleStore(n)
    u = splitmix_u01(seed, 0, np.arange(3 * nf, dtype=np.uint64)).reshape(nf, 3)
    p = fl + (2.0 * u - 1.0) * (jitter * dx)
    for a, L in ((0, Lx), (1, Ly)):  # periodic wrap of the jittered lattice
        p[:, a] = np.where(p[:, a] < 0.0, p[:, a] + L, np.where(p[:, a] >= L, p[:, a] - L, p[:, a]))
    st.pos[:nf] = p
    st.pos[nf:] = wl
    rig = np.zeros(n, bool)
    rig[:nf] = owner >= 0
    st.kind[:nf] = abi.FLUID
    st.kind[nf:] = abi.BOUNDARY
    st.kind[rig] = abi.RIGID
    st.group[rig] = owner[owner >= 0].astype(np.uint32)
    st.material[:nf] = 0
    st.material[rig] = 1
    sub = np.zeros(n, bool)
    sub[nf:] = wl[:, 2] < 0.0
    st.material[nf:] = 4
    st.material[sub] = 3
    st.dirichlet_T[sub] = 0
    dens = np.full(n, rho_gas)
    dens[rig | sub] = rho
    st.mass[:] = dens * dx ** 3
    st.density[:] = dens
    st.temperature[:] = T0
    bodies = empty_bodies(len(centers))
    bodies["material"] = 1
    body_quantities(st, bodies, params)
    _finish(st, bodies)
    info = dict(n=n, n_fluid=int((st.kind == abi.FLUID).sum()), n_rigid=int(rig.sum()), n_boundary=nw,
                n_bodies=len(centers), rigid_fraction=float(rig.mean()),
                bed_height_dx=float(np.max(centers[:, 2] + radii) / dx) if len(centers) else 0.0)
    return Scenario(name, params, st, bodies, steps, info)


def paper_strong_scaling(nside=150, n_grid=6, dx=0.2, D=2.5, rho_f=1.0, nu=1.0, rho_s=10.0, g=1.0, c=50.0,
                         dt=1e-3, kc=1e3, zeta=0.1, jitter=0.0, seed=2123, name="paper46", steps=100):
    """The paper's own strong-scaling case: a cubic box of edge L = 30
    (150^3 lattice at dx = 0.2) inside 3-layer boundary walls (156^3 - 150^3 = 421,416), 216 = 6^3
    rigid spheres of diameter 2.5 and density 10 on a regular grid, fluid rho 1, nu 1, c 50
    (p0 = p_b = 2500), gravity 1 downward on fluid and bodies, 48^3 cells of edge 0.65
    (cell_edge_override), dt = 1e-3: 3,796,416 particles, as the paper's 3.79e6 (3.15e6 fluid,
    2.20e5 rigid, 4.21e5 boundary).  Pinned (the paper does not state them for this case): k_c = 1e3
    with damping ratio 0.1 (contact limit 0.22 sqrt(m_r/k_c) = 2.0e-3 >= dt), no jitter (the paper
    starts from the lattice at rest).  nside / n_grid shrink it for the parity tests (same dx, box
    edge nside dx, sphere centres at (k + 1/2) L / n_grid)."""
    L = nside * dx
    nl = 3
    lo = (-nl * dx,) * 3
    hi = (L + nl * dx,) * 3
    p0 = rho_f * c * c
    grav = (0.0, 0.0, -g)
    mats = [material(rho_f, nu=nu, c=c, pb=p0, g=grav),  # 0 fluid
            material(rho_s, c=0.0, g=grav),              # 1 solid
            material(rho_f, c=c)]                        # 2 wall
    m_r = rho_s * dx ** 3
    params = _params(dx, dt, lo, hi, (0, 0, 0), mats, kc=kc, dc=damping_from_ratio(zeta, kc, m_r))
    # the paper's dt = 1e-3 is exactly the CFL limit 0.25 h / c at rest, so any flow exceeds it: the
    # runtime assertion warns instead of refusing the paper's own setting
    params.dt_check = abi.DT_WARN
    if nside == 150:
        params.cell_edge_override = 0.65  # 48^3 cells over the 31.2 box
    fl = lattice_box((0.0,) * 3, (L,) * 3, dx)
    wl = lattice_box(lo, hi, dx)
    wl = wl[np.any((wl < 0.0) | (wl > L), axis=1)]
    nf, nw = len(fl), len(wl)
    sp = L / n_grid
    ax = (np.arange(n_grid) + 0.5) * sp
    centers = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3)
    radii = np.full(len(centers), 0.5 * D)
    owner = mark_spheres((nside,) * 3, (0.0,) * 3, dx, (L,) * 3, centers, radii, (False,) * 3)
    n = nf + nw
    st = ParticleStore(n)
    if jitter > 0.0:
        u = splitmix_u01(seed, 0, np.arange(3 * nf, dtype=np.uint64)).reshape(nf, 3)
        fl = fl + (2.0 * u - 1.0) * (jitter * dx)
    st.pos[:nf] = fl
    st.pos[nf:] = wl
    rig = np.zeros(n, bool)
    rig[:nf] = owner >= 0
    st.kind[:nf] = abi.FLUID
    st.kind[nf:] = abi.BOUNDARY
    st.kind[rig] = abi.RIGID
    st.group[rig] = owner[owner >= 0].astype(np.uint32)
    st.material[rig] = 1
    st.material[nf:] = 2
    dens = np.full(n, rho_f)
    dens[rig] = rho_s
    st.mass[:] = dens * dx ** 3
    st.density[:] = dens
    bodies = empty_bodies(len(centers))
    bodies["material"] = 1
    body_quantities(st, bodies, params)
    _finish(st, bodies)
    info = dict(n=n, n_fluid=int((st.kind == abi.FLUID).sum()), n_rigid=int(rig.sum()), n_boundary=nw,
                n_bodies=len(centers), rigid_fraction=float(rig.mean()))
    return Scenario(name, params, st, bodies, steps, info)


def hydrostatic_tank(nxy=10, nz=20, dx=1e-3, dt=1e-5, rho=1000.0, c=10.0, nu=1e-6, g=-9.81, pb=0.0,
                     hydrostatic=True, sphere_radius=0.0, rho_s=1200.0, jitter=0.0, seed=2129,
                     name="tank", steps=0):
    """A water column for the reference's hydrostatic KATs: periodic in x and y
    (nxy dx), fluid 0 <= z <= H = nz dx between 3-layer fixed walls below z = 0 and above z = H
    (closed, so no free surface), gravity g along z.  hydrostatic=True starts from the analytic
    field p = rho0 |g| (H - z), rho = rho0 + p / c^2 (the EOS inverse, material.hpp:64-67);
    otherwise rho = rho0, p = 0.  sphere_radius > 0 relabels a sphere (radius in dx, centred at
    mid-depth) as a rigid body of density rho_s (SPEC:287 submerged body).  Materials: 0 fluid,
    1 wall, 2 solid."""
    L = nxy * dx
    H = nz * dx
    nl = 3
    lo = (0.0, 0.0, -nl * dx)
    hi = (L, L, H + nl * dx)
    mats = [material(rho, nu=nu, c=c, pb=pb, g=(0.0, 0.0, g)), material(rho, c=c), material(rho_s, c=0.0)]
    params = _params(dx, dt, lo, hi, (1, 1, 0), mats, tvf=1 if pb > 0 else 0)
    fl = lattice_box((0.0, 0.0, 0.0), (L, L, H), dx)
    wl = lattice_box(lo, hi, dx)
    wl = wl[(wl[:, 2] < 0.0) | (wl[:, 2] > H)]
    nf, nw = len(fl), len(wl)
    n = nf + nw
    st = ParticleStore(n)
    pos = fl.copy()
    if jitter:
        u = splitmix_u01(seed, 0, np.arange(3 * nf, dtype=np.uint64)).reshape(nf, 3)
        pos = pos + (2.0 * u - 1.0) * (jitter * dx)
        for a in range(2):
            pos[:, a] = np.mod(pos[:, a], L)
    st.pos[:nf] = pos
    st.pos[nf:] = wl
    st.kind[:nf] = abi.FLUID
    st.kind[nf:] = abi.BOUNDARY
    st.material[nf:] = 1
    st.mass[:] = rho * dx ** 3
    st.density[:] = rho
    if hydrostatic:
        p = rho * abs(g) * (H - pos[:, 2])
        st.pressure[:nf] = p
        st.density[:nf] = rho + p / (c * c)
    nb = 0
    if sphere_radius > 0.0:
        cen = np.array([0.5 * L, 0.5 * L, 0.5 * H])
        owner = mark_spheres((nxy, nxy, nz), (0.0, 0.0, 0.0), dx, (L, L, H), [cen], [sphere_radius * dx],
                             (True, True, False))
        rig = np.zeros(n, bool)
        rig[:nf] = owner >= 0
        st.kind[rig] = abi.RIGID
        st.material[rig] = 2
        st.group[rig] = 0
        st.mass[rig] = rho_s * dx ** 3
        st.density[rig] = rho_s
        st.pressure[rig] = 0.0
        nb = 1
    bodies = empty_bodies(nb)
    bodies["material"] = 2
    body_quantities(st, bodies, params)
    _finish(st, bodies)
    info = dict(n=n, n_fluid=int((st.kind == abi.FLUID).sum()), n_rigid=int((st.kind == abi.RIGID).sum()),
                n_boundary=nw, n_bodies=nb, H=H)
    return Scenario(name, params, st, bodies, steps, info)


def conduction_rod(nx=20, nyz=10, dx=1.0, rho=1.0, cp=1.0, kappa=1.0, T_lo=0.0, T_hi=1.0, name="rod", steps=0):
    """The reference's steady-conduction KAT in 3D: a bar of particles 0 <= x <= nx dx
    (periodic in y and z, so the problem is one-dimensional) between 3-layer Dirichlet end walls
    held at T_lo (x < 0) and T_hi (x > nx dx).  The bar is a fixed (immobile) rigid body, so only
    conduction acts; dt = 0.5 x the conduction limit 0.1 rho c_p h^2 / kappa."""
    nl = 3
    Lx = nx * dx
    W = nyz * dx
    lo = (-nl * dx, 0.0, 0.0)
    hi = (Lx + nl * dx, W, W)
    dt = 0.5 * 0.1 * rho * cp * dx * dx / kappa
    mats = [material(rho, c=1.0, cp=cp, kappa=kappa), material(rho, cp=cp, kappa=kappa)]  # 0 fluid (unused), 1 solid
    params = _params(dx, dt, lo, hi, (0, 1, 1), mats, tvf=0, thermal=1)
    params.n_dirichlet = 2
    for gidx, v in ((0, T_lo), (1, T_hi)):
        params.dirichlet_T[gidx].n = 1
        params.dirichlet_T[gidx].t_end[0] = 1e30
        params.dirichlet_T[gidx].value[0] = v
    pts = lattice_box(lo, hi, dx)
    n = len(pts)
    st = ParticleStore(n)
    st.pos[:] = pts
    wall = (pts[:, 0] < 0.0) | (pts[:, 0] > Lx)
    st.kind[:] = abi.RIGID
    st.kind[wall] = abi.BOUNDARY
    st.material[:] = 1
    st.group[~wall] = 0
    st.mass[:] = rho * dx ** 3
    st.density[:] = rho
    st.dirichlet_T[pts[:, 0] < 0.0] = 0
    st.dirichlet_T[pts[:, 0] > Lx] = 1
    st.temperature[:] = 0.5 * (T_lo + T_hi)
    st.temperature[pts[:, 0] < 0.0] = T_lo
    st.temperature[pts[:, 0] > Lx] = T_hi
    bodies = empty_bodies(1)
    bodies["material"] = 1
    bodies["mobile"] = 0
    body_quantities(st, bodies, params)
    _finish(st, bodies)
    info = dict(n=n, n_fluid=0, n_rigid=int((~wall).sum()), n_boundary=int(wall.sum()), n_bodies=1, Lx=Lx)
    return Scenario(name, params, st, bodies, steps, info)


def buffer_channel(nx=32, ny=10, nz=16, dx=1e-3, dt=1e-5, rho=1000.0, c=10.0, nu=1e-6, u_mean=0.05,
                   t_start=0.0, zone=4, jitter=0.05, seed=2131, name="channel", steps=200):
    """Inflow / outflow buffer zones (§4.4) [P23]: a channel
    periodic in x and y between 3-layer walls below z = 0 and above z = H.  The first `zone` dx of x are
    the inflow zone and the last `zone` dx the outflow zone; both prescribe the parabolic profile
    u_x = u_mean 6 xi (1 - xi), xi = z / H, for t > t_start.  The periodic wrap carries particles
    leaving the outflow zone into the inflow zone (particle recycling)."""
    Lx, W, H = nx * dx, ny * dx, nz * dx
    nl = 3
    lo = (0.0, 0.0, -nl * dx)
    hi = (Lx, W, H + nl * dx)
    mats = [material(rho, nu=nu, c=c, pb=rho * c * c), material(rho, c=c)]  # 0 fluid, 1 wall
    params = _params(dx, dt, lo, hi, (1, 1, 0), mats)
    params.n_buffers = 2
    for b, (x0, x1) in enumerate(((0.0, zone * dx), (Lx - zone * dx, Lx))):
        B = params.buffers[b]
        B.axis, B.profile_axis = 0, 2
        B.lo[0], B.hi[0] = x0, x1
        B.lo[1], B.hi[1] = 0.0, W
        B.lo[2], B.hi[2] = 0.0, H
        B.u_mean, B.t_start = u_mean, t_start
    fl = lattice_box((0.0, 0.0, 0.0), (Lx, W, H), dx)
    wl = lattice_box(lo, hi, dx)
    wl = wl[(wl[:, 2] < 0.0) | (wl[:, 2] > H)]
    nf, nw = len(fl), len(wl)
    st = ParticleStore(nf + nw)
    u = splitmix_u01(seed, 0, np.arange(3 * nf, dtype=np.uint64)).reshape(nf, 3)
    pos = fl + (2.0 * u - 1.0) * (jitter * dx)
    for a in range(2):
        pos[:, a] = np.mod(pos[:, a], (Lx, W)[a])
    st.pos[:nf] = pos
    st.pos[nf:] = wl
    st.kind[nf:] = abi.BOUNDARY
    st.material[nf:] = 1
    st.mass[:] = rho * dx ** 3
    st.density[:] = rho
    bodies = empty_bodies(0)
    _finish(st, bodies)
    info = dict(n=nf + nw, n_fluid=nf, n_rigid=0, n_boundary=nw, n_bodies=0, rigid_fraction=0.0, H=H, Lx=Lx)
    return Scenario(name, params, st, bodies, steps, info)


def buffer_velocity_host(params, pos, t):
    """The prescribed velocity of every position inside a buffer zone at time t (NaN outside), with the
    pinned arithmetic of sphg_buffer [P23] (numpy float64, no FMA): a host check for the tests."""
    out = np.full((len(pos), 3), np.nan)
    done = np.zeros(len(pos), bool)
    for b in range(params.n_buffers):
        B = params.buffers[b]
        inside = ~done
        for a in range(3):
            inside &= (pos[:, a] >= B.lo[a]) & (pos[:, a] < B.hi[a])
        u = np.zeros(int(inside.sum()))
        if t > B.t_start:
            f = np.ones_like(u)
            if B.profile_axis >= 0:
                a = B.profile_axis
                xi = (pos[inside, a] - B.lo[a]) / (B.hi[a] - B.lo[a])
                f = (6.0 * xi) * (1.0 - xi)
            u = B.u_mean * f
        v = np.zeros((len(u), 3))
        v[:, B.axis] = u
        out[inside] = v
        done |= inside
    return out


def config4(**kw):
    """BASELINE configs[3] (C4): powder bed under a moving Gaussian heat flux (powder_bed)."""
    return powder_bed(**kw)


def config3(**kw):
    """BASELINE configs[2]: 128^3 two-phase liquid/gas with 200 rigid cubes and spheres."""
    return two_phase_with_bodies(**kw)


def config2(**kw):
    """BASELINE configs[1]: 64^3 + walls, 27 spheres, bottom wall 1800 K, 500 steps of 5e-6 s."""
    return closed_box_melting(**kw)


def by_name(name, **kw):
    return {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5, "dissolve": dissolving_bodies,
            "paper46": paper_strong_scaling,
            "couette": couette_channel, "channel": buffer_channel}[name](**kw)
