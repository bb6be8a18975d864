"""Comparison helpers for GPU-vs-oracle parity (DESIGN.md §5 tolerance metric).

A field passes when |x_gpu - x_cpu| <= tol * max(|x_cpu|, S) per particle, where
S is the oracle's sum of |pair contributions| for that particle:
interior accelerations cancel to a small residual, so plain relative error is not
a meaningful bar for them.
"""
import numpy as np

TOL = 1e-10  # BASELINE north_star: fp64 fields within 1e-10 relative
# absolute allowance per unit of the oracle's pressure sensitivity (acc_p / force_p = sum over pairs of
# |d term / d p| c^2 rho): 4 ulp of the EOS magnitude c^2 rho behind each pressure.  p = c^2 (rho - rho0)
# cancels, so two density sums that differ in their last bit (any reordering of the ~107 terms) give
# pressures that differ by ~ulp(c^2 rho) however small p is; where a force hinges on one small pressure
# (a rigid particle whose only fluid pair sits at the cut-off) that input difference, not the force
# arithmetic, sets the error.
EOS_ULPS = 4 * 2.0 ** -52


def vec_err(g, o, scale, tol=TOL, allow=0.0):
    """max over particles of |g-o| / (tol * max(|o|, scale) + allow); <= 1 passes."""
    g = np.asarray(g, float)
    o = np.asarray(o, float)
    if g.ndim == 1:
        d = np.abs(g - o)
        ref = np.maximum(np.abs(o), scale)
    else:
        d = np.linalg.norm(g - o, axis=1)
        ref = np.maximum(np.linalg.norm(o, axis=1), scale)
    den = np.maximum(tol * ref + allow, 1e-300)
    return float(np.max(d / den)) if len(d) else 0.0


def assert_close(name, g, o, scale, tol=TOL, allow=0.0):
    e = vec_err(g, o, scale, tol, allow)
    assert e <= 1.0, f"{name}: max error {e:.3g} x tolerance ({tol:g})"
    return e


def run_pair(sc, lib_sim, oracle_cls, init=True):
    sim = lib_sim(sc.params)
    orc = oracle_cls(sc.params)
    for e in (sim, orc):
        e.upload(sc.store, sc.bodies)
        if init:
            e.initialize()
    return sim, orc


def compare_state(sim, orc, params, tol=TOL, what=""):
    """Compares every hot-path field of the two engines; returns the error table."""
    g, gb = sim.download()
    o, ob = orc.download()
    return compare_fields(g, gb, o, ob, orc.scales(), params, tol, what)


def floored(S):
    """Per-particle pair-sum scales S, floored at one ulp (1e-16) of the field's largest S: a value whose
    every pair term sits at the kernel's cut-off (dW ~ (3-q)^4 ~ 1e-20 of the field) is zero to
    round-off of the field, and its relative digits are the last bits of q."""
    S = np.asarray(S, float)
    return np.maximum(S, 1e-16 * float(np.max(S))) if S.size else S


def compare_fields(g, gb, o, ob, s, params, tol=TOL, what=""):
    """g/o: stores (or anything with the store's field attributes); s: the oracle's scales()."""
    out = {}
    fl = o.kind == 0
    rg = o.kind == 1
    wl = o.kind != 0
    assert np.array_equal(g.kind, o.kind), f"{what}: kind flags differ"
    assert np.array_equal(g.material, o.material), f"{what}: materials differ"
    assert np.array_equal(g.group[rg], o.group[rg]), f"{what}: body ids differ"
    rho0 = np.array([params.mat[m].rho0 for m in range(params.n_mat)])
    c2 = np.array([params.mat[m].c ** 2 for m in range(params.n_mat)])
    out["density"] = assert_close(f"{what} density", g.density[fl], o.density[fl], 0.0, tol)
    out["pressure"] = assert_close(f"{what} pressure", g.pressure[fl], o.pressure[fl],
                                   (c2[o.material] * o.density)[fl], tol)
    acc_p = s["acc_p"][fl] if "acc_p" in s else 0.0
    force_p = s["force_p"][rg] if "force_p" in s else 0.0
    out["acc"] = assert_close(f"{what} acc", g.acc[fl], o.acc[fl], floored(s["acc"][fl]), tol, EOS_ULPS * acc_p)
    out["acc_bg"] = assert_close(f"{what} acc_bg", g.acc_bg[fl], o.acc_bg[fl], floored(s["acc_bg"][fl]), tol)
    # wall/rigid pressures are Shepard averages of fluid pressures: their scale is the
    # fluid pressure scale c^2 rho0 of the fluid materials (a solid's own c is 0)
    p0_fluid = max(float(rho0[m] * c2[m]) for m in range(params.n_mat))
    out["wall_pressure"] = assert_close(f"{what} wall_pressure", g.wall_pressure[wl], o.wall_pressure[wl],
                                        p0_fluid, tol)
    uscale = max(float(np.max(np.abs(o.vel))), 1e-12)
    # u~_w = 2 u_w - Shepard average of fluid velocities: integrated velocities, so the velocity bar
    out["wall_velocity"] = assert_close(f"{what} wall_velocity", g.wall_velocity[wl], o.wall_velocity[wl], uscale,
                                        max(tol, 1e-9))
    out["force"] = assert_close(f"{what} force", g.force[rg], o.force[rg], floored(s["force"][rg]), tol,
                                EOS_ULPS * force_p)
    out["dT_dt"] = assert_close(f"{what} dT_dt", g.dT_dt, o.dT_dt, floored(s["dT_dt"]), tol)
    out["temperature"] = assert_close(f"{what} T", g.temperature, o.temperature, 0.0, tol)
    if params.diffusion:
        out["dC_dt"] = assert_close(f"{what} dC_dt", g.dC_dt, o.dC_dt, floored(s["dC_dt"]), tol)
        out["concentration"] = assert_close(f"{what} C", g.concentration, o.concentration, 1.0, tol)
        assert np.array_equal(g.dirichlet_C, o.dirichlet_C), f"{what}: concentration groups differ"
    L = np.array([params.hi[a] - params.lo[a] for a in range(3)])
    out["pos"] = assert_close(f"{what} pos", g.pos, o.pos, float(np.max(L)), 1e-14)
    out["vel"] = assert_close(f"{what} vel", g.vel, o.vel, uscale, 1e-9)
    if len(ob):
        assert np.array_equal(gb["alive"], ob["alive"]), f"{what}: alive bodies differ"
        al = ob["alive"] == 1
        out["body_mass"] = assert_close(f"{what} body mass", gb["mass"][al], ob["mass"][al], 0.0, 1e-12)
        out["body_force"] = assert_close(f"{what} body force", gb["force"][al], ob["force"][al],
                                         s["body_force"][al], tol)
        out["body_torque"] = assert_close(f"{what} body torque", gb["torque"][al], ob["torque"][al],
                                          s["body_torque"][al], tol)
        out["body_inertia"] = assert_close(f"{what} body inertia", gb["inertia"][al], ob["inertia"][al],
                                           np.abs(ob["inertia"][al][:, :3]).max(axis=1), 1e-12)
    return out
