"""Diagnostic: the worst rigid-force mismatches of the C5 200^3 init (device vs oracle), with the
per-particle ingredients (wall pressure, density, fluid pairs, q range)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2103_07925_b200 import scenarios, Simulation, abi
from oracle.oracle import Oracle
from tests.helpers import floored

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 200
sc = scenarios.config5(nside=ns, n_spheres=int(round(20000 * (ns / 400) ** 3)))
sim = Simulation(sc.params, device=0); orc = Oracle(sc.params)
for e in (sim, orc):
    e.upload(sc.store, sc.bodies); e.initialize()
g, gb = sim.download(); o, ob = orc.download(); s = orc.scales()
rg = np.nonzero(o.kind == abi.RIGID)[0]
S = floored(s["force"][rg])
d = np.linalg.norm(g.force[rg] - o.force[rg], axis=1)
ref = np.maximum(np.linalg.norm(o.force[rg], axis=1), S)
r = d / (1e-10 * ref)
print("rigid", len(rg), "max err/tol", r.max(), "n over", (r > 1).sum(), "n over 0.5", (r > 0.5).sum())
L = sc.params.hi[0] - sc.params.lo[0]
h = sc.params.h
off, nbr = orc.get_nlist()
for k in np.argsort(-r)[:8]:
    i = rg[k]
    js = nbr[off[i]:off[i + 1]]
    dd = o.pos[i] - o.pos[js]; dd -= L * np.round(dd / L)
    q = np.sqrt((dd ** 2).sum(1)) / h
    fl = (o.kind[js] == 0) & (q < 3)
    rr = (o.kind[js] != 0) & (q < 3)
    print(f"gid {i} err/tol {r[k]:.3g} |f| {np.linalg.norm(o.force[i]):.3e} S {S[k]:.3e} "
          f"pw g/o {g.wall_pressure[i]:.17g} {o.wall_pressure[i]:.17g} rel {abs(g.wall_pressure[i]-o.wall_pressure[i])/max(abs(o.wall_pressure[i]),1e-300):.2e} "
          f"nfluid {fl.sum()} qmin {q[fl].min() if fl.any() else -1:.4f} qmax {q[fl].max() if fl.any() else -1:.6f} nrigid {rr.sum()}")
    print("   f g", g.force[i], "\n   f o", o.force[i])
