"""Debug helper: the worst rigid-force particle of paper46_small at initialize (GPU vs oracle)."""
import numpy as np
from paper_2103_07925_b200 import scenarios, Simulation, abi
from oracle.oracle import Oracle
import sys
full = "--full" in sys.argv
sc = scenarios.paper_strong_scaling() if full else scenarios.paper_strong_scaling(nside=30, n_grid=2)
g_, o_ = Simulation(sc.params, device=0), Oracle(sc.params)
for e in (g_, o_):
    e.upload(sc.store, sc.bodies)
    e.initialize()
    if "--step" in sys.argv:
        e.step(1)
g, gb = g_.download()
o, ob = o_.download()
s = o_.scales()
rg = np.nonzero(o.kind == abi.RIGID)[0]
from tests.helpers import floored
err = np.linalg.norm(g.force[rg] - o.force[rg], axis=1) / (1e-10 * np.maximum(np.linalg.norm(o.force[rg], axis=1), floored(s["force"][rg])))
order = np.argsort(-err)[:5]
off, nbr = o_.get_nlist()
h = sc.params.dx
for k in order:
    i = rg[k]
    js = nbr[off[i]:off[i + 1]]
    fl = js[o.kind[js] == abi.FLUID]
    d = np.linalg.norm(o.pos[fl] - o.pos[i], axis=1) / h
    inr = fl[d <= 3.0]
    print(f"   min(3-q) {np.min(3.0 - d[d <= 3.0]) if len(inr) else -1:.3e} max q-dist {np.max(3.0 - d[d <= 3.0]) if len(inr) else -1:.3e}")
    print(f"gid {i} err {err[k]:.3g} |f|={np.linalg.norm(o.force[i]):.3e} S={s['force'][i]:.3e} "
          f"fluid nb in rc={len(inr)} min(3-q)={np.min(3.0 - d[d <= 3.0]) if len(inr) else -1:.3e} "
          f"q={np.sort(d[d<=3.0])[:6]}")
    print("   f gpu", g.force[i], "orc", o.force[i])
    print("   wall p gpu/orc", g.wall_pressure[i], o.wall_pressure[i], " wall v", g.wall_velocity[i], o.wall_velocity[i])
    dd = np.abs(g.pressure[inr] - o.pressure[inr]).max() if len(inr) else 0
    print("   max |dp| of its fluid nbrs", dd, "max |drho|", np.abs(g.density[inr] - o.density[inr]).max() if len(inr) else 0)
