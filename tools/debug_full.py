"""Debug helper: worst dT/dt particle of c2_full_melt after one step (GPU vs oracle)."""
import numpy as np
from paper_2103_07925_b200 import scenarios, Simulation, abi
from oracle.oracle import Oracle
sc = scenarios.config2(melt_forcing=True)
g_, o_ = Simulation(sc.params, device=0), Oracle(sc.params)
for e in (g_, o_):
    e.upload(sc.store, sc.bodies)
    e.initialize()
    e.step(1)
g, _ = g_.download()
o, _ = o_.download()
s = o_.scales()["dT_dt"]
err = np.abs(g.dT_dt - o.dT_dt) / (1e-10 * np.maximum(np.abs(o.dT_dt), s))
off, nbr = o_.get_nlist()
h = sc.params.dx
for i in np.argsort(-err)[:6]:
    js = nbr[off[i]:off[i + 1]]
    d = np.linalg.norm(o.pos[js] - o.pos[i], axis=1) / h
    dT = o.temperature[js] - o.temperature[i]
    act = (d <= 3.0) & (dT != 0.0)
    print(f"i {i} kind {o.kind[i]} mat {o.material[i]} err {err[i]:.3g} dTdt {o.dT_dt[i]:.4e} S {s[i]:.3e} "
          f"T {o.temperature[i]} nb_nonzero_dT {act.sum()} q_of_those {np.sort(d[act])[:5]}")
