import sys, numpy as np
sys.path.insert(0, '.')
from paper_2103_07925_b200 import scenarios, Simulation
from oracle.oracle import Oracle
sc = scenarios.config1(nside=20, n_spheres=3, r_range=(3.0, 4.0), seed=11)
sim, orc = Simulation(sc.params), Oracle(sc.params)
for e in (sim, orc):
    e.upload(sc.store, sc.bodies); e.build_pairs(); e.density_summation()
g, _ = sim.download(); o, _ = orc.download()
fl = o.kind == 0
print('density max rel', np.max(np.abs(g.density[fl] - o.density[fl]) / o.density[fl]))
print('pressure max abs', np.max(np.abs(g.pressure[fl] - o.pressure[fl])))
for e in (sim, orc):
    e.extrapolate_wall_quantities()
g, _ = sim.download(); o, _ = orc.download()
wl = o.kind != 0
err = np.abs(g.wall_pressure - o.wall_pressure)
k = np.argmax(np.where(wl, err, 0))
print('worst wall', k, 'gpu', g.wall_pressure[k], 'orc', o.wall_pressure[k], 'err', err[k])
off, nb = orc.get_nlist()
nbrs = nb[off[k]:off[k+1]]
d = o.pos[nbrs] - o.pos[k]
L = 0.02
d = np.where(d > L/2, d - L, np.where(d < -L/2, d + L, d))
r = np.sqrt((d**2).sum(1)) / 1e-3
fn = nbrs[(o.kind[nbrs] == 0) & (r <= 3.0)]
print('fluid nbrs within rc', len(fn), 'q', np.sort(r[(o.kind[nbrs] == 0) & (r <= 3.0)])[:10])
print('their p gpu-orc', g.pressure[fn] - o.pressure[fn])
