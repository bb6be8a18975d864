"""Diagnostic: device vs oracle on the buffer channel, step by step (first step whose density differs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2103_07925_b200 import scenarios, Simulation, abi
from oracle.oracle import Oracle
sc = scenarios.buffer_channel(u_mean=2.0)
for mode in sys.argv[1:] or ["single", "multi"]:
    sim = Simulation(sc.params, device=0); orc = Oracle(sc.params)
    for e in (sim, orc):
        e.upload(sc.store, sc.bodies); e.initialize()
    for k in range(1, 22):
        if mode == "single":
            sim.step(1); orc.step(1)
        else:
            if k > 1: break
            sim.step(21); orc.step(21)
        g, _ = sim.download(); o, _ = orc.download()
        fl = o.kind == 0
        dr = np.abs(g.density[fl] - o.density[fl]).max() / 1000
        dp = np.abs(g.pos - o.pos).max()
        dv = np.abs(g.vel - o.vel).max()
        i = np.argmax(np.abs(g.vel - o.vel).max(1))
        j = np.argmax(np.abs(g.density - o.density) * fl)
        if dr > 1e-6:
            print("   density worst gid", j, "x", o.pos[j], "rho g/o", g.density[j], o.density[j], "kind", o.kind[j],
                  "vel g/o", g.vel[j], o.vel[j], flush=True)
        print(mode, k, "rho %.2e pos %.2e vel %.2e" % (dr, dp, dv), "worst gid", i, "x", o.pos[i], "vg", g.vel[i], "vo", o.vel[i],
              "rebuilds", sim.stats().rebuilds, orc.stats().rebuilds, flush=True)
