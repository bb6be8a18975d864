"""Long-run stability on the headline store: C5 64M for 5 x 100 steps on one B200 — ms/step per block
(CUDA events on the library stream), Verlet rebuilds, total mass (exact) and linear momentum of fluid +
bodies against the start (relative to sum m |u|), the largest speed, dt-limit warnings.
usage: python tools/long_run.py [blocks] [steps_per_block] [nside]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2103_07925_b200 import scenarios, Simulation  # noqa: E402

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 5
per = int(sys.argv[2]) if len(sys.argv) > 2 else 100
nside = int(sys.argv[3]) if len(sys.argv) > 3 else 400
sc = scenarios.config5(nside=nside, n_spheres=int(round(20000 * (nside / 400.0) ** 3)))
sim = Simulation(sc.params)
sim.upload(sc.store, sc.bodies)
sim.initialize()


def totals():
    st, b = sim.download(fields=("vel", "mass", "kind"))
    fl = st.kind == 0
    pf = (st.mass[fl, None] * st.vel[fl]).sum(0)
    al = b["alive"] == 1
    pb = (b["mass"][al, None] * b["vel"][al]).sum(0)
    scale = (st.mass[fl] * np.linalg.norm(st.vel[fl], axis=1)).sum() + (b["mass"][al] * np.linalg.norm(b["vel"][al], axis=1)).sum()
    mass = st.mass.sum()
    return pf + pb, scale, mass, float(np.abs(st.vel).max())


p0, s0, m0, _ = totals()
rows = []
for k in range(blocks):
    a = sim.stats()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.step(per)
    e1.record()
    e1.synchronize()
    b = sim.stats()
    rows.append({"block": k, "ms_per_step": b.last_step_call_ms / per, "rebuilds": b.rebuilds - a.rebuilds,
                 "dt_warnings": b.dt_violations - a.dt_violations})
p1, s1, m1, umax = totals()
print(json.dumps({"particles": sc.store.n, "steps": blocks * per, "blocks": rows,
                  "momentum_drift_rel": float(np.linalg.norm(p1 - p0) / max(s0, 1e-300)),
                  "mass_exact": bool(m1 == m0), "max_speed": umax}))
