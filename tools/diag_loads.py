"""Times k_forces_fluid against its loads-only twin (build with -DSPHG_DIAG_LOADS_ONLY, see
kernels_pairs.cu) on a C5 sample: how much of the forces kernel is the gather."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07925_b200 import scenarios, Simulation
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
sc = scenarios.config5(nside=n, n_spheres=int(20000 * (n / 400) ** 3))
sim = Simulation(sc.params)
sim.upload(sc.store, sc.bodies)
sim.initialize()
sim.step(3)
sim.set_timing(True)
a = sim.stats()
sim.step(5)
b = sim.stats()
f = (b.stage_ms[10] - a.stage_ms[10]) / 5
d = (b.stage_ms[12] - a.stage_ms[12]) / 5
v = [(b.stage_ms[k] - a.stage_ms[k]) / 5 for k in (13, 14, 15)]
if os.environ.get("SPHG_DIAG_MODE", "").startswith("G"):
    print(f"nside {n}: forces_fluid {f:.3f} ms; loads-only twin G=4 {d:.3f}, G=2 {v[0]:.3f}, G=8 {v[1]:.3f}, "
          f"G=16 {v[2]:.3f} ms")
else:
    print(f"nside {n}: forces_fluid {f:.3f} ms, loads-only twin (3 SoA records) {d:.3f} ms, "
          f"3 loads from one 128 B AoS record {v[0]:.3f} ms, G0 record only {v[1]:.3f} ms")
