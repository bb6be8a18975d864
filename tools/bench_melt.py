"""Transition-heavy runs: C4 (16M, powder bed) with the bed at T0 = T_t - 0.3 K so the spot melts grains from
the first steps, and C2 melt-forcing (flags flip at step 1); ms/step, the transition counts and a stage-timed
pass (ms per step per stage, transitions included).  usage: python tools/bench_melt.py [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2103_07925_b200 import abi, scenarios, Simulation  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for name, mk in (("c4_melt", lambda: scenarios.config4(T0=1699.7)),
                 ("c2_melt", lambda: scenarios.config2(melt_forcing=True))):
    sc = mk()
    sim = Simulation(sc.params, device=0)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    sim.step(3)
    s0 = sim.stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.step(steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    s1 = sim.stats()
    sim.set_timing(True)
    sa = sim.stats()
    k = max(2, steps // 2)
    sim.step(k)
    sb = sim.stats()
    stage = {abi.STAGE_NAMES[i]: round((sb.stage_ms[i] - sa.stage_ms[i]) / k, 3) for i in range(12)
             if sb.stage_ms[i] != sa.stage_ms[i]}
    print(json.dumps({"case": name, "n": sc.store.n, "ms_per_step": 1e3 * dt / steps,
                      "melt": s1.transitions_melt - s0.transitions_melt,
                      "solidify": s1.transitions_solidify - s0.transitions_solidify,
                      "bodies": sim.num_bodies(), "rebuilds": s1.rebuilds - s0.rebuilds, "stage_ms": stage,
                      "repart_all": os.environ.get("SPHG_REPART_ALL", "0")}))
    sim.close()
