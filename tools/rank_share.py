"""Per-rank device time of an N-way decomposed C5 step, measured on one GPU with communication excluded.

Rank 0's owned + ghost set of the N-way cube split (the ghost shell of bench_multi, margin 1h) runs the
library's decomposed step (interior/boundary density split, halo pack/unpack kernels, device body merge)
with an exchange callback that moves nothing: the halos keep their values and MAX / BODIES see this rank
alone, so the physics of the run is not meaningful but every kernel of a rank's step runs on the sizes it
would have.  Strong scaling (64M over N) compares this with the one-GPU step; the NCCL exchange time of a
real N-GPU run comes on top.  usage: python tools/rank_share.py N [steps] [nside] [spheres]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2103_07925_b200 import scenarios, Simulation  # noqa: E402
from paper_2103_07925_b200.parallel import DistributedSimulation, Grid  # noqa: E402
from paper_2103_07925_b200.store import ParticleStore, VEC_FIELDS, SCALAR_FIELDS, TAG_FIELDS  # noqa: E402

N = int(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
nside = int(sys.argv[3]) if len(sys.argv) > 3 else 400
spheres = int(sys.argv[4]) if len(sys.argv) > 4 else 20000
sc = scenarios.config5(nside=nside, n_spheres=spheres)
ds = DistributedSimulation(sc.params, lambda p: Simulation(p, device=0), tensor_device="cuda:0",
                           engine_device="cuda:0", margin_h=1.0)
ds.world = N
ds.params.nranks = N
ds.grid = Grid(sc.params, N)
ds._transfer = lambda phase: None   # no communication: halos keep their values, MAX / BODIES stay local
ds._halo = lambda phase: None
ds._bodies = lambda: None
owner = ds.grid.owner_of(sc.store.pos)
gids, n_own = ds.local_gids(sc.store.pos, owner, 0)
loc = ParticleStore(len(gids))
for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS):
    getattr(loc, f)[:] = getattr(sc.store, f)[gids]
loc.owner[:] = owner[gids].astype(np.uint32)
ds.distribute_local(loc, gids, n_own, sc.store.n, sc.bodies)
del loc
ds.initialize()
ds.step(3)
e = ds.engine
c0 = e.counters()
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
t0 = time.perf_counter()
ds.step(steps)
torch.cuda.synchronize()
ev1.record()
ev1.synchronize()
wall = time.perf_counter() - t0
c1 = e.counters()
ms = ev0.elapsed_time(ev1) / steps
ghosts = len(gids) - n_own
print(json.dumps({"ranks": N, "grid": ds.grid.dims, "particles": sc.store.n, "owned": int(n_own), "ghosts": int(ghosts),
                  "ghost_fraction": ghosts / n_own, "ghost_width_h": ds.width / ds.h, "ms_per_step": ms,
                  "wall_ms_per_step": 1e3 * wall / steps, "rebuilds": c1[1] - c0[1],
                  "host_syncs_per_step": (c1[2] - c0[2]) / steps, "launches_per_step": (c1[3] - c0[3]) / steps,
                  "halo_doubles_per_step": sum((len(s) + len(r)) for _, s, r in ds.peers) * (14 + 4 + 6),
                  "note": "rank 0 of an N-way split on one GPU, exchanges not executed"}))
