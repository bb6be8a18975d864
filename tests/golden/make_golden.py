"""Generates the golden fixtures in tests/golden/*.npz (run in the build container, where the
oracle is compiled against the reference's own headers from /root/reference/proj/include).

    python tests/golden/make_golden.py

Each fixture holds one small seeded case: the exact sphg_params bytes, the input store and body
table, and the oracle's outputs after initialize() and after STEPS steps (all hot-path fields,
the tolerance scales, cell ids, (cell, gid) order and a SHA-256 of the Verlet lists).  The GPU
tests compare the device against these files directly, so the GPU box needs neither the
reference nor the scenario generator to check parity; the CPU tests re-run the oracle and check
it still reproduces them.
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2103_07925_b200 import scenarios  # noqa: E402
from paper_2103_07925_b200.store import VEC_FIELDS, SCALAR_FIELDS, TAG_FIELDS  # noqa: E402

STEPS = 2
OUT_FIELDS = ("pos", "vel", "density", "pressure", "acc", "acc_bg", "force", "temperature", "dT_dt",
              "wall_pressure", "wall_velocity", "kind", "group", "material", "concentration", "dC_dt",
              "dirichlet_C")
SCALE_KEYS = ("acc", "acc_bg", "dT_dt", "force", "density", "body_force", "body_torque", "dC_dt", "acc_p", "force_p")

CASES = {
    "c1": lambda: scenarios.config1(nside=10, n_spheres=2, r_range=(1.5, 2.5), seed=3),
    "c2m": lambda: scenarios.config2(nside=10, n_grid=2, r_range=(1.5, 2.0), seed=5, melt_forcing=True),
    "c3": lambda: scenarios.config3(nside=10, n_bodies=2, r_range=(1.5, 2.0), seed=9),
    "dissolve": lambda: scenarios.dissolving_bodies(nside=10, n_bodies=2, r_range=(1.5, 2.0), seed=21, forcing=True),
    # powder bed under the moving surface heat flux [P21]: exposed grain surfaces melt at step 1
    "c4": lambda: scenarios.config4(nx=12, ny=12, nz=24, n_grains=4, median=2.5, r0_dx=4.0, T0=1699.0, seed=3),
}


def nlist_digest(off, nbr):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(off, np.int64).tobytes())
    h.update(np.ascontiguousarray(nbr, np.uint32).tobytes())
    return h.hexdigest()


def snapshot(eng, tag, d):
    s, b = eng.download()
    for f in OUT_FIELDS:
        d[f"{tag}_{f}"] = getattr(s, f)
    d[f"{tag}_bodies"] = b
    sc = eng.scales()
    for k in SCALE_KEYS:
        d[f"{tag}_scale_{k}"] = sc[k]


def make(name):
    sc = CASES[name]()
    from oracle.oracle import Oracle
    d = {"params": np.frombuffer(bytes(sc.params), np.uint8), "bodies": sc.bodies}
    for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS):
        d[f"in_{f}"] = getattr(sc.store, f)
    o = Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.build_pairs()
    d["cells"], d["order"] = o.get_cells()
    d["nlist_sha256"] = np.array(nlist_digest(*o.get_nlist()))
    o.initialize()
    snapshot(o, "init", d)
    o.step(STEPS)
    snapshot(o, "step", d)
    st = o.stats()
    d["stats"] = np.array([st.transitions_melt, st.transitions_solidify, st.rebuilds, o.num_bodies()], np.int64)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{name}.npz"), **d)
    return d


if __name__ == "__main__":
    for n in CASES:
        d = make(n)
        print(n, len(d["in_pos"]), "particles, stats", d["stats"].tolist())
