"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py from the oracle built
against the reference's headers).

CPU: the oracle still reproduces every fixture (cells, order and Verlet-list digest exact; fields
to 1e-12 of the DESIGN.md §5 scale, i.e. only libm/compiler noise allowed between hosts).
GPU: the device, through the C ABI, matches the fixtures at the north_star bars without the
oracle or the scenario generator in the loop.
"""
import ctypes as C
import glob
import os
import types

import numpy as np
import pytest

from paper_2103_07925_b200 import abi
from paper_2103_07925_b200.store import ParticleStore, VEC_FIELDS, SCALAR_FIELDS, TAG_FIELDS
from tests.golden.make_golden import OUT_FIELDS, SCALE_KEYS, STEPS, nlist_digest
from tests.helpers import compare_fields

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
NAMES = [os.path.basename(p)[:-4] for p in GOLDEN]


def load(name):
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", f"{name}.npz"))
    raw = d["params"].tobytes()
    # fields appended to sphg_params after a fixture was made (buffer zones, ...) default to zero
    raw = raw + bytes(max(0, C.sizeof(abi.Params) - len(raw)))
    params = abi.Params.from_buffer_copy(raw)
    st = ParticleStore(len(d["in_pos"]))
    for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS):
        setattr(st, f, np.ascontiguousarray(d[f"in_{f}"]))
    return d, params, st, np.ascontiguousarray(d["bodies"])


def expected(d, tag):
    o = types.SimpleNamespace(**{f: d[f"{tag}_{f}"] for f in OUT_FIELDS})
    s = {k: d[f"{tag}_scale_{k}"] for k in SCALE_KEYS}
    return o, d[f"{tag}_bodies"], s


def check_engine(eng, name, tol_init, tol_step):
    d, params, st, bodies = load(name)
    eng = eng(params)
    eng.upload(st, bodies)
    eng.build_pairs()
    cells, order = eng.get_cells()
    assert np.array_equal(cells, d["cells"]), f"{name}: cell ids differ"
    assert np.array_equal(order, d["order"]), f"{name}: (cell, gid) order differs"
    assert nlist_digest(*eng.get_nlist()) == str(d["nlist_sha256"]), f"{name}: Verlet lists differ"
    eng.initialize()
    g, gb = eng.download()
    o, ob, s = expected(d, "init")
    compare_fields(g, gb, o, ob, s, params, tol_init, f"{name} init")
    eng.step(STEPS)
    g, gb = eng.download()
    o, ob, s = expected(d, "step")
    compare_fields(g, gb, o, ob, s, params, tol_step, f"{name} step{STEPS}")
    stt = eng.stats()
    assert [stt.transitions_melt, stt.transitions_solidify, stt.rebuilds, eng.num_bodies()] == d["stats"].tolist()


def test_fixtures_present():
    assert set(NAMES) >= {"c1", "c2m", "c3", "dissolve"}


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(name, oracle_mod):
    check_engine(oracle_mod.Oracle, name, 1e-12, 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_matches_golden(name):
    from paper_2103_07925_b200 import Simulation
    check_engine(lambda p: Simulation(p, device=0), name, 1e-10, 1e-9)
