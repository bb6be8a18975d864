"""The seeded BASELINE.json configs: sizes, determinism and body bookkeeping."""
import numpy as np

from paper_2103_07925_b200 import abi, scenarios


def test_config1_shape():  # BASELINE configs[0]
    sc = scenarios.config1()
    assert sc.store.n == 32 ** 3
    assert sc.info["n_bodies"] == 4
    assert 4 * 200 < sc.info["n_rigid"] < 4 * 300  # R = 4dx spheres ~257-280 lattice points each
    L = sc.params.hi[0]
    assert np.all((sc.store.pos >= 0) & (sc.store.pos < L))
    fl = sc.store.kind == abi.FLUID
    assert np.all(np.abs(sc.store.vel[fl]) <= 0.01)


def test_config2_shape():  # BASELINE configs[1]
    sc = scenarios.config2()
    assert sc.info["n_fluid"] + sc.info["n_rigid"] == 64 ** 3
    assert sc.info["n_boundary"] == 70 ** 3 - 64 ** 3
    assert sc.info["n_bodies"] == 27
    bottom = sc.store.dirichlet_T == 0
    assert bottom.sum() == 3 * 70 * 70 and np.all(sc.store.temperature[bottom] == 1800.0)


def test_generation_is_deterministic():
    a = scenarios.config1(nside=16, n_spheres=2)
    b = scenarios.config1(nside=16, n_spheres=2)
    for f in ("pos", "vel", "kind", "group", "mass", "body_frame_pos"):
        assert np.array_equal(getattr(a.store, f), getattr(b.store, f))
    assert np.array_equal(a.bodies, b.bodies)


def test_body_frame_positions_are_centred():  # chi_rk mass-weighted mean = 0
    sc = scenarios.config1(nside=24, n_spheres=3, r_range=(3.0, 4.0))
    s = sc.store
    for k in range(sc.info["n_bodies"]):
        m = (s.kind == abi.RIGID) & (s.group == k)
        chi = s.body_frame_pos[m]
        assert np.all(np.abs((s.mass[m, None] * chi).sum(0) / s.mass[m].sum()) < 1e-15)
        assert abs(sc.bodies["mass"][k] - s.mass[m].sum()) <= 1e-15 * s.mass[m].sum()


def test_spheres_do_not_overlap():
    sc = scenarios.config5(nside=60, n_spheres=60)
    assert sc.info["n_bodies"] == 60
    assert 0.05 < sc.info["rigid_fraction"] < 0.3


def test_splitmix_uniform_range():
    u = scenarios.splitmix_u01(123, 0, np.arange(100000, dtype=np.uint64))
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01


def test_paper_strong_scaling_counts():  # 3.79e6 = 3.15e6 fluid + 2.20e5 rigid + 4.21e5 boundary
    sc = scenarios.paper_strong_scaling()
    assert sc.store.n == 3796416
    assert sc.info["n_boundary"] == 156 ** 3 - 150 ** 3
    assert round(sc.info["n_fluid"] / 1e6, 2) == 3.15
    assert round(sc.info["n_rigid"] / 1e5, 1) == 2.2
    assert sc.info["n_bodies"] == 216
    ext = sc.params.hi[0] - sc.params.lo[0]
    assert int(ext // sc.params.cell_edge_override) == 48  # 48^3 cells of edge 0.65


def test_powder_bed_shape():  # BASELINE configs[3]: ~16M particles, ~5000 grains, log-normal radii
    sc = scenarios.config4(nx=80, ny=40, nz=80, n_grains=100)
    assert sc.store.n == 80 * 40 * 86
    assert sc.info["n_bodies"] == 100  # every grain fits under the lid
    r = []
    for k in range(sc.info["n_bodies"]):
        m = sc.store.group[sc.store.kind == 1] == k
        r.append(m.sum())
    assert min(r) > 0
    _, radii = scenarios.deposit_grains(2119, 2000, 1.0, 1.0, 0.0, 1e-3)
    med = np.median(radii / 1e-3)
    assert 3.8 < med < 4.2  # median 4 dx
    assert 0.25 < np.std(np.log(radii)) < 0.32  # sigma 0.3 (clipped tails)
