"""Inflow / outflow buffer zones ("a buffer-zone with prescribed parabolic
velocity and particle recycling") [P23]: the pinned rules on the CPU oracle, their device
twins, and device-vs-oracle parity (-m gpu)."""
import numpy as np
import pytest

from paper_2103_07925_b200 import abi, scenarios
from tests.helpers import compare_state, run_pair


@pytest.fixture(params=["oracle", pytest.param("device", marks=pytest.mark.gpu)])
def make(request):
    if request.param == "oracle":
        from oracle.oracle import Oracle
        return Oracle
    from paper_2103_07925_b200 import Simulation
    return lambda p: Simulation(p, device=0)


def _loaded(make, sc):
    e = make(sc.params)
    e.upload(sc.store, sc.bodies)
    e.initialize()
    return e


def test_buffer_velocity_is_prescribed(make):
    """Every fluid particle inside a zone moves with exactly U(x, t) (held at rest before t_start);
    the parabolic profile averages to u_mean over the zone (PAPER:808 'mean velocity')."""
    sc = scenarios.buffer_channel(u_mean=2.0, t_start=2.5e-5)
    e = _loaded(make, sc)
    for k in range(1, 5):
        e.step(1)
        s, _ = e.download()
        t = e.stats().time
        U = scenarios.buffer_velocity_host(sc.params, s.pos, t)
        inz = ~np.isnan(U[:, 0]) & (s.kind == abi.FLUID)
        assert inz.sum() == 2 * 4 * 10 * 16  # two 4 dx zones of the 10 x 16 cross-section
        assert np.array_equal(s.vel[inz], U[inz])  # bit-exact: the pinned arithmetic of [P23]
        if t <= 2.5e-5:
            assert np.all(s.vel[inz] == 0.0)
        else:
            assert abs(U[inz, 0].mean() / 2.0 - 1.0) < 0.01
            assert np.all(U[inz, 1:] == 0.0)


def test_buffer_recycling_drives_the_channel(make):
    """Particles leave the inflow zone as fluid, enter the outflow zone as buffer particles and wrap
    into the inflow zone again: particle count and mass exact, the interior flow follows the buffers."""
    sc = scenarios.buffer_channel(u_mean=2.0)
    e = _loaded(make, sc)
    e.step(200)
    s, _ = e.download()
    assert s.n == sc.store.n and s.mass.sum() == sc.store.mass.sum()
    x0, x1 = sc.store.pos[:, 0], s.pos[:, 0]
    left_inflow = (x0 < 4e-3) & (x1 >= 4e-3) & (x1 < sc.info["Lx"] - 4e-3)
    assert left_inflow.sum() > 100
    mid = (s.kind == abi.FLUID) & (x1 > 0.012) & (x1 < 0.020)
    assert s.vel[mid, 0].mean() > 0.5 * 2.0


def test_buffer_zone_validation():
    from paper_2103_07925_b200.sim import Simulation
    from oracle.oracle import Oracle
    sc = scenarios.buffer_channel()
    sc.params.buffers[0].profile_axis = 0  # profile along the flow axis
    for cls in (Simulation, Oracle):
        msg = cls.validate(sc.params) if cls is Oracle else cls.validate(sc.params, None)
        assert "buffer zone axes invalid" in msg


@pytest.mark.gpu
def test_buffer_parity():
    """Device vs oracle: step 1 at 1e-10 (zones active from t = 0), then 20 steps with particles
    crossing zone faces: the same zone membership, buffer velocities to round-off of the positions
    they are evaluated at, fields at the multistep bar."""
    from paper_2103_07925_b200 import Simulation
    from oracle.oracle import Oracle
    sc = scenarios.buffer_channel(u_mean=2.0)
    sim, orc = run_pair(sc, lambda p: Simulation(p, device=0), Oracle)
    sim.step(1)
    orc.step(1)
    compare_state(sim, orc, sc.params, what="buffer step1")
    sim.step(20)
    orc.step(20)
    g, _ = sim.download()
    o, _ = orc.download()
    U = scenarios.buffer_velocity_host(sc.params, o.pos, orc.stats().time)
    inz = ~np.isnan(U[:, 0])
    assert np.array_equal(np.isnan(scenarios.buffer_velocity_host(sc.params, g.pos, sim.stats().time)[:, 0]), ~inz)
    assert np.abs(g.vel[inz] - o.vel[inz]).max() <= 1e-12 * 2.0
    compare_state(sim, orc, sc.params, tol=1e-7, what="buffer 21 steps")
