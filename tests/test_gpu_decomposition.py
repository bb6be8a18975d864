"""The GPU engine under the decomposition layer: 2 ranks as 2 processes sharing one
B200 over gloo (host-staged halo buffers; no kernel waits on another rank), compared
with the single-rank GPU run and with the oracle.  Exercises the device halo
pack/unpack kernels, ghost-aware stages and body partials."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests.test_decomposition import _free_port, _case, NSTEPS

pytestmark = pytest.mark.gpu


def _gpu_worker(rank, world, port, case, out, nsteps=None):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_07925_b200 import Simulation
    from paper_2103_07925_b200.parallel import DistributedSimulation
    sc = _case(case)
    ds = DistributedSimulation(sc.params, lambda p: Simulation(p, device=0), tensor_device="cpu",
                               engine_device="cuda:0", margin_h=0.3)
    ds.event_log = True
    ds.distribute(sc.store, sc.bodies)
    ds.initialize()
    k = NSTEPS[case] if nsteps is None else nsteps
    ds.step(1)
    c0 = ds.engine.counters()
    r0 = ds.rebuilds
    ds.step(k - 1)
    c1 = ds.engine.counters()
    g, b = ds.gather()
    if rank == 0:
        np.savez(out, pos=g.pos, acc=g.acc, density=g.density, force=g.force, T=g.temperature,
                 bforce=b["force"], btorque=b["torque"], binertia=b["inertia"], rebuilds=ds.rebuilds,
                 repart=ds.repartitions, syncs=c1[2] - c0[2], steps=k - 1,
                 rebuilds_late=ds.rebuilds - r0, kind=g.kind, group=g.group, material=g.material,
                 bmass=b["mass"], balive=b["alive"], batches=ds.batches,
                 events=np.array([tuple(e) for e in ds.events], np.int64).reshape(-1, 5))
    dist.destroy_process_group()


def test_gpu_two_ranks_one_step_parity(tmp_path):
    """One decomposed step (2 ranks, in-library exchanges over gloo) against one single-rank step on the
    same device: every per-step field at the 1e-10 bar of DESIGN.md §5 (the sums run over the same
    neighbour sets in another order, ghosts in place of owned copies)."""
    from paper_2103_07925_b200 import Simulation, abi
    from oracle.oracle import Oracle
    from tests.helpers import vec_err, EOS_ULPS
    out = str(tmp_path / "g1.npz")
    mp.spawn(_gpu_worker, args=(2, _free_port(), "c1", out, 1), nprocs=2, join=True)
    d = np.load(out)
    sc = _case("c1")
    sim = Simulation(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    sim.step(1)
    g, b = sim.download()
    o = Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    o.step(1)
    s = o.scales()
    fl, rg = g.kind == abi.FLUID, g.kind == abi.RIGID
    assert vec_err(d["pos"], g.pos, float(sc.params.hi[0] - sc.params.lo[0]), 1e-14) <= 1
    assert vec_err(d["density"][fl], g.density[fl], 0.0) <= 1
    assert vec_err(d["acc"][fl], g.acc[fl], s["acc"][fl], allow=EOS_ULPS * s["acc_p"][fl]) <= 1
    assert vec_err(d["force"][rg], g.force[rg], s["force"][rg], allow=EOS_ULPS * s["force_p"][rg]) <= 1
    al = b["alive"] == 1
    assert vec_err(d["bforce"][al], b["force"][al], s["body_force"][al]) <= 1
    assert vec_err(d["btorque"][al], b["torque"][al], s["body_torque"][al]) <= 1


@pytest.mark.parametrize("case", ["c1fast", "c2", "c1wrap"])
def test_gpu_two_ranks_match_single_rank(case, tmp_path):
    from paper_2103_07925_b200 import Simulation, abi
    from oracle.oracle import Oracle
    from tests.helpers import vec_err
    out = str(tmp_path / "gds.npz")
    mp.spawn(_gpu_worker, args=(2, _free_port(), case, out), nprocs=2, join=True)
    d = np.load(out)
    sc = _case(case)
    sim = Simulation(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    sim.step(NSTEPS[case])
    g, b = sim.download()
    o = Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    o.step(NSTEPS[case])
    s = o.scales()
    fl = g.kind == abi.FLUID
    rg = g.kind == abi.RIGID
    if case == "c1fast":
        assert d["rebuilds"] >= 2 and d["repart"] >= 1
    if case == "c2":  # slow flow, no rebuild after step 1: one flag readback per decomposed step + one per call
        assert int(d["rebuilds_late"]) == 0 and int(d["syncs"]) <= int(d["steps"]) + 1, (d["syncs"], d["steps"])
    assert vec_err(d["pos"], g.pos, float(sc.params.hi[0] - sc.params.lo[0]), 1e-14) <= 1
    assert vec_err(d["density"][fl], g.density[fl], 0.0, 1e-10) <= 1
    assert vec_err(d["acc"][fl], g.acc[fl], s["acc"][fl], 1e-8) <= 1
    assert vec_err(d["force"][rg], g.force[rg], s["force"][rg], 1e-8) <= 1
    al = b["alive"] == 1
    assert vec_err(d["bforce"][al], b["force"][al], s["body_force"][al], 1e-8) <= 1


@pytest.mark.parametrize("case", ["c2melt", "dissolve"])
def test_gpu_two_ranks_transitions(case, tmp_path):
    """SPEC:500 on the device engine: 2 decomposed GPU ranks (transition batch applied at rank 0 in a
    scratch single-rank context, records broadcast) against the single-rank GPU run: flags, materials, body
    ids, liveness, body masses and the event log bit-exact; fields at the multistep bar."""
    from paper_2103_07925_b200 import Simulation, abi
    from oracle.oracle import Oracle
    from tests.helpers import vec_err
    out = str(tmp_path / "gt.npz")
    mp.spawn(_gpu_worker, args=(2, _free_port(), case, out), nprocs=2, join=True)
    d = np.load(out)
    sc = _case(case)
    sim = Simulation(sc.params)
    sim.set_event_log(True)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    sim.step(NSTEPS[case])
    g, b = sim.download()
    ev = sim.transition_events()
    assert len(ev) > 0 and int(d["batches"]) >= 1
    assert np.array_equal(d["events"], np.array([tuple(e) for e in ev.tolist()], np.int64).reshape(-1, 5))
    assert np.array_equal(d["kind"], g.kind) and np.array_equal(d["material"], g.material)
    rg = g.kind == abi.RIGID
    assert np.array_equal(d["group"][rg], g.group[rg])
    assert np.array_equal(d["balive"], b["alive"]) and np.array_equal(d["bmass"], b["mass"])
    o = Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    o.step(NSTEPS[case])
    s = o.scales()
    fl = g.kind == abi.FLUID
    assert vec_err(d["density"][fl], g.density[fl], 0.0, 1e-10) <= 1
    assert vec_err(d["acc"][fl], g.acc[fl], s["acc"][fl], 1e-7) <= 1
    assert vec_err(d["T"], g.temperature, 0.0, 1e-12) <= 1


def test_body_partials_device_pointers():
    """sphg_body_partials / sphg_body_apply_totals accept device pointers (the NCCL path of
    DistributedSimulation._bodies) and give the same result as host pointers."""
    import ctypes as C
    import torch
    from paper_2103_07925_b200 import scenarios, Simulation
    sc = scenarios.config1(nside=20, n_spheres=3, r_range=(3.0, 4.0), seed=11)
    dp = C.POINTER(C.c_double)
    out = []
    for dev in ("host", "cuda"):
        sim = Simulation(sc.params, device=0)
        sim.upload(sc.store, sc.bodies)
        sim.initialize()
        nb = sim.num_bodies()
        if dev == "host":
            part = np.zeros((nb, 12, 2))
            sim._check(sim._fn("body_partials")(sim._h, part.ctypes.data_as(dp)), "partials")
            tot = np.ascontiguousarray(part[..., 0] + part[..., 1])
            sim._check(sim._fn("body_apply_totals")(sim._h, tot.ctypes.data_as(dp)), "apply")
        else:
            part = torch.zeros((nb, 12, 2), dtype=torch.float64, device="cuda")
            sim._check(sim._fn("body_partials")(sim._h, C.cast(part.data_ptr(), dp)), "partials")
            tot = (part[..., 0] + part[..., 1]).contiguous()
            torch.cuda.synchronize()
            sim._check(sim._fn("body_apply_totals")(sim._h, C.cast(tot.data_ptr(), dp)), "apply")
            part = part.cpu().numpy()
        _, b = sim.download()
        out.append((part, b))
    assert np.array_equal(out[0][0], out[1][0])
    for f in ("force", "torque", "acc", "alpha"):
        assert np.array_equal(out[0][1][f], out[1][1][f]), f


def test_bench_two_ranks_line(tmp_path):
    """bench.py under torchrun with 2 ranks (gloo, both on this GPU): one JSON line from rank 0 with the
    whole-job value, max-over-ranks timing, the rank-0 roofline object, imbalance and a CPU baseline."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SPHG_DIST_BACKEND="gloo", OMP_NUM_THREADS="4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "4", "--warmup", "3", "--nside", "40", "--spheres", "20", "--e2e-steps", "1",
           "--cpu-nside", "16"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 4 and d["warmup"] == 3
    assert d["roofline"]["bound"] == "fp64" and 0 < d["roofline"]["frac"] < 1
    assert d["config"]["imbalance"] < 0.2 and sum(d["config"]["owned_per_rank"]) == d["config"]["particles"]
    assert d["cpu_baseline"]["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


def test_upload_records_roundtrip_and_validation():
    """sphg_record_pack of a whole store -> sphg_upload_records into a fresh context gives the same state
    (download bit-identical) and the same next step; a record with an invalid body id is refused with code 2
    and leaves the context unchanged."""
    import torch
    from paper_2103_07925_b200 import scenarios, Simulation
    from paper_2103_07925_b200.sim import SPHError
    sc = scenarios.config1(nside=16, n_spheres=2, r_range=(3.0, 3.0), seed=5)
    a = Simulation(sc.params)
    a.upload(sc.store, sc.bodies)
    a.initialize()
    a.step(2)
    a.build_pairs()  # storage order and lists from the current positions, as the reloaded context will build
    ids = torch.arange(a.n, dtype=torch.int32, device="cuda")
    recs = a.record_pack(ids, out=torch.empty((a.n, a.record_doubles()), dtype=torch.float64, device="cuda"))
    _, bodies = a.download()
    b = Simulation(sc.params)
    b.upload(sc.store, sc.bodies)
    torch.cuda.synchronize()
    b.upload_records(recs, a.n, bodies)
    ga, ba = a.download()
    gb, bb = b.download()
    for f in ("pos", "vel", "vel_adv", "density", "pressure", "acc", "acc_bg", "force", "temperature",
              "body_frame_pos", "kind", "group", "material"):
        assert np.array_equal(getattr(ga, f), getattr(gb, f)), f
    assert np.array_equal(ba, bb)
    # one more step: the reloaded context rebuilds its lists after the drift, the original reuses its own
    # (same interacting pairs, possibly another storage order): equal to round-off
    for e in (a, b):
        e.step(1)
    ga, _ = a.download()
    gb, _ = b.download()
    assert np.array_equal(ga.pos, gb.pos)
    assert np.max(np.abs(ga.vel - gb.vel)) <= 1e-12 * np.max(np.abs(ga.vel))
    bad = recs.clone()
    rg = np.nonzero(ga.kind == 1)[0][0]
    bad[rg, 5] = 1e6  # body id out of range
    torch.cuda.synchronize()
    with pytest.raises(SPHError) as ei:
        b.upload_records(bad, a.n, bodies)
    assert ei.value.code == 2 and "invalid" in str(ei.value)
    g2, _ = b.download()
    assert np.array_equal(g2.pos, gb.pos)


def test_record_ids_out_of_range_on_device():
    """Device id lists are checked where they are read: an id >= n fails with code 2, nothing is read out
    of bounds."""
    import torch
    from paper_2103_07925_b200 import scenarios, Simulation
    from paper_2103_07925_b200.sim import SPHError
    sc = scenarios.config1(nside=12, n_spheres=1, r_range=(2.0, 2.0), seed=3)
    sim = Simulation(sc.params)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    ids = torch.tensor([0, 1, sim.n], dtype=torch.int32, device="cuda")
    out = torch.empty((3, sim.record_doubles()), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    with pytest.raises(SPHError) as ei:
        sim.record_pack(ids, out=out)
    assert ei.value.code == 2 and "out of range" in str(ei.value)


def test_cpp_decomposed_host_matches_single_rank():
    """The C++ multi-GPU host (include/sphfsi_gpu/decomposed_simulation.hpp) as 2 and 4 ranks (threads on
    this GPU, LocalTransport) against one DeviceSimulation: fluid + bodies with rebuilds and a migration,
    and melting / solidification through the SPEC:500 batch (tests/cpp/test_decomposed.cpp)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "tests", "cpp", "_build", "test_decomposed")
    assert os.path.exists(exe), "build() compiles tests/cpp (make -C tests/cpp)"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [x for x in r.stdout.splitlines() if x.startswith("ok ")]
    assert len(lines) == 4, r.stdout
    assert any("melting ranks=2" in x for x in lines) and any("fluid+bodies ranks=4" in x for x in lines)


def test_cpp_nccl_transport_single_rank():
    """NcclTransport on a one-rank NCCL communicator (tests/cpp/test_nccl_transport.cpp): the grouped
    send / receive of a halo phase, the MAX all-reduce of the displacement words, the all-gather of the body
    partials and the host byte all-to-all are issued through NCCL on this GPU, stream-ordered, and checked."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "tests", "cpp", "_build", "test_nccl_transport")
    assert os.path.exists(exe), "build() compiles tests/cpp (make -C tests/cpp)"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok nccl transport" in r.stdout, r.stdout + r.stderr


def test_gpu_two_ranks_sm_local_grids(tmp_path, monkeypatch):
    """The decomposed step with the SM-local persistent grids forced on its short lists (SPHG_SM_LOCAL_MIN=0,
    4 lanes per particle): the interior density pass (own stream, own tile counters) overlaps the STATE halo
    and the boundary density pass; rebuilds and a repartition included.  Same checks as the flat grids."""
    monkeypatch.setenv("SPHG_SM_LOCAL_MIN", "0")
    monkeypatch.setenv("SPHG_GROUP_DENSITY", "4")
    monkeypatch.setenv("SPHG_GROUP_FORCES", "4")
    test_gpu_two_ranks_match_single_rank("c1fast", tmp_path)
    test_gpu_two_ranks_match_single_rank("c2", tmp_path)
