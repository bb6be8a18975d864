#!/usr/bin/env python
"""bench.py — particle-steps/s of the full fp64 SPH step (BASELINE.json metric).

Workload at N=1: BASELINE configs[4] (C5), 400^3 = 64M particles, periodic, ~20k
rigid spheres R~U[3,6]dx, config-1 physics (fluid + rigid + contact, TVF, no
thermal), synthetic seeded inputs (no dataset exists for this path).

A "step" is one full kick-drift-kick step over the whole store:
half kick + drift + body integration, Verlet check (rebuild when triggered),
density, wall/rigid extrapolation, forces (fluid + coupling + contact), body
reduction, final kick.  Timed with CUDA events on the library's stream.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

--impl reference times the CPU oracle (oracle/_ref, the reference headers +
the SPEC restatement, OpenMP on all host cores) on the same C5 store (a capped
number of steps: ~25 s per step at 64M); the cpu_baseline leg of the device
arm times a bounded 96^3 sample of it.
"""
import argparse
import glob
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-steps/sec (full SPH step, fp64)"
UNIT = "particle-steps/s"
# compulsory-state bytes per particle for the forces pass:
# R r, u, u~, rho, p, V, m, mat; W a, a_bg
FORCES_BYTES_PER_FLUID = 156.0
FLOPS_PER_PAIR_FORCES = 91.0   # SURVEY §8(d) counting convention
FLOPS_PER_PAIR_DENSITY = 17.0
STEP_BYTES_PER_PARTICLE = 480.0


DEFAULT_NSIDE = {"c5": 400, "c1": 32, "c2": 64, "c3": 128, "c4": 200, "dissolve": 64, "paper46": 150}


def make_scenario(args):
    from paper_2103_07925_b200 import scenarios
    if args.config == "c5":
        return scenarios.config5(nside=args.nside, n_spheres=args.spheres)
    if args.config == "c1":
        return scenarios.config1(nside=args.nside)
    if args.config == "c4":  # 400 x 200 x 200 (with walls) = 16M; --nside scales y and z (x = 2 nside)
        return scenarios.config4(nx=2 * args.nside, ny=args.nside, nz=args.nside - 6,
                                 n_grains=int(round(5000 * (args.nside / 200.0) ** 2)))
    return scenarios.by_name(args.config, nside=args.nside)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # C5: 100 steps (Verlet rebuilds included as they occur)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sph", choices=["sph", "reference"])
    ap.add_argument("--config", default="c5", choices=["c5", "c1", "c2", "c3", "c4", "dissolve", "paper46"],
                    help="c5 = the headline workload (BASELINE metric); the others are secondary measurements "
                         "(paper46 = the paper's own strong-scaling case, PAPER:1011-1014)")
    ap.add_argument("--nside", type=int, default=None, help="lattice side (default: the config's BASELINE size)")
    ap.add_argument("--spheres", type=int, default=20000)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1: strong = the 64M C5 box split over N GPUs; weak = 8M particles per GPU")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-nside", type=int, default=96)
    args = ap.parse_args()
    if args.nside is None:
        args.nside = DEFAULT_NSIDE[args.config]
    return args


def load_peaks():
    peaks = {"hbm_gbs": 6553.3, "source": "BASELINE.md (MEASURED_PEAKS.json absent)"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        peaks["hbm_gbs"] = d.get("hbm_gbs", peaks["hbm_gbs"])
        peaks["source"] = "MEASURED_PEAKS.json"
    fp = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(fp):
        with open(fp) as f:
            d = json.load(f)
            # the kernel is timed inside a multi-step run: the sustained figure (burst when absent)
            peaks["fp64_tflops"] = d.get("fp64_tflops_sustained", d["fp64_tflops"])
    return peaks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 3 + k and r[3 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(nside, spheres_total, nside_total, steps_max=20, budget_s=15.0):
    """The oracle (reference headers + SPEC restatement, OpenMP) on a bounded sample of C5."""
    from paper_2103_07925_b200 import scenarios
    from oracle.oracle import Oracle
    ns = max(1, int(round(spheres_total * (nside / nside_total) ** 3)))
    sc = scenarios.config5(nside=nside, n_spheres=ns)
    o = Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    o.step(1)  # warm-up
    t0 = time.perf_counter()
    k = 0
    while k < steps_max:
        o.step(1)
        k += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    host = host_info()
    return {"value": sc.store.n * k / dt, "unit": UNIT, "cores": host["omp_threads"], "kind": "port",
            "sample": f"C5 physics, {nside}^3={sc.store.n} particles periodic, {ns} spheres, {k} steps "
                      f"(oracle: SPEC restatement on the reference headers, OpenMP); the same-config 64M "
                      f"number is the --impl reference arm", "host": host}


def cpu_baseline_scenario(sc, what, steps_max=10, budget_s=20.0):
    """The oracle on the full scenario (bounded step count): the paper46 case is small enough."""
    from oracle.oracle import Oracle
    o = Oracle(sc.params)
    o.upload(sc.store, sc.bodies)
    o.initialize()
    o.step(1)  # warm-up
    t0 = time.perf_counter()
    k = 0
    while k < steps_max:
        o.step(1)
        k += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": sc.store.n * k / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{what}: {sc.store.n} particles, {k} steps (oracle, OpenMP)"}


def host_info():
    """The host the CPU legs ran on (state nproc and the lscpu model)."""
    model, tpc = None, None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() == "Model name":
                model = v.strip()
            elif k.strip() == "Thread(s) per core":
                tpc = int(v.strip())
    except Exception:
        pass
    if model is None and os.path.exists("/proc/cpuinfo"):
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"cpu_model": model, "nproc": os.cpu_count(), "threads_per_core": tpc, "omp_threads": threads}


# The reference arm on the full headline store: at 64M one oracle step takes ~20-30 s on the box's
# 16 host cores, so the arm runs at most this many warm-up / timed steps whatever --warmup/--steps ask
# (the whole arm then ends in a few minutes); the line states both.
REF_MAX_WARMUP = 1
REF_MAX_STEPS = 3


def run_reference(args):
    """--impl reference: the reference's CPU path (the oracle: SPEC restatement compiled on the reference's
    own headers, oracle/_ref, OpenMP over all host cores) on the SAME workload as the device arm (C5
    400^3 = 64M particles, 20,000 spheres, identical seeded store), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.oracle import Oracle
    t_gen = time.perf_counter()
    sc = make_scenario(args)
    t_gen = time.perf_counter() - t_gen
    info, n = sc.info, sc.store.n
    o = Oracle(sc.params)
    t_up = time.perf_counter()
    o.upload(sc.store, sc.bodies)
    sc.store = None  # the oracle holds its own copy: keep the host footprint to one store + the lists
    o.initialize()
    t_up = time.perf_counter() - t_up
    w = min(args.warmup, REF_MAX_WARMUP)
    k = max(1, min(args.steps, REF_MAX_STEPS))
    for _ in range(w):
        o.step(1)
    t0 = time.perf_counter()
    o.step(k)
    dt = time.perf_counter() - t0
    v = n * k / dt
    host = host_info()
    cfg = workload_config(args, info, n)
    cfg["parallelism"] = f"openmp x{host['omp_threads']} (host CPU)"
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": k,
            "warmup": w, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": 1e3 * dt / k, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64 lattice + jitter)",
            "impl": "reference", "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": host["omp_threads"], "kind": "port",
                             "sample": f"the full workload ({n} particles), {k} timed steps after {w} warm-up "
                                       f"(capped at {REF_MAX_STEPS}/{REF_MAX_WARMUP}: ~{1e-3 * dt / k * 1e3:.0f} s per "
                                       f"step); untimed setup: generation {t_gen:.0f} s, upload + Verlet build + "
                                       f"initialize {t_up:.0f} s",
                             "host": host},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def workload_config(args, info, n):
    """The config block both arms print (same keys and values for the same workload)."""
    return {"workload": (f"C5 {args.nside}^3 periodic, {info['n_bodies']} rigid spheres R~U[3,6]dx"
                         if args.config == "c5" else
                         f"{args.config} nside {args.nside}, {info['n_bodies']} bodies, "
                         f"{info.get('n_boundary', 0)} wall particles (secondary measurement)"),
            "particles": n, "fluid": info["n_fluid"], "rigid": info["n_rigid"],
            "rigid_fraction": round(info["rigid_fraction"], 4)}


def store_bytes(store):
    return store.nbytes()


def run_sph(args):
    import torch
    from paper_2103_07925_b200 import scenarios, Simulation, abi
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        from paper_2103_07925_b200 import parallel
        line = parallel.bench_multi(args, clock_factory=ClockSampler)
        if line is not None:  # rank 0 (the process group is gone; the other ranks have finished)
            k0 = line["kernel_per_rank"][0]
            line["roofline"] = make_roofline(k0["forces_fluid_ms"], k0["pairs_fluid_i"], k0["fluid_owned"], None)
            line["roofline"]["scope"] = "rank 0's k_forces_fluid (its owned fluid particles), stage-timed pass"
            if not args.no_cpu_baseline:
                line["cpu_baseline"] = cpu_baseline(args.cpu_nside, args.spheres, args.nside)
            print(json.dumps(line))
        return
    torch.cuda.set_device(local)
    t_gen = time.perf_counter()
    sc = make_scenario(args)
    t_gen = time.perf_counter() - t_gen
    n = sc.store.n
    sim = Simulation(sc.params, device=local)
    sim.upload(sc.store, sc.bodies)
    sim.initialize()
    for _ in range(args.warmup):
        sim.step(1)
    cand, inter, inter_fluid, inter_other = sim.count_pairs()
    # timed region: K full steps, CUDA events recorded on the library's stream around sphg_step
    st0 = sim.stats()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        sim.step(args.steps)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    st1 = sim.stats()
    ms_step = st1.last_step_call_ms / args.steps
    # per-stage breakdown (separate pass; per-stage events on the same stream)
    sim.set_timing(True)
    sa = sim.stats()
    kk = max(2, min(20, args.steps // 2))
    sim.step(kk)
    sb = sim.stats()
    stage_ms = {abi.STAGE_NAMES[k]: (sb.stage_ms[k] - sa.stage_ms[k]) / kk for k in range(12)}
    # one Verlet rebuild (binning + radix sort + reorder + list build + index lists), forced twice
    sim.run_stage(abi.STAGE_REBUILD)
    sc0 = sim.stats()
    sim.run_stage(abi.STAGE_REBUILD)
    sim.run_stage(abi.STAGE_REBUILD)
    sc1 = sim.stats()
    sim.set_timing(False)
    rebuild_ms = (sc1.stage_ms[abi.STAGE_REBUILD] - sc0.stage_ms[abi.STAGE_REBUILD]) / 2
    launches = (st1.kernel_launches - st0.kernel_launches)
    value = n / (ms_step * 1e-3)
    info = sc.info
    nf = info["n_fluid"]
    # dominant kernel: k_forces_fluid (stage 10), average launch duration from CUDA events on
    # the library stream over the breakdown pass; algorithmic flops = 91 per interacting pair
    # with a fluid i; algorithmic bytes = 156 B per fluid particle (CSM model).
    roofline = make_roofline(stage_ms["forces_fluid"], inter_fluid, nf, n)
    fp64 = {"pairs_candidate": cand, "pairs_interacting": inter, "pairs_fluid_i": inter_fluid,
            "pairs_nonfluid_i": inter_other,
            "step_tflops": (FLOPS_PER_PAIR_FORCES * inter_fluid + FLOPS_PER_PAIR_DENSITY * inter_fluid)
                           / (ms_step * 1e-3) / 1e12}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64 lattice + jitter)",
            "config": dict(workload_config(args, info, n), parallelism="1 GPU",
                           fluid_rigid_rate=(nf + info["n_rigid"]) / (ms_step * 1e-3),
                           l2="inputs larger than L2 (state ~%.1f GB)" % (store_bytes(sc.store) / 1e9)),
            "roofline": roofline, "fp64": fp64, "stage_ms": stage_ms, "rebuild_ms": rebuild_ms,
            "step_roofline": {"bytes_per_particle": STEP_BYTES_PER_PARTICLE,
                              "achieved_gbs": STEP_BYTES_PER_PARTICLE * n / (ms_step * 1e-3) / 1e9},
            "wall_s_timed": wall, "gpu_launches": int(launches),
            "rebuilds_in_timed_region": int(st1.rebuilds - st0.rebuilds),
            "clocks": clk.summary(), "gen_s": t_gen,
            "device_memory_gb": round((torch.cuda.mem_get_info(local)[1] - torch.cuda.mem_get_info(local)[0]) / 1e9, 1)}
    return finish_line(args, sim, sc, n, line, rank)


def make_roofline(forces_ms, inter_fluid, nf, n):
    """The dominant kernel, k_forces_fluid_sm (k_forces_fluid on its SM-local persistent grid): average launch duration (CUDA events on the library stream,
    stage-timed pass), algorithmic flops = 91 per interacting pair with a fluid i,
    algorithmic bytes = 156 B per fluid particle (CSM model).  n = store size when the committed ncu
    capture is of the same store (64M), for the measured DRAM traffic and L1 figures."""
    peaks = load_peaks()
    t_ff = forces_ms * 1e-3
    flops = FLOPS_PER_PAIR_FORCES * inter_fluid
    achieved_tf = flops / t_ff / 1e12
    fp64_peak = peaks.get("fp64_tflops")
    hbm_achieved = FORCES_BYTES_PER_FLUID * nf / t_ff / 1e9
    traffic, l1 = None, None
    profs = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_full_64m.json")))
    if profs and n == 64000000:
        tp = profs[-1]
        for k in json.load(open(tp)):
            if "k_forces_fluid" in k["kernel"] and "nan" not in k["dram__bytes_read.sum"]:
                rd = float(k["dram__bytes_read.sum"].split()[0]) * 1e9
                wr = float(k["dram__bytes_write.sum"].split()[0]) * 1e9
                src = os.path.relpath(tp, ROOT) + " (ncu --set full, one launch)"
                traffic = {"bytes_per_launch": rd + wr, "source": src,
                           "note": "Verlet rows (~29 GB) + neighbour records that miss L1 and L2 (SM-local ranges: an "
                                   "SM's records stay in its L1, neighbouring SMs share little in L2); the CSM "
                                   "bytes model is 8.8 GB"}
                wf = k.get("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed")
                fp = k.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
                if wf:
                    hit = k.get("l1tex__t_sector_hit_rate.pct")
                    l1 = {"lsu_wavefronts_pct": float(wf.split()[0]), "fp64_pipe_pct": float(fp.split()[0]) if fp else None,
                          "l1_sector_hit_pct": float(hit.split()[0]) if hit else None,
                          "source": src, "note": "the binding unit: L1 data-pipe wavefronts (one per distinct 32 B "
                                                 "sector of a gather), see DESIGN.md section 4"}
    roofline = {"bound": "fp64", "kernel": "k_forces_fluid_sm (momentum_rhs + TVF; SM-local persistent grid)",
                "achieved": achieved_tf, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": (achieved_tf / fp64_peak) if fp64_peak else None,
                "traffic": traffic, "l1": l1, "launch_ms": forces_ms,
                "flops_per_launch": flops, "flops_model": "91 flop per interacting fluid pair (SURVEY 8(d))",
                "peak_source": "profiles/fp64_peak.json (DFMA microbenchmark tools/fp64_peak.cu, sustained 4 s "
                               "figure, SM clock sampled)",
                "hbm": {"achieved": hbm_achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": hbm_achieved / peaks["hbm_gbs"], "bytes_model": "156 B per fluid particle (CSM)",
                        "peak_source": peaks["source"]}}
    if fp64_peak:
        roofline["frac_nominal"] = achieved_tf / 37.2  # against the datasheet FP64 figure as well
    return roofline


def finish_line(args, sim, sc, n, line, rank):
    import torch
    # e2e: through the public API with host buffers, every step: H2D of the step's kinematic input
    # (positions + velocities from pinned host memory, Simulation.upload_state) -> step(1) ->
    # D2H of the step's fields (positions, velocities, density, pressure) into the ParticleStore
    if not args.no_e2e and args.e2e_steps > 0:
        store = sc.store
        fields = ("pos", "vel", "density", "pressure")
        sim.download(store, fields=fields + ("kind", "material", "owner", "group"))
        pin_pos = torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy()
        pin_vel = torch.empty((n, 3), dtype=torch.float64, pin_memory=True).numpy()
        pin_pos[:] = store.pos
        pin_vel[:] = store.vel
        # the step's results land in pinned host arrays of the store (the download DMAs into them)
        for f, shape in (("pos", (n, 3)), ("vel", (n, 3)), ("density", (n,)), ("pressure", (n,))):
            setattr(store, f, torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy())
        sim.upload_state(pin_pos, pin_vel)  # untimed: first use of the copy stream and staging
        sim.step_download(1, store=store, fields=fields)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            sim.upload_state(pin_pos, pin_vel)
            sim.step_download(1, store=store, fields=fields)  # pos / density / pressure leave during the forces
        e2e_s = time.perf_counter() - t0
        # the requested fields, packed into gid order on the device: pos, vel (24 B), density, pressure (8 B)
        d2h = n * (24 + 24 + 8 + 8)
        line["e2e"] = {"value": n * args.e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(48 * n),
                       "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps,
                       "path": "Simulation.upload_state(pos, vel from pinned host) -> step_download(1: pos, vel, "
                               "density, pressure into pinned host arrays; pos/density/pressure copied while the "
                               "step's force kernels run); host wall clock"}
    if not args.no_cpu_baseline and rank == 0 and args.config == "c5":
        line["cpu_baseline"] = cpu_baseline(args.cpu_nside, args.spheres, args.nside)
    if not args.no_cpu_baseline and rank == 0 and args.config == "paper46":
        line["cpu_baseline"] = cpu_baseline_scenario(make_scenario(args), "the paper's strong-scaling case itself")
    sim.close()
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_sph(args)


if __name__ == "__main__":
    main()
