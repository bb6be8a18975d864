"""Spatial domain decomposition over ranks (one process per GPU) — the paper's
parallel concept with torch.distributed plumbing.

Ownership and ghosts
  The domain is split into px*py*pz equal boxes (2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2,
  longest axes first).  A rank owns the particles whose position lies in its box
  (`owner`, store.hpp:46) and holds read-only ghost copies of every particle within
  an L-infinity distance w = r_c + 0.1h + margin of the box (periodic images
  included).  The margin keeps Verlet rebuilds rank-local: particles are
  re-partitioned only when the accumulated displacement bound exceeds margin/2.

Per step (bulk-synchronous; the same stage sequence as sphg_step):
  KICK_DRIFT -> allreduce(max displacement) -> halo STATE -> [REBUILD on all ranks]
  -> DENSITY -> halo DENSITY -> [HEAT] -> EXTRAPOLATE -> halo WALL -> FORCES
  -> body partials: all_gather + merge in rank order (compensated, identical on
     every rank; PAPER:303-373 host->owner->host collapsed into a replicated reduce)
  -> FINAL_KICK.
Halo records are packed/unpacked by the engine (device kernels for the GPU
engine, host loops for the oracle) into tensors exchanged with point-to-point
send/recv (NCCL on GPUs, gloo in the CPU tests).

Phase transitions ("Event detection is worker-local; application is
serialized per affected body at the owner, followed by a broadcast of updated
body state and re-linking of affected particles"): each rank detects over the
particles it owns at the end of the step; when any rank has events the engine
returns NEED_TRANSITIONS and `_transition_batch` gathers, at rank 0, every
particle the batch reads (the events and all members of the bodies they can
touch), applies the batch there with the single-rank kernels in a scratch
context, and broadcasts the updated particle records and body table, which every
rank writes into its owned and ghost copies.
"""
import ctypes as C
import math
import os
import time

import numpy as np
import torch
import torch.distributed as dist

from . import abi
from .store import ParticleStore, VEC_FIELDS, SCALAR_FIELDS, TAG_FIELDS, BODY_DTYPE


# SPHG_HALO_P2P=1: halos as per-peer isend / irecv pairs instead of one all_to_all_single per phase
_HALO_P2P = os.environ.get("SPHG_HALO_P2P", "0") not in ("", "0")


def factor_dims(nranks, extent):
    """Rank grid: repeatedly halve the currently longest per-rank extent (powers of 2),
    falling back to a 1D split along the longest axis otherwise."""
    dims = [1, 1, 1]
    n = nranks
    ext = list(extent)
    while n > 1 and n % 2 == 0:
        a = int(np.argmax([ext[k] / dims[k] for k in range(3)]))
        dims[a] *= 2
        n //= 2
    if n > 1:
        a = int(np.argmax(ext))
        dims[a] *= n
    return dims


class Grid:
    def __init__(self, params, nranks):
        self.lo = np.array([params.lo[a] for a in range(3)])
        self.hi = np.array([params.hi[a] for a in range(3)])
        self.L = self.hi - self.lo
        self.periodic = np.array([bool(params.periodic[a]) for a in range(3)])
        self.dims = factor_dims(nranks, self.L)
        self.nranks = nranks

    def coords(self, r):
        return np.array([r // (self.dims[1] * self.dims[2]), (r // self.dims[2]) % self.dims[1], r % self.dims[2]])

    def box(self, r):
        c = self.coords(r)
        w = self.L / np.array(self.dims)
        lo = self.lo + c * w
        hi = self.lo + (c + 1) * w
        return lo, hi

    def owner_of(self, pos):
        w = self.L / np.array(self.dims)
        c = np.floor((pos - self.lo) / w).astype(np.int64)
        for a in range(3):
            c[:, a] = np.clip(c[:, a], 0, self.dims[a] - 1)
        return (c[:, 0] * self.dims[1] + c[:, 1]) * self.dims[2] + c[:, 2]

    def near_box(self, pos, r, width):
        """Particles within L-infinity distance `width` of rank r's box (periodic images)."""
        lo, hi = self.box(r)
        ok = np.ones(len(pos), bool)
        for a in range(3):
            x = pos[:, a]
            inside = (x >= lo[a] - width) & (x <= hi[a] + width)
            if self.periodic[a]:
                inside |= (x + self.L[a] >= lo[a] - width) & (x + self.L[a] <= hi[a] + width)
                inside |= (x - self.L[a] >= lo[a] - width) & (x - self.L[a] <= hi[a] + width)
            ok &= inside
        return ok


def _merge_partials(parts):
    """Merge per-rank (sum, comp) partials in rank order with TwoSum.  Works on numpy arrays
    (host) and torch tensors (device): single IEEE adds/subs, no FMA, so both give the same bits."""
    s = parts[0][..., 0].clone() if torch.is_tensor(parts[0]) else parts[0][..., 0].copy()
    c = parts[0][..., 1].clone() if torch.is_tensor(parts[0]) else parts[0][..., 1].copy()
    for p in parts[1:]:
        s2, c2 = p[..., 0], p[..., 1]
        t = s + s2
        bp = t - s
        e = (s - (t - bp)) + (s2 - bp)
        c = (c + c2) + e
        s = t
    return s + c


class DistributedSimulation:
    """One rank of a decomposed run.  `make_engine(params)` returns a Simulation
    (GPU) or the oracle's engine (CPU tests); `tensor_device` is where halo
    buffers live (the engine's device)."""

    def __init__(self, params, make_engine, tensor_device="cpu", margin_h=2.0, group=None, engine_device=None,
                 fused=True):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.params = params
        self.params.rank = self.rank
        self.params.nranks = self.world
        self.make_engine = make_engine
        self.dev = torch.device(tensor_device)  # where the exchanged tensors live (the backend's device)
        # where the engine packs/unpacks (its own memory: cuda for the GPU engine, cpu for the oracle)
        self.edev = torch.device(engine_device) if engine_device is not None else self.dev
        self.grid = Grid(params, self.world)
        h = params.h if params.h > 0 else params.dx
        self.h = h
        self.rv = 3.0 * h + 0.1 * h
        self.half_skin = 0.05 * h
        self.margin = margin_h * h
        self.width = self.rv + self.margin
        self.engine = None
        self.disp_since_partition = 0.0
        self.repartitions = 0
        self.rebuilds = 0
        self.steps = 0
        self.comm_s = 0.0
        # in-library decomposed step (sphg_set_exchange): the engine runs the whole step on its stream
        # and calls back for the transfers; False = the stage-by-stage driver below
        self.fused = fused
        self.event_log = False
        self.events = []      # transition event log, global gids; filled on rank 0
        self.batches = 0      # decomposed transition batches applied
        self._cb = None
        self._ext = None
        self._xerr = None

    # ------------------------------------------------------------ layout
    def local_gids(self, pos, owner, r):
        """Owned particles of rank r, then its ghosts ordered by (owner rank, gid)."""
        own = np.nonzero(owner == r)[0]
        ghost = np.nonzero((owner != r) & self.grid.near_box(pos, r, self.width))[0]
        ghost = ghost[np.lexsort((ghost, owner[ghost]))]
        return np.concatenate([own, ghost]), len(own)

    def distribute(self, store, bodies):
        """Every rank holds the same global store (seeded generation is deterministic)."""
        owner = self.grid.owner_of(store.pos)
        gids, n_own = self.local_gids(store.pos, owner, self.rank)
        local = ParticleStore(len(gids))
        for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS):
            getattr(local, f)[:] = getattr(store, f)[gids]
        local.owner[:] = owner[gids].astype(np.uint32)
        self.distribute_local(local, gids, n_own, store.n, bodies)

    def distribute_local(self, local, gids, n_own, global_n, bodies):
        """Takes this rank's owned + ghost particles (owner field set, global gids)."""
        self.global_n = global_n
        self.gids = np.asarray(gids)
        self.n_own = n_own
        r = self.rank
        owner = local.owner.astype(np.int64)
        ghost_local = np.arange(n_own, local.n)
        # halo lists: send = my owned particles that are ghosts on q; recv = my ghosts owned by q;
        # both ordered by global gid, so the two sides agree without a handshake
        self.peers = []
        for q in range(self.world):
            if q == r:
                continue
            near = np.nonzero(self.grid.near_box(local.pos[:n_own], q, self.width))[0]
            send_l = near[np.argsort(self.gids[near], kind="stable")]
            recv_l = ghost_local[owner[ghost_local] == q]
            recv_l = recv_l[np.argsort(self.gids[recv_l], kind="stable")]
            if len(send_l) == 0 and len(recv_l) == 0:
                continue
            self.peers.append((q, send_l.astype(np.uint32), recv_l.astype(np.uint32)))
        if self.engine is None:
            self.engine = self.make_engine(self.params)
        self.engine.upload(local, bodies)
        for k, (q, s, rcv) in enumerate(self.peers):
            self._halo_set(2 * k, s)
            self._halo_set(2 * k + 1, rcv)
        self.disp_since_partition = 0.0
        self._bufs = {}
        if self._fused_ok():
            self._bind_fused()

    def _halo_set(self, slot, ids):
        ids = np.ascontiguousarray(ids, np.uint32)
        e = self.engine
        e._check(e._fn("halo_set")(e._h, slot, ids.ctypes.data_as(C.POINTER(C.c_uint32)), len(ids)), "halo_set")

    # ------------------------------------------------- in-library decomposed step
    def _fused_ok(self):
        e = self.engine
        return self.fused and e is not None and getattr(e.lib, e.prefix + "set_exchange", None) is not None

    def _bind_fused(self):
        """Buffers the engine packs into / unpacks from at the exchange points of its decomposed step
        (halo records per peer, the two MAX words, body partials and their all-gather), plus the
        exchange callback.  They live where the engine computes (device for the GPU engine)."""
        e = self.engine
        f = lambda name: getattr(e.lib, e.prefix + name)
        mk = lambda m, dt=torch.float64: torch.zeros(max(int(m), 1), dtype=dt, device=self.edev)
        self._fb = {}
        self._a2a = {}
        for phase in (abi.HALO_STATE, abi.HALO_DENSITY, abi.HALO_WALL):
            d = f("halo_doubles")(phase)
            # one send and one receive tensor per phase, the peers' slots at rank-ordered offsets, so a halo
            # is a single all_to_all_single (NCCL groups the sends / receives) instead of 2 P2P ops per peer
            ins, outs = [0] * self.world, [0] * self.world
            for q, snd, rcv in self.peers:
                ins[q], outs[q] = len(snd) * d, len(rcv) * d
            send, recv = mk(sum(ins)), mk(sum(outs))
            self._a2a[phase] = (send[: sum(ins)], recv[: sum(outs)], ins, outs)
            so, ro = 0, 0
            for k, (q, snd, rcv) in enumerate(self.peers):
                for slot, buf, off, m in ((2 * k, send, so, len(snd) * d), (2 * k + 1, recv, ro, len(rcv) * d)):
                    b = buf[off: off + m]
                    self._fb[(phase, slot)] = b
                    e._check(f("halo_bind")(e._h, phase, slot, C.c_void_p(buf.data_ptr() + 8 * off)), "halo_bind")
                so += len(snd) * d
                ro += len(rcv) * d
        self._maxw = mk(2, torch.int64)
        e._check(f("max_bind")(e._h, C.c_void_p(self._maxw.data_ptr())), "max_bind")
        nb = e.num_bodies()
        self._bpart = mk(nb * 24)
        self._bgath = mk(self.world * nb * 24)
        e._check(f("body_bind")(e._h, C.c_void_p(self._bpart.data_ptr()), C.c_void_p(self._bgath.data_ptr()),
                                self.world), "body_bind")
        self._nb = nb
        if self._cb is None:
            self._cb = abi.EXCHANGE_FN(self._exchange_cb)  # keep the thunk alive with the context
        self._sync_engine_dev()  # the zero-filled buffers before the library writes into them
        e._check(f("set_exchange")(e._h, self._cb, None), "set_exchange")

    def _exchange_cb(self, phase, stream, user):
        try:
            t0 = time.perf_counter()
            if self.edev.type == "cuda":
                # every transfer is enqueued on the engine's stream: the NCCL work waits for the pack
                # kernels and the unpack kernels wait for it, without blocking the host
                if self._ext is None or self._ext_ptr != stream:
                    self._ext = torch.cuda.ExternalStream(stream, device=self.edev)
                    self._ext_ptr = stream
                with torch.cuda.stream(self._ext):
                    self._transfer(phase)
            else:
                self._transfer(phase)
            self.comm_s += time.perf_counter() - t0
            return 0
        except Exception as ex:  # surfaces as the engine's error return
            self._xerr = ex
            return 1

    def _transfer(self, phase):
        staged = self.edev != self.dev  # engine on the GPU, transport (gloo) on the host
        to_t = (lambda t: t.to(self.dev)) if staged else (lambda t: t)  # D2H in stream order (blocking)
        if phase in (abi.HALO_STATE, abi.HALO_DENSITY, abi.HALO_WALL) and not _HALO_P2P:
            send, recv, ins, outs = self._a2a[phase]
            st = to_t(send)
            rt = torch.empty(recv.numel(), dtype=recv.dtype, device=self.dev) if staged else recv
            dist.all_to_all_single(rt, st, output_split_sizes=outs, input_split_sizes=ins, group=self.group)
            if staged:
                recv.copy_(rt)
        elif phase in (abi.HALO_STATE, abi.HALO_DENSITY, abi.HALO_WALL):
            d = getattr(self.engine.lib, self.engine.prefix + "halo_doubles")(phase)
            ops, recv = [], []
            for k, (q, snd, rcv) in enumerate(self.peers):
                if len(snd):
                    ops.append(dist.P2POp(dist.isend, to_t(self._fb[(phase, 2 * k)][: len(snd) * d]), q, group=self.group))
                if len(rcv):
                    rb = self._fb[(phase, 2 * k + 1)][: len(rcv) * d]
                    rt = torch.empty(rb.numel(), dtype=rb.dtype, device=self.dev) if staged else rb
                    ops.append(dist.P2POp(dist.irecv, rt, q, group=self.group))
                    recv.append((rb, rt))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            if staged:
                for rb, rt in recv:
                    rb.copy_(rt)
        elif phase == abi.XCHG_MAX:
            t = to_t(self._maxw)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            if staged:
                self._maxw.copy_(t)
        elif phase == abi.XCHG_BODIES:
            m = self._nb * 24
            part = to_t(self._bpart[:m])
            gath = torch.empty(self.world * m, dtype=torch.float64, device=self.dev) if staged else self._bgath
            if self.dev.type == "cuda":
                dist.all_gather_into_tensor(gath[: self.world * m], part, group=self.group)
            else:
                dist.all_gather([gath[r * m:(r + 1) * m] for r in range(self.world)], part, group=self.group)
            if staged:
                self._bgath[: self.world * m].copy_(gath)
        else:
            raise ValueError(f"unknown exchange phase {phase}")

    def drift(self):
        """(global max displacement since the last rebuild, sum of the displacements at rebuilds since
        the partition, global max fluid speed)."""
        e = self.engine
        out = (C.c_double * 3)()
        e._check(getattr(e.lib, e.prefix + "drift")(e._h, out), "drift")
        return tuple(out)

    # ------------------------------------------------------------ exchanges
    def _halo(self, phase):
        t0 = time.perf_counter()
        e = self.engine
        d = getattr(e.lib, e.prefix + "halo_doubles")(phase)
        ops, recv = [], []
        for k, (q, s, rcv) in enumerate(self.peers):
            key = (phase, k)
            if key not in self._bufs:
                mk = lambda m, dev: torch.empty(max(m, 1) * d, dtype=torch.float64, device=dev)
                staged = self.edev != self.dev
                self._bufs[key] = (mk(len(s), self.edev), mk(len(rcv), self.edev),
                                   mk(len(s), self.dev) if staged else None, mk(len(rcv), self.dev) if staged else None)
            sb, rb, sbx, rbx = self._bufs[key]
            if len(s):
                # halo_pack is synchronous on the engine's stream: the send below sees the packed data
                e._check(e._fn("halo_pack")(e._h, phase, 2 * k, sb.data_ptr()), "halo_pack")
                if sbx is not None:
                    sbx.copy_(sb)
                ops.append(dist.P2POp(dist.isend, (sb if sbx is None else sbx)[: len(s) * d], q, group=self.group))
            if len(rcv):
                ops.append(dist.P2POp(dist.irecv, (rb if rbx is None else rbx)[: len(rcv) * d], q, group=self.group))
                recv.append((k, rb, rbx))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            if self.dev.type == "cuda":
                # NCCL's wait() only orders torch's current stream; the engine unpacks on its own
                # stream, so the host waits for the receives to land first
                torch.cuda.current_stream(self.dev).synchronize()
        for k, rb, rbx in recv:
            if rbx is not None:
                rb.copy_(rbx)
            e._check(e._fn("halo_unpack")(e._h, phase, 2 * k + 1, rb.data_ptr()), "halo_unpack")
        self.comm_s += time.perf_counter() - t0

    def _bodies(self):
        e = self.engine
        nb = e.num_bodies()
        if nb == 0:
            return
        dp = C.POINTER(C.c_double)
        if self.dev.type == "cuda" and self.edev.type == "cuda":
            # device path: partials -> NCCL all_gather -> TwoSum merge in rank order on the GPU -> totals
            mine = torch.empty((nb, 12, 2), dtype=torch.float64, device=self.dev)
            e._check(e._fn("body_partials")(e._h, C.cast(mine.data_ptr(), dp)), "body_partials")
            t0 = time.perf_counter()
            gathered = [torch.empty_like(mine) for _ in range(self.world)]
            dist.all_gather(gathered, mine, group=self.group)
            tot = _merge_partials(gathered).contiguous()
            torch.cuda.current_stream(self.dev).synchronize()  # the engine reads tot on its own stream
            self.comm_s += time.perf_counter() - t0
            e._check(e._fn("body_apply_totals")(e._h, C.cast(tot.data_ptr(), dp)), "body_apply_totals")
            return
        part = np.zeros((nb, 12, 2))
        e._check(e._fn("body_partials")(e._h, part.ctypes.data_as(dp)), "body_partials")
        t0 = time.perf_counter()
        mine = torch.from_numpy(part).to(self.dev)
        gathered = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(gathered, mine, group=self.group)
        parts = [g.cpu().numpy() for g in gathered]
        self.comm_s += time.perf_counter() - t0
        tot = np.ascontiguousarray(_merge_partials(parts))
        e._check(e._fn("body_apply_totals")(e._h, tot.ctypes.data_as(dp)), "body_apply_totals")

    def _allmax(self, x):
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    # ------------------------------------------------------------ stepping
    def _evaluate(self, thermal):
        e = self.engine
        e.run_stage(abi.STAGE_DENSITY)
        self._halo(abi.HALO_DENSITY)
        if thermal:
            e.run_stage(abi.STAGE_HEAT)
        e.run_stage(abi.STAGE_EXTRAPOLATE)
        self._halo(abi.HALO_WALL)
        e.run_stage(abi.STAGE_FORCES)
        self._bodies()

    def initialize(self):
        self.engine.run_stage(abi.STAGE_REBUILD)
        self._evaluate(thermal=False)

    def step(self, nsteps=1):
        e = self.engine
        if self._fused_ok():
            # the engine runs kick .. final kick with its own exchanges, nsteps at a time; it stops with
            # NEED_PARTITION before a step the partition may not cover (a particle may drift up to
            # margin/2 before its ghosts could miss a neighbour), the host migrates and steps on
            f = lambda name: getattr(e.lib, e.prefix + name)
            e._check(f("set_partition_limit")(e._h, 0.5 * self.margin), "set_partition_limit")
            s0, r0 = e.counters()[:2]
            done = 0
            while done < nsteps:
                rc = f("step")(e._h, nsteps - done)
                s1 = e.counters()[0]
                done += s1 - s0
                s0 = s1
                if rc == abi.NEED_PARTITION:
                    self.repartition()
                    continue
                if rc == abi.NEED_TRANSITIONS:  # the step completed; its transition batch is applied here
                    self._transition_batch()
                    continue
                if rc != 0:
                    if self._xerr is not None:
                        raise RuntimeError(f"exchange failed: {self._xerr!r}") from self._xerr
                    e._check(rc, "step")
            self.steps += nsteps
            r1 = e.counters()[1]
            self.rebuilds += r1 - r0
            return
        if self.params.transitions:
            raise RuntimeError("phase transitions under decomposition need the in-library decomposed step "
                               "(fused=True)")
        thermal = bool(self.params.thermal) or bool(self.params.diffusion)  # one stage for T and C
        for _ in range(nsteps):
            e.run_stage(abi.STAGE_KICK_DRIFT)
            d = C.c_double(0.0)
            e._check(e._fn("max_displacement")(e._h, C.byref(d)), "max_displacement")
            disp = self._allmax(d.value)
            self._halo(abi.HALO_STATE)
            if disp > self.half_skin:  # SPEC:212, all ranks together
                self.disp_since_partition += disp
                if self.disp_since_partition > 0.5 * self.margin:
                    self.repartition()
                e.run_stage(abi.STAGE_REBUILD)
                self.rebuilds += 1
            self._evaluate(thermal)
            e.run_stage(abi.STAGE_FINAL_KICK)
            self.steps += 1

    def imbalance(self):
        """SPEC:222 (static blocks; imbalance is only reported): owned particles per rank and
        max / mean - 1."""
        t = torch.tensor([float(self.n_own)], dtype=torch.float64, device=self.dev)
        allc = [torch.zeros_like(t) for _ in range(self.world)]
        if self.world > 1:
            dist.all_gather(allc, t, group=self.group)
        else:
            allc = [t]
        counts = [int(x.item()) for x in allc]
        mean = sum(counts) / len(counts)
        return counts, (max(counts) / mean - 1.0) if mean > 0 else 0.0

    # ------------------------------------------------------------ transitions
    def _single_rank_params(self):
        p = type(self.params)()
        C.memmove(C.byref(p), C.byref(self.params), C.sizeof(p))
        p.rank, p.nranks = 0, 1
        return p

    def _apply_batch(self, gids, recs, bodies):
        """Rank 0: the batch on a scratch single-rank context holding exactly the gathered particles
        (global gid order, so every gid-ordered rule — spawn ids, attach ties, split ids — and every
        body-major sum runs as in the single-rank run).  Returns (records, bodies, events)."""
        m = len(gids)
        st = ParticleStore(m)
        st.pos[:] = recs[:, 0:3]
        st.kind[:] = recs[:, 3].astype(np.uint8)
        st.material[:] = recs[:, 4].astype(np.uint16)
        st.group[:] = recs[:, 5].astype(np.uint32)
        st.mass[:] = recs[:, 6]
        st.density[:] = [self.params.mat[int(k)].rho0 for k in st.material]
        eng = self.make_engine(self._single_rank_params())
        try:
            if self.event_log:
                eng.set_event_log(True)
            eng.upload(st, bodies)
            ids = np.arange(m, dtype=np.uint32)
            eng.record_unpack(ids, recs, keep_position=False)
            eng.run_stage(abi.STAGE_TRANSITIONS)
            out = eng.record_pack(ids)
            _, nbodies = eng.download(ParticleStore(m), fields=())
            ev = eng.transition_events() if self.event_log else None
        finally:
            eng.close()
        if ev is not None and len(ev):
            ev["gid"] = gids[ev["gid"]].astype(ev["gid"].dtype)  # scratch ids -> global gids
            ev["step"] = self.engine.counters()[0]
        return out, nbodies, ev

    def _transition_batch(self):
        """apply the transition batch the last decomposed step detected (see the module doc)."""
        e = self.engine
        nb = e.num_bodies()
        _, bodies = e.download(ParticleStore(e.n), fields=())
        mask = e.event_bodies(np.zeros(nb, np.uint8))
        t = torch.from_numpy(mask.astype(np.int32)).to(self.dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        mask = t.cpu().numpy().astype(np.uint8)
        ids = e.event_members(mask)
        mine = (self.gids[ids].astype(np.int64), e.record_pack(ids))
        allp = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(allp, mine, group=self.group)
        else:
            allp = [mine]
        if self.rank == 0:
            gids = np.concatenate([a[0] for a in allp])
            recs = np.concatenate([a[1] for a in allp])
            order = np.argsort(gids, kind="stable")
            gids, recs = gids[order], recs[order]
            out, nbodies, ev = self._apply_batch(gids, recs, bodies)
            res = [(gids, out, nbodies)]
            if ev is not None:
                self.events.extend(ev.tolist())
        else:
            res = [None]
        if self.world > 1:
            dist.broadcast_object_list(res, src=0, group=self.group)
        gids, out, nbodies = res[0]
        # every listed particle present here, owned or ghost: local ids through the sorted gid map
        order = np.argsort(self.gids, kind="stable")
        pos = np.searchsorted(self.gids[order], gids)
        pos = np.minimum(pos, len(order) - 1)
        here = self.gids[order][pos] == gids
        local = order[pos[here]].astype(np.uint32)
        e.record_unpack(local, out[here], keep_position=True)
        e.replace_bodies(nbodies)
        if len(nbodies) != self._nb and self._fused_ok():
            self._bind_fused()  # body buffers are sized by the body count
        self._bodies()  # reduce_force_torque of the new membership (the single-rank batch ends with it)
        self.batches += 1

    # ------------------------------------------------------------ global views
    def gather(self):
        """Owned particles of every rank -> global store (gid order) and the replicated bodies."""
        local, bodies = self.engine.download()
        own = slice(0, self.n_own)
        payload = {f: getattr(local, f)[own] for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS)}
        payload["gid"] = self.gids[: self.n_own]
        allp = [None] * self.world
        dist.all_gather_object(allp, payload, group=self.group)
        g = ParticleStore(self.global_n)
        for p in allp:
            for f in VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS):
                getattr(g, f)[p["gid"]] = p[f]
        return g, bodies

    # ------------------------------------------------------------ migration (device-resident)
    def _owner_t(self, pos):
        """Grid.owner_of on a (m, 3) float64 tensor (the same IEEE operations as the numpy form)."""
        g = self.grid
        dev = pos.device
        lo = torch.tensor(g.lo, dtype=torch.float64, device=dev)
        w = torch.tensor(g.L / np.array(g.dims), dtype=torch.float64, device=dev)
        dims = torch.tensor(g.dims, dtype=torch.int64, device=dev)
        c = torch.floor((pos - lo) / w).to(torch.int64)
        c = torch.minimum(torch.clamp(c, min=0), dims - 1)
        return (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]

    def _near_box_t(self, pos, r, width):
        """Grid.near_box on a tensor: within L-infinity distance `width` of rank r's box (periodic images)."""
        g = self.grid
        lo, hi = g.box(r)
        ok = torch.ones(pos.shape[0], dtype=torch.bool, device=pos.device)
        for a in range(3):
            x = pos[:, a]
            inside = (x >= lo[a] - width) & (x <= hi[a] + width)
            if g.periodic[a]:
                inside |= (x + g.L[a] >= lo[a] - width) & (x + g.L[a] <= hi[a] + width)
                inside |= (x - g.L[a] >= lo[a] - width) & (x - g.L[a] <= hi[a] + width)
            ok &= inside
        return ok

    def _exchange_t(self, outgoing, width):
        """outgoing[q] = (m, width) float64 tensor for rank q -> {q: tensor received from q} (on the
        engine's device): counts first, then the payload, point to point (NCCL on the device; gloo
        through host copies)."""
        peers = [q for q in range(self.world) if q != self.rank]
        cnt_out = {q: torch.tensor([int(outgoing[q].shape[0]) if q in outgoing else 0], dtype=torch.int64,
                                   device=self.dev) for q in peers}
        cnt_in = {q: torch.zeros(1, dtype=torch.int64, device=self.dev) for q in peers}
        ops = []
        for q in peers:
            ops.append(dist.P2POp(dist.isend, cnt_out[q], q, group=self.group))
            ops.append(dist.P2POp(dist.irecv, cnt_in[q], q, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        ops, recv = [], {}
        for q in peers:
            m_out, m_in = int(cnt_out[q].item()), int(cnt_in[q].item())
            if m_out:
                ops.append(dist.P2POp(dist.isend, outgoing[q].contiguous().to(self.dev), q, group=self.group))
            if m_in:
                recv[q] = torch.empty((m_in, width), dtype=torch.float64, device=self.dev)
                ops.append(dist.P2POp(dist.irecv, recv[q], q, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if self.dev.type == "cuda":
            torch.cuda.current_stream(self.dev).synchronize()
        return {q: t.to(self.edev) for q, t in recv.items()}

    def _sync_engine_dev(self):
        """Device tensors made on torch's stream are read on the library's own stream: finish them first."""
        if self.edev.type == "cuda":
            torch.cuda.current_stream(self.edev).synchronize()

    def repartition(self):
        """Particle migration, device-resident: each rank packs its owned particles as
        engine records (sphg_record_pack into a device tensor), sends the ones that left its box to their
        new owner, then ships every peer the owned particles inside that peer's ghost shell, and reloads
        its owned + ghost set from the records (sphg_upload_records): no rank holds more than its own
        owned + ghost set and nothing crosses to the host but counts.  Rare: after margin/2 of motion."""
        e = self.engine
        R = e.record_doubles()
        n_own = self.n_own
        ids = torch.arange(n_own, dtype=torch.int32, device=self.edev)
        out = torch.empty((n_own, R), dtype=torch.float64, device=self.edev)
        self._sync_engine_dev()
        recs = e.record_pack(ids, out=out)  # complete on return (the library syncs its stream)
        gid = torch.from_numpy(self.gids[:n_own].astype(np.float64)).to(self.edev)  # exact below 2^53
        full = torch.cat([gid[:, None], recs], dim=1)
        new_owner = self._owner_t(full[:, 1:4])
        outgoing = {q: full[new_owner == q] for q in range(self.world) if q != self.rank}
        got = self._exchange_t(outgoing, R + 1)
        owned = torch.cat([full[new_owner == self.rank]] + [got[q] for q in sorted(got)])
        owned = owned[torch.argsort(owned[:, 0], stable=True)]
        shells = {q: owned[self._near_box_t(owned[:, 1:4], q, self.width)]
                  for q in range(self.world) if q != self.rank}
        got = self._exchange_t(shells, R + 1)
        ghosts, gowner = [], []
        for q in sorted(got):  # (owner rank, gid) order, as local_gids
            t = got[q][torch.argsort(got[q][:, 0], stable=True)]
            ghosts.append(t)
            gowner.append(np.full(t.shape[0], q, np.int64))
        allrec = torch.cat([owned] + ghosts) if ghosts else owned
        _, bodies = e.download(ParticleStore(e.n), fields=())
        self.repartitions += 1
        self._install(allrec, int(owned.shape[0]), np.concatenate(gowner) if gowner else np.zeros(0, np.int64),
                      bodies)

    def _install(self, allrec, n_own, ghost_owner, bodies):
        """Load an owned + ghost set given as [gid | record] rows (owned by gid, then ghosts by (owner,
        gid)) into the engine and derive the per-peer halo lists, all from device tensors."""
        e = self.engine
        self.gids = allrec[:, 0].to(torch.int64).cpu().numpy()
        self.n_own = n_own
        recs = allrec[:, 1:].contiguous()
        self._sync_engine_dev()
        e.upload_records(recs, n_own, bodies)
        pos_own = allrec[:n_own, 1:4]
        self.peers = []
        for q in range(self.world):
            if q == self.rank:
                continue
            send_l = torch.nonzero(self._near_box_t(pos_own, q, self.width)).flatten().cpu().numpy()  # gid order
            recv_l = n_own + np.nonzero(ghost_owner == q)[0]  # one block, gid order
            if len(send_l) == 0 and len(recv_l) == 0:
                continue
            self.peers.append((q, send_l.astype(np.uint32), recv_l.astype(np.uint32)))
        for k, (q, snd, rcv) in enumerate(self.peers):
            self._halo_set(2 * k, snd)
            self._halo_set(2 * k + 1, rcv)
        self.disp_since_partition = 0.0
        self._bufs = {}
        if self._fused_ok():
            self._bind_fused()


# ---------------------------------------------------------------- bench N>1
def bench_multi(args, clock_factory=None):
    """Strong scaling on the C5 config: rank 0 generates the seeded global store and
    ships each rank its box + ghost shell; K steps; value = all particles x K / max rank time.
    Returns rank 0's JSON line (dict), None on the other ranks."""
    import json
    from . import scenarios
    from .sim import Simulation
    local = int(os.environ.get("LOCAL_RANK", "0"))
    gpu = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(gpu)
    # NCCL over NVLink on a real multi-GPU node; SPHG_DIST_BACKEND=gloo runs the same code with
    # host-staged buffers (used to smoke-test this path with several ranks sharing one GPU)
    backend = os.environ.get("SPHG_DIST_BACKEND", "nccl")
    # communicator evidence (ranks, transports, NVLS) in the log; INIT only, so the one JSON line stays
    # easy to find
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
    else:
        dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    comm = torch.device("cuda", gpu) if backend == "nccl" else torch.device("cpu")
    # rank 0 generates the seeded global store once and sends every rank only its
    # owned + ghost subset (host memory stays O(N) overall instead of O(N x ranks))
    dev = comm
    if rank == 0:
        if getattr(args, "scaling", "strong") == "weak":
            # BASELINE C5 weak scaling: 8M particles (200^3) per GPU, sphere density of C5
            nside = int(round(200 * world ** (1.0 / 3.0)))
            nsph = int(round(args.spheres * (nside / 400.0) ** 3))
            sc = scenarios.config5(nside=nside, n_spheres=nsph)
        else:
            sc = scenarios.config5(nside=args.nside, n_spheres=args.spheres)
        meta = [sc.params, sc.bodies, sc.info, sc.store.n]
    else:
        meta = [None, None, None, None]
    dist.broadcast_object_list(meta, src=0)
    params, bodies, info, n_total = meta
    # ghost margin 1h (shell r_c + skin + 1h = 4.1h): particles may drift h/2 before a migration, ~170 steps
    # of C5 flow; the default 2h costs ~30 % more ghosts at 8 ranks
    ds = DistributedSimulation(params, lambda p: Simulation(p, device=gpu), tensor_device=str(comm),
                               engine_device=f"cuda:{gpu}", margin_h=getattr(args, "margin_h", 1.0))
    fields = VEC_FIELDS + SCALAR_FIELDS + tuple(TAG_FIELDS)
    if rank == 0:
        owner = ds.grid.owner_of(sc.store.pos)
        for r in range(world - 1, -1, -1):
            gids, n_own = ds.local_gids(sc.store.pos, owner, r)
            if r == 0:
                my = (gids, n_own)
                continue
            hdr = torch.tensor([len(gids), n_own], dtype=torch.int64, device=dev)
            dist.send(hdr, r)
            dist.send(torch.from_numpy(gids.astype(np.int64)).to(dev), r)
            for f in fields:  # raw bytes: every dtype travels as uint8
                a = np.ascontiguousarray(getattr(sc.store, f)[gids])
                dist.send(torch.from_numpy(a.reshape(-1).view(np.uint8)).to(dev), r)
            dist.send(torch.from_numpy(owner[gids].astype(np.int64)).to(dev), r)
        gids, n_own = my
        loc = ParticleStore(len(gids))
        for f in fields:
            getattr(loc, f)[:] = getattr(sc.store, f)[gids]
        loc.owner[:] = owner[gids].astype(np.uint32)
        del sc
    else:
        hdr = torch.empty(2, dtype=torch.int64, device=dev)
        dist.recv(hdr, 0)
        m, n_own = int(hdr[0]), int(hdr[1])
        g = torch.empty(m, dtype=torch.int64, device=dev)
        dist.recv(g, 0)
        gids = g.cpu().numpy()
        loc = ParticleStore(m)
        for f in fields:
            a = getattr(loc, f)
            t = torch.empty(a.nbytes, dtype=torch.uint8, device=dev)
            dist.recv(t, 0)
            a.reshape(-1).view(np.uint8)[:] = t.cpu().numpy()
        t = torch.empty(m, dtype=torch.int64, device=dev)
        dist.recv(t, 0)
        loc.owner[:] = t.cpu().numpy().astype(np.uint32)
    ds.distribute_local(loc, gids, n_own, n_total, bodies)
    del loc
    ds.initialize()
    ds.step(args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    st0 = ds.engine.stats()
    import contextlib
    clk = clock_factory(gpu) if clock_factory is not None else contextlib.nullcontext()
    # device clock: CUDA events on this rank's current stream bracket the K steps (each decomposed
    # step ends host-synchronised, so the end event fires when the last kernel / exchange is done)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clk:
        ev0.record()
        ds.step(args.steps)
        torch.cuda.synchronize()
        ev1.record()
        ev1.synchronize()
        dt = ev0.elapsed_time(ev1) * 1e-3
    launches = ds.engine.stats().kernel_launches - st0.kernel_launches
    dist.barrier()
    tmax = torch.tensor([dt], dtype=torch.float64, device=dev)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dt = float(tmax.item())
    tl = torch.tensor([float(launches)], dtype=torch.float64, device=dev)
    dist.all_reduce(tl, op=dist.ReduceOp.SUM)
    # e2e through the public API on every rank: pinned host positions / velocities of the rank's
    # particles -> upload_state -> one decomposed step -> download of pos, vel, density, pressure
    e2e = None
    if not getattr(args, "no_e2e", False) and getattr(args, "e2e_steps", 0) > 0:
        eng = ds.engine
        m = eng.n
        loc, _ = eng.download(fields=("pos", "vel"))
        pin = {f: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
               for f, shape in (("pos", (m, 3)), ("vel", (m, 3)), ("density", (m,)), ("pressure", (m,)))}
        pin["pos"][:] = loc.pos
        pin["vel"][:] = loc.vel
        out = ParticleStore(0)
        out.n = m
        for f in VEC_FIELDS + SCALAR_FIELDS:
            setattr(out, f, pin.get(f, np.zeros((m, 3) if f in VEC_FIELDS else m)))
        for f, dt_ in TAG_FIELDS.items():
            setattr(out, f, np.zeros(m, dt_))
        torch.cuda.synchronize()
        dist.barrier()
        t1 = time.perf_counter()
        for _ in range(args.e2e_steps):
            eng.upload_state(pin["pos"], pin["vel"])
            ds.step(1)
            eng.download(out, fields=("pos", "vel", "density", "pressure"))
        te = time.perf_counter() - t1
        te_t = torch.tensor([te], dtype=torch.float64, device=dev)
        dist.all_reduce(te_t, op=dist.ReduceOp.MAX)
        hb = torch.tensor([48.0 * m, 64.0 * m], dtype=torch.float64, device=dev)
        dist.all_reduce(hb, op=dist.ReduceOp.SUM)
        e2e = {"value": n_total * args.e2e_steps / float(te_t.item()), "unit": "particle-steps/s",
               "h2d_bytes_per_step": int(hb[0].item()), "d2h_bytes_per_step": int(hb[1].item()),
               "steps": args.e2e_steps,
               "path": "per rank: upload_state(pos, vel of owned + ghost particles from pinned host) -> "
                       "DistributedSimulation.step(1) -> download(pos, vel, density, pressure into pinned host); "
                       "host wall clock, max over ranks"}
    counts, imb = ds.imbalance()
    # dominant kernel on this rank: a stage-timed pass (CUDA events per stage, after the timed region)
    eng = ds.engine
    kk = max(2, min(10, args.steps // 2))
    eng.set_timing(True)
    sa = eng.stats()
    ds.step(kk)
    sb = eng.stats()
    eng.set_timing(False)
    _, _, inter_fluid, _ = eng.count_pairs()
    loc, _ = eng.download(ParticleStore(eng.n), fields=("kind", "owner"))
    nf_own = int(((loc.kind == abi.FLUID) & (loc.owner == rank)).sum())
    kern = {"forces_fluid_ms": (sb.stage_ms[10] - sa.stage_ms[10]) / kk, "pairs_fluid_i": int(inter_fluid),
            "fluid_owned": nf_own, "rank": rank}
    kern_all = [None] * world
    dist.all_gather_object(kern_all, kern)
    n = n_total
    if rank == 0:
        weak = getattr(args, "scaling", "strong") == "weak"
        line = {"metric": "particle-steps/sec (full SPH step, fp64)", "value": n * args.steps / dt,
                "unit": "particle-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
                "scaling": "weak" if weak else "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64 lattice + jitter)",
                "config": {"workload": f"C5 {round(n ** (1 / 3))}^3 periodic, {info['n_bodies']} spheres"
                                       + (" (8M per GPU)" if weak else ""),
                           "particles": n, "parallelism": f"domain decomposition {ds.grid.dims}, {backend} halo",
                           "ghost_width_h": ds.width / ds.h, "owned_per_rank": counts,
                           "imbalance": imb},
                "timing": "CUDA events on each rank's stream between barriers + cuda synchronize, "
                          "max over ranks (the per-rank step mixes kernels and NCCL exchanges)",
                "comm_s_rank0": ds.comm_s, "rebuilds": ds.rebuilds, "repartitions": ds.repartitions,
                "gpu_launches": int(tl.item()), "e2e": e2e,
                "kernel_per_rank": kern_all}  # bench.py turns rank 0's entry into the roofline object
        if clock_factory is not None:
            line["clocks"] = clk.summary()
    dist.destroy_process_group()
    return line if rank == 0 else None
