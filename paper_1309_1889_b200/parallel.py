"""Parareal with its fine slices sharded over GPUs.

One process per GPU (torchrun), `torch.distributed` for the plumbing: NCCL
between B200s, gloo in the CPU tests.  This is the reference's parareal_run
(src/parareal.cpp:182-239) with the Executor's parallel_for over fine slices
(src/parareal.cpp:146-151) spread over ranks:

* parareal_init (src/parareal.cpp:94-115) and every corrected coarse sweep
  (src/parareal.cpp:155-173) run redundantly on every rank.  The coarse
  propagator is deterministic, so every rank holds bit-identical rows and no
  state has to be sent for them.
* The fine propagations of one iteration (the `work` list, after the
  metastable-skip heuristic, src/parareal.cpp:117-145) go round-robin to ranks:
  work[i] runs on rank i % world.  Each resulting delta F(lambda_{n-1}) - g_n
  (state_sub, src/parareal.cpp:58-73) and its rms_pos are broadcast from the
  owner -- the "broadcast of slice boundary states" of the north star.
* Convergence bookkeeping (src/parareal.cpp:200-234) is identical on every rank.

Results do not depend on the number of ranks: a 1-rank run equals the
single-GPU C++ driver (msmb_parareal_run) bit for bit, and an N-rank run equals
the 1-rank run bit for bit (deltas are broadcast exactly; coarse rows are
recomputed identically).

The device work goes through a backend.  `DeviceBackend` is the product: msmb
fields, device-resident propagation (msmb_system_propagate_ex) and the raw
device-state algebra of include/msmb.h, on torch CUDA tensors that NCCL sends
directly.  The CPU tests drive this same module with a host backend built on the
oracle (tests/parallel_host.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import (ConfigError, Error, GpuField, MsmField, NonConvergenceError, ParticleSystem, PararealConfig,
               PararealResult, _ERR, _check, _native, _p)

_CODE = {cls: code for code, cls in _ERR.items()}
_MSG_BYTES = 1024


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def validate(cfg: PararealConfig) -> None:
    """PararealConfig::validate (src/parareal.cpp:43-56), same messages."""
    if cfg.window_points < 1:
        raise ConfigError("window_points must be >= 1")
    if cfg.max_iter < 1:
        raise ConfigError("max_iter must be >= 1")
    if not (cfg.tol > 0.0):
        raise ConfigError("tol must be > 0")
    cfg.fine.validate()
    cfg.coarse.validate()
    cfg.units.validate()
    sf, sg = cfg.fine.slice_span(), cfg.coarse.slice_span()
    if abs(sf - sg) > 1e-12 * max(abs(sf), abs(sg)):
        raise ConfigError("fine and coarse propagators span different slice lengths")
    if cfg.skip_threshold is not None and not (cfg.skip_threshold >= 0.0):
        raise ConfigError("skip threshold must be >= 0")


# ---------------------------------------------------------------------------- backend
class DeviceBackend:
    """States as torch float64 CUDA tensors of shape (6, n) -- x, y, z, vx, vy, vz
    (SoA, the layout of a msmb_system) -- and deltas as flat tensors of 6n + 1
    doubles: the reference's StateDelta (dpos Vec3s, dvel Vec3s) followed by its
    rms_pos.  Every call runs the library's kernels on the field's stream and
    returns after synchronising it."""

    def __init__(self, cfg: PararealConfig, v: ParticleSystem):
        import torch
        self.torch = torch
        F, G = cfg.fine.force_field, cfg.coarse.force_field
        if not isinstance(F, GpuField) or not isinstance(G, GpuField):
            raise ConfigError("the device backend needs GPU fine and coarse propagators")
        self.cfg = cfg
        self.n = v.size()
        self.device = torch.device("cuda", F._device)
        self.lib = _native.lib()
        from . import DeviceSystem
        self.sys = {"fine": DeviceSystem(F, v), "coarse": DeviceSystem(G, v)}
        self.spec = {"fine": cfg.fine, "coarse": cfg.coarse}
        self.units = cfg.units._c()
        self.F = F

    # layout helpers
    def from_system(self, s: ParticleSystem):
        t = self.torch
        host = np.concatenate([s.positions.T, s.velocities.T]).astype(np.float64)
        return t.from_numpy(np.ascontiguousarray(host)).to(self.device)

    def to_host(self, state):
        a = state.cpu().numpy()
        return np.ascontiguousarray(a[:3].T), np.ascontiguousarray(a[3:].T)

    def empty_delta(self):
        return self.torch.empty(6 * self.n + 1, dtype=self.torch.float64, device=self.device)

    def _ready(self):
        # torch-side producers (collectives, allocations) before the library reads
        self.torch.cuda.current_stream(self.device).synchronize()

    @staticmethod
    def _ptr(t):
        return C.c_void_p(t.data_ptr())

    # the reference's operations
    def propagate(self, which: str, state):
        self._ready()
        sysd, sp = self.sys[which], self.spec[which]
        h = sp.force_field.handle
        _check(h, self.lib.msmb_system_set_state_device(sysd._h, self._ptr(state)))
        _check(h, self.lib.msmb_system_propagate_ex(h, sysd._h, sp.dt, sp.steps_per_slice, C.byref(self.units)))
        out = self.torch.empty_like(state)
        _check(h, self.lib.msmb_system_get_state_device(sysd._h, self._ptr(out)))
        return out

    def sub(self, a, b):
        self._ready()
        d = self.empty_delta()
        rms = C.c_double()
        _check(self.F.handle, self.lib.msmb_state_sub_device(self.F.handle, self.n, self._ptr(a), self._ptr(b),
                                                             self._ptr(d), C.byref(rms)))
        d[-1] = rms.value
        return d

    def add(self, base, delta):
        self._ready()
        out = self.torch.empty_like(base)
        _check(self.F.handle, self.lib.msmb_state_add_device(self.F.handle, self.n, self._ptr(base),
                                                             self._ptr(delta), self._ptr(out)))
        return out

    def rms_change(self, a, b) -> float:
        self._ready()
        r = C.c_double()
        _check(self.F.handle, self.lib.msmb_state_rms_change_device(self.F.handle, self.n, self._ptr(a),
                                                                    self._ptr(b), C.byref(r)))
        return r.value

    @staticmethod
    def delta_rms(delta) -> float:
        return float(delta[-1].item())

    def clone(self, state):
        return state.clone()


# ---------------------------------------------------------------------------- driver
@dataclass
class ShardInfo:
    rank: int = 0
    world: int = 1
    fine_slices_run: int = 0       # fine propagations executed by this rank
    bytes_broadcast: int = 0       # delta payload this rank sent


class _Comm:
    def __init__(self, group=None):
        self.dist = _dist()
        self.group = group
        if self.dist is None:
            self.rank, self.world = 0, 1
        else:
            self.rank = self.dist.get_rank(group)
            self.world = self.dist.get_world_size(group)

    def owner(self, idx: int) -> int:
        return idx % self.world

    def bcast(self, t, src: int):
        if self.world > 1:
            g = self.dist.get_global_rank(self.group, src) if self.group is not None else src
            self.dist.broadcast(t, g, group=self.group)

    def first_failure(self, my_slice: int, code: int, msg: str, device):
        """All ranks agree on the failing slice with the lowest index (the one a
        sequential executor meets first) and its error."""
        if self.world == 1:
            return (my_slice, code, msg) if code else None
        import torch
        big = 1 << 62
        st = torch.tensor([my_slice if code else big, code, self.rank], dtype=torch.int64, device=device)
        allst = [torch.zeros_like(st) for _ in range(self.world)]
        self.dist.all_gather(allst, st, group=self.group)
        rows = sorted(tuple(int(v) for v in x.cpu().tolist()) for x in allst)
        sl, cd, who = rows[0]
        if sl == big:
            return None
        buf = torch.zeros(_MSG_BYTES, dtype=torch.uint8, device=device)
        if who == self.rank:
            b = msg.encode()[: _MSG_BYTES - 1]
            buf[: len(b)] = torch.tensor(list(b), dtype=torch.uint8, device=device)
        self.bcast(buf, who)
        text = bytes(buf.cpu().numpy().tolist()).split(b"\0", 1)[0].decode()
        return sl, cd, text


class _Window:
    def __init__(self):
        self.points = 0
        self.rows = 0
        self.lam0 = None
        self.lam_prev = self.lam_prev2 = None
        self.g_prev = self.d_prev = None


def _init(be, v_state, cfg, t, counts) -> _Window:  # parareal_init, src/parareal.cpp:94-115
    w = _Window()
    w.points = t
    w.lam0 = v_state
    row = [v_state] + [None] * t
    for n in range(1, t + 1):
        row[n] = be.propagate("coarse", row[n - 1])
        counts["g_evals"] += 1
    w.lam_prev = row
    w.g_prev = list(row)  # the initialization is its own g-row
    w.d_prev = [None] * (t + 1)
    w.rows = 1
    return w


def _iterate(be, comm: _Comm, w: _Window, cfg, counts, info: ShardInfo):  # src/parareal.cpp:129-180
    t = w.points
    prev = w.rows - 1
    skip = [False] * (t + 1)
    if cfg.skip_threshold is not None and w.rows >= 2:  # metastable_skip_indices :117-127
        for n in range(1, t + 1):
            if be.rms_change(w.lam_prev[n - 1], w.lam_prev2[n - 1]) < cfg.skip_threshold:
                skip[n] = True
    deltas = [None] * (t + 1)
    for n in range(1, t + 1):
        if skip[n]:
            deltas[n] = w.d_prev[n]
            counts["f_skipped"] += 1
    work = [n for n in range(1, t + 1) if not skip[n]]
    # fine sweep: work[i] on rank i % world
    fail_slice, fail_code, fail_msg = 0, 0, ""
    for idx, n in enumerate(work):
        if comm.owner(idx) != comm.rank:
            deltas[n] = be.empty_delta()
            continue
        try:
            f = be.propagate("fine", w.lam_prev[n - 1])
            deltas[n] = be.sub(f, w.g_prev[n])
            info.fine_slices_run += 1
        except Error as e:
            fail_slice, fail_code, fail_msg = n, _CODE.get(type(e), 9), str(e)
            deltas[n] = be.empty_delta()
            break
    bad = comm.first_failure(fail_slice, fail_code, fail_msg, getattr(be, "device", None))
    if bad is not None:
        _, code, msg = bad
        raise _ERR.get(code, Error)(msg)
    for idx, n in enumerate(work):
        src = comm.owner(idx)
        if src == comm.rank and comm.world > 1:
            info.bytes_broadcast += deltas[n].numel() * deltas[n].element_size()
        comm.bcast(deltas[n], src)
    counts["f_evals"] += len(work)
    # corrected coarse sweep (redundant on every rank)
    row = [w.lam0] + [None] * t
    grow = [None] * (t + 1)
    for n in range(1, t + 1):
        if prev == 0 and n == 1:
            g = w.g_prev[1]
        else:
            g = be.propagate("coarse", row[n - 1])
            counts["g_evals"] += 1
        row[n] = be.add(g, deltas[n])
        grow[n] = g
    w.lam_prev2, w.lam_prev = w.lam_prev, row
    w.g_prev, w.d_prev = grow, deltas
    w.rows += 1


@dataclass
class ShardedPararealResult(PararealResult):
    report_rows: list = None          # (window, point, iteration, delta_rms, converged)
    point_iterations: list = None
    shard: Optional[ShardInfo] = None


def parareal_run(v: ParticleSystem, total_points: int, cfg: PararealConfig, group=None,
                 backend=None) -> ShardedPararealResult:
    """paramd::parareal_run (src/parareal.cpp:182-239) with the fine slices of every
    iteration sharded over the ranks of `group` (default: the whole job, or a
    single process when torch.distributed is not initialised)."""
    validate(cfg)
    if total_points < 1:
        raise ConfigError("total_points must be >= 1")
    be = backend if backend is not None else DeviceBackend(cfg, v)
    comm = _Comm(group)
    info = ShardInfo(comm.rank, comm.world)
    counts = dict(g_evals=0, f_evals=0, f_skipped=0)
    rows, point_iters, traj = [], [], []
    current = be.from_system(v)
    remaining, window_idx = total_points, 0
    while remaining > 0:
        window_idx += 1
        t = min(cfg.window_points, remaining)
        w = _init(be, current, cfg, t, counts)
        prefix = 0
        for k in range(cfg.max_iter):
            _iterate(be, comm, w, cfg, counts, info)
            prefix, unbroken = 0, True
            for n in range(1, t + 1):
                change = be.rms_change(w.lam_prev[n], w.lam_prev2[n])
                ok = change <= cfg.tol
                rows.append((window_idx, n, k, be.delta_rms(w.d_prev[n]), ok))
                if unbroken and ok:
                    prefix = n
                else:
                    unbroken = False
            if cfg.short_circuit and prefix == t:
                break
        if prefix == 0:
            e = NonConvergenceError(f"window {window_idx} did not converge within max_iter={cfg.max_iter}")
            e.report = dict(rows=rows, counts=dict(counts), windows=window_idx)  # ConvergenceReport
            raise e
        for n in range(1, prefix + 1):
            pos, vel = be.to_host(w.lam_prev[n])
            traj.append(ParticleSystem(pos, vel, v.charges, v.masses, v.box))
            point_iters.append(w.rows - 1)
        current = w.lam_prev[prefix]
        remaining -= prefix
    return ShardedPararealResult(traj, counts, window_idx, True, rows, point_iters, info)


# ============================================================================ spatial
def exchange_max_bits(tensors, group=None, use_dist: bool = True):
    """Exact exchange of disjointly owned values (include/msmb.h, spatial decomposition).

    `tensors` are the int64 views of one buffer on each local part. Unowned
    entries are INT64_MIN, so an element-wise MAX over parts and ranks leaves
    every owner's bit pattern in place. This also covers -0.0 (== INT64_MIN),
    NaNs and infinities. Local parts are combined first, then the result is
    all-reduced (MAX) over the ranks of `group` and copied back to every local
    part.
    """
    import torch
    m = tensors[0]
    if len(tensors) > 1:
        m = tensors[0].clone()
        for t in tensors[1:]:
            torch.maximum(m, t, out=m)
    dist = _dist() if use_dist else None
    if dist is not None and dist.get_world_size(group) > 1:
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    for t in tensors:
        if t is not m:
            t.copy_(m)
    return m


class SpatialDecomposition:
    """MSM force + velocity-Verlet propagation split over parts.

    One part per process/GPU under torchrun (``group``, default: the whole job),
    or ``local_parts`` parts in this process (one GPU). The latter runs the
    identical phase/exchange sequence; the tests use it to check the decomposed
    trajectory against the single-GPU one. Every part holds the whole particle
    state, owns an x-slab of the work, and exchanges exactly (see
    csrc/msmb_dd.cu and include/msmb.h). Results equal
    ``propagate(PropagatorSpec(MsmField(config), dt, steps), s)`` bit for bit.
    Only the energy differs: it is summed per part.
    """

    def __init__(self, config, system: ParticleSystem, units=None, group=None, local_parts: int = 0,
                 device: Optional[int] = None):
        import torch
        from . import DeviceSystem, UnitsConfig
        self.torch = torch
        self.group = group
        self.units = units or UnitsConfig.physical()
        self._uc = self.units._c()
        if local_parts:
            nparts, mine, self.distributed = int(local_parts), list(range(int(local_parts))), False
        else:
            comm = _Comm(group)
            nparts, mine, self.distributed = comm.world, [comm.rank], comm.world > 1
        self.nparts = nparts
        dev = torch.cuda.current_device() if device is None else device
        self.device = torch.device("cuda", dev)
        lib = _native.lib()
        self.lib = lib
        self.parts = []
        for p in mine:
            f = MsmField(config, self.units, device=dev)
            _check(f.handle, lib.msmb_dd_set_part(f.handle, nparts, p))
            ds = DeviceSystem(f, system)
            sizes = np.zeros(3, dtype=np.int64)
            _check(f.handle, lib.msmb_dd_sizes(f.handle, ds._h, sizes.ctypes.data_as(C.POINTER(C.c_int64))))
            bufs = [torch.empty(int(max(sz, 1)), dtype=torch.int64, device=self.device) for sz in sizes]
            self.parts.append((f, ds, bufs))
        self.system = system
        self.n = system.size()
        self.exchanged_bytes = 0

    def _phase(self, phase: int, dt: float = 0.0, kicks: int = 0, drift: int = 0) -> float:
        self.torch.cuda.current_stream(self.device).synchronize()
        energy = 0.0
        for f, ds, bufs in self.parts:
            e = C.c_double()
            xin = C.c_void_p(bufs[min(phase, 3) - 1].data_ptr()) if phase > 0 else None
            xout = C.c_void_p(bufs[phase].data_ptr()) if phase < 3 else None
            _check(f.handle, self.lib.msmb_dd_phase(f.handle, ds._h, phase, dt, kicks, drift, C.byref(self._uc),
                                                    xin, xout, C.byref(e)))
            energy += e.value
        return energy

    def _exchange(self, which: int, part: str = "all"):
        """Exchange buffer `which`; for the state buffer (2) `part` selects the
        positions ("pos", every step) or the velocities ("vel", after a list rebuild
        and at the end of a call: ownership only changes at rebuilds)."""
        bufs = [b[which] for _, _, b in self.parts]
        if which == 2 and part != "all":
            n3 = 3 * self.n
            bufs = [b[:n3] if part == "pos" else b[n3:2 * n3] for b in bufs]
        exchange_max_bits(bufs, self.group, use_dist=self.distributed)
        self.exchanged_bytes += bufs[0].numel() * 8
        self.torch.cuda.current_stream(self.device).synchronize()

    def _energy_sum(self, e: float) -> float:
        if not self.distributed:
            return e
        t = self.torch.tensor([e], dtype=self.torch.float64, device=self.device)
        _dist().all_reduce(t, group=self.group)
        return float(t.item())

    def _state(self):
        _, ds, _ = self.parts[0]
        t = self.torch.empty(6 * self.n, dtype=self.torch.float64, device=self.device)
        _check(self.parts[0][0].handle, self.lib.msmb_system_get_state_device(ds._h, C.c_void_p(t.data_ptr())))
        return t

    def _set_state(self, t):
        for f, ds, _ in self.parts:
            _check(f.handle, self.lib.msmb_system_set_state_device(ds._h, C.c_void_p(t.data_ptr())))

    def propagate(self, dt: float, steps: int, download: bool = True):
        """propagate(spec, s, units) (src/integrate.cpp:13-36): one evaluation, then
        `steps` velocity-Verlet steps. Returns (final ParticleSystem, energy of the
        last evaluation), or (None, energy) with download=False (the state stays on
        the devices). On error the state is left as it was, and the reference's
        exception is raised on every part."""
        if not (dt > 0.0):
            raise ConfigError("dt must be > 0")
        if steps < 0:
            raise ConfigError("steps_per_slice must be >= 1")
        backup = self._state()
        energy = 0.0
        vel_pending = False  # velocities of the last phase 2 not yet exchanged
        try:
            for s in range(steps + 1):
                if steps == 0:
                    kicks, drift = 0, 0
                elif s == 0:
                    kicks, drift = 1, 1      # opening half-kick + drift of step 1
                elif s < steps:
                    kicks, drift = 2, 1      # closing kick of step s, opening kick + drift of s+1
                else:
                    kicks, drift = 1, 0      # closing half-kick of the last step
                rebuilt = self._phase(0) > 0  # the (replicated) pair-list rebuild decision
                if rebuilt and vel_pending:  # new owners need the old owners' velocities
                    self._exchange(2, "vel")
                    self._phase(4)
                    vel_pending = False
                self._exchange(0)
                self._phase(1)
                self._exchange(1)
                energy = self._phase(2, dt, kicks, drift)
                if kicks or drift:
                    self._exchange(2, "pos")
                    self._phase(3)
                    vel_pending = True
            if vel_pending:
                self._exchange(2, "vel")
                self._phase(4)
        except Error:
            self._set_state(backup)
            raise
        energy = self._energy_sum(energy)
        if not download:
            return None, energy
        pos, vel = self.parts[0][1].download()
        s = self.system
        return ParticleSystem(pos, vel, s.charges, s.masses, s.box), energy
