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
recomputed identically).  This rests on every propagate call being a pure
function of its input state: each call builds its pair list afresh
(include/msmb.h, msmb_set_list_reuse), so a rank's coarse rows do not depend on
which fine slices it ran before -- every rank reaches the same skip and
convergence decisions and the same collectives.

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
class SpatialDecomposition:
    """MSM force + velocity-Verlet propagation split into x-slabs over GPUs
    (SURVEY.md 8(e) E1), driven by the C++ engine (csrc/msmb_slab.cu, msmb_slab_*).

    * Under torchrun (``group`` or the default process group with world > 1):
      one part per process/GPU.  Rank 0 creates an NCCL unique id
      (msmb_nccl_unique_id), torch.distributed broadcasts the 128 bytes, and
      every rank joins the library's own NCCL communicator; all halo and plane
      exchanges then run inside the C++ step (ncclSend/Recv), with no Python in
      the loop.
    * ``local_parts = P``: P parts driven by this process (one field per part, on
      ``devices`` or all on the current device), exchanging by stream-ordered
      copies -- the same plans and kernels, used by the tests to check the
      decomposed trajectory against the single-GPU one bit for bit.

    ``propagate(dt, steps)`` is propagate(spec, s, units) (src/integrate.cpp:13-36)
    on the whole system; every rank passes and receives the whole state.
    """

    def __init__(self, config, system: ParticleSystem, units=None, group=None, local_parts: int = 0,
                 device: Optional[int] = None, devices=None, transport: str = "auto"):
        from . import UnitsConfig
        self.units = units or UnitsConfig.physical()
        self.system = system
        self.n = system.size()
        lib = _native.lib()
        self.lib = lib
        self._h = C.c_void_p()
        if local_parts:
            nparts = int(local_parts)
            devs = list(devices) if devices else [0 if device is None else device] * nparts
            self.fields = [MsmField(config, self.units, device=devs[k % len(devs)]) for k in range(nparts)]
            arr = (C.c_void_p * nparts)(*[f.handle for f in self.fields])
            rc = lib.msmb_slab_create(arr, nparts, nparts, 0, None, None, C.byref(self._h))
            self.rank, self.world = 0, nparts
        else:
            import torch
            comm = _Comm(group)
            self.rank, self.world = comm.rank, comm.world
            dev = torch.cuda.current_device() if device is None else device
            self.fields = [MsmField(config, self.units, device=dev)]
            arr = (C.c_void_p * 1)(self.fields[0].handle)
            idbuf = (C.c_ubyte * 128)()
            # transport "nccl" forces the NCCL path even for one rank (a one-rank communicator)
            use_nccl = self.world > 1 or transport == "nccl"
            if use_nccl:
                if self.rank == 0:
                    _check(self.fields[0].handle, lib.msmb_nccl_unique_id(idbuf))
                if self.world > 1:
                    obj = [bytes(idbuf)]
                    comm.dist.broadcast_object_list(obj, src=0, group=group)
                    C.memmove(idbuf, obj[0], 128)
            rc = lib.msmb_slab_create(arr, 1, self.world, self.rank, idbuf if use_nccl else None, None,
                                      C.byref(self._h))
        _check(self.fields[0].handle, rc)
        self.last_energy = 0.0

    def propagate(self, dt: float, steps: int, download: bool = True, step_ms=None):
        """Returns (final ParticleSystem, energy of the last evaluation); the
        reference's exception on error (the same on every rank)."""
        s = self.system
        pos = np.array(s.positions, dtype=np.float64, copy=True)
        vel = np.array(s.velocities, dtype=np.float64, copy=True)
        e = C.c_double()
        u = self.units._c()
        rc = self.lib.msmb_slab_propagate(self._h, self.n, _p(pos), _p(vel), _p(s.charges), _p(s.masses), _p(s.box),
                                          float(dt), int(steps), C.byref(u), C.byref(e), _p(step_ms))
        _check(self.fields[0].handle, rc)  # the error is set on every part's field
        self.last_energy = e.value
        out = ParticleSystem(pos, vel, s.charges, s.masses, s.box)
        return (out if download else None), e.value

    def stats(self) -> dict:
        out = np.zeros(7, dtype=np.int64)
        self.lib.msmb_slab_stats(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)), 7)
        keys = ["bytes_per_step", "bytes_rebuild", "owned", "halo", "rebuilds", "migrated", "parts"]
        return dict(zip(keys, map(int, out)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            try:
                _native.lib().msmb_slab_destroy(h)
            except Exception:
                pass
            self._h = C.c_void_p()
