#!/usr/bin/env python
"""Benchmark: MSM force + velocity-Verlet atom-steps/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2s]

Workload (N=1): BASELINE.json configs[1] -- 100,000 rigid 3-site waters (300,000
atoms) in a 144 A cube, MSM a=12 A, h=2.5 A, 6 levels (top 8^3), fp64, velocity
Verlet.  The literal input aborts in the reference at step 1 (CoverageError,
reproduced bit-exactly by tests/test_gpu_errors.py), so throughput is measured on
the survivable variant c2s (same N, box, a/h/l; O-O min separation 2.5 A,
dt 0.02 fs) -- SURVEY.md 8(d) protocol P2.  Inputs are seeded synthetic.

A "step" = one Verlet step = one full MSM energy/force evaluation + kick/drift
(src/integrate.cpp:23-34).  The timed region is one device-resident propagate
(initial evaluation + K steps + closing half-kick, as the reference library's
propagate), timed with CUDA events on the engine's stream around every step, with
a 256 MB (> L2) buffer written between steps outside the events.

Multi-GPU (torchrun, --gpus N > 1): the paths that shard.  The line is
configs[2] C3-S (2^24 charges) propagated through the spatial slab decomposition
(parallel.SpatialDecomposition -> csrc/msmb_slab.cu, NCCL halos, one part per GPU),
and it carries a nested `parareal` object: configs[4] C5-S with the fine slices
sharded over the ranks.  The N = 1 line carries both at one GPU in
`scaling_base` (same code paths), so per-N values of the same workloads can be
compared.  Device time = CUDA events per step on the part's stream, max over ranks.

`--impl reference` times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference sources) on a bounded sample per step; rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MSM force+Verlet atom-steps/s"
UNIT = "atom-steps/s"

CONFIG_TEXT = {
    "c2s": "configs[1] survivable variant c2s: 100,000 rigid 3-site water-like molecules (300,000 atoms, "
           "O -0.834 / H +0.417, 16/1 amu), 144 A cube, MSM a=12 A h=2.5 A cubic, 6 levels (top 8^3), "
           "O-O min separation 2.5 A, dt 0.02 fs",
    "c2": "configs[1] literal (aborts at step 1 in the reference; not benchmarkable)",
    "c1s": "configs[0] survivable variant: 8,192 atoms, 40 A, a=10 h=2.5 l=2, RSA 1.5 A, dt 0.02 fs",
    "c5f": "configs[4] fine propagator on the literal C5 system: 2^20 atoms, 219 A, a=12 h=2.5 l=4, dt 0.5 fs",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2s")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-scaling-base", action="store_true", help="N=1: skip the C3-S / C5-S one-GPU lines")
    ap.add_argument("--multi-path", action="store_true",
                    help="run the --gpus N > 1 line's code path even on one rank (one-rank NCCL communicator)")
    ap.add_argument("--no-full-reference", action="store_true",
                    help="--impl reference: skip the one full-size short_range calibration")
    return ap.parse_args()


# ----------------------------------------------------------------------------- dist
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.dist, self.torch, self.backend = dist, torch, backend

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64,
                              device=f"cuda:{self.local}" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clocks + throttle reasons during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int, period=0.01):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        self.stop_ev = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.t.join()

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU reference
def reference_step_estimate(w, sample_atoms: int, seed: int):
    """One bounded sample of the reference's per-step cost on this host (1 thread).

    reference msm_potential = short_range (O(N^2) i<j loop, src/msm_phases.cpp:224-252)
    + grid phases (anterpolate .. interpolate, src/msm_phases.cpp:39-222) + long-range
    forces (src/msm.cpp:16-48, ~3x interpolate) + the Verlet update (negligible).
    short_range is timed on a random `sample_atoms` subset of the same box and scaled
    by N(N-1)/(M(M-1)) (its pair-check count); the grid phases run at full N."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    if oracle_lib.have("ref"):
        chk, kind = oracle_lib.checker("ref"), "reference"
    else:  # the C restatement, when the reference could not be compiled here
        chk, kind = oracle_lib.checker("port"), "port"
    rng = np.random.default_rng(seed)
    m = min(sample_atoms, w.n)
    idx = np.sort(rng.choice(w.n, size=m, replace=False))
    pos = np.ascontiguousarray(w.pos[idx])
    q = np.ascontiguousarray(w.q[idx])
    t0 = time.perf_counter()
    if kind == "reference":
        t_sr = chk.lib.ref_time_short_range(m, oracle_lib._p(pos), oracle_lib._p(q), w.a, 332.0636, 1)
        ph = np.zeros(6)
        buf = C.create_string_buffer(256)
        chk.lib.ref_time_phases.argtypes = [C.c_int64, oracle_lib._D, oracle_lib._D, oracle_lib._D, C.c_double,
                                            C.c_double, C.c_int, oracle_lib._D, C.c_char_p, C.c_int]
        rc = chk.lib.ref_time_phases(w.n, oracle_lib._p(np.ascontiguousarray(w.pos)), oracle_lib._p(w.q),
                                     oracle_lib._p(w.box), w.a, w.h, w.levels, oracle_lib._p(ph), buf, 256)
        if rc != 0:
            raise RuntimeError(buf.value.decode())
        t_grid = float(ph.sum()) + 3.0 * float(ph[5])
    else:
        t = time.perf_counter()
        chk.short_range(pos, q, w.a)
        t_sr = time.perf_counter() - t
        t = time.perf_counter()
        chk.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels)
        t_grid = time.perf_counter() - t
    wall = time.perf_counter() - t0
    scale = (w.n * (w.n - 1.0)) / (m * (m - 1.0))
    t_step = t_sr * scale + t_grid
    return {"t_step_s": t_step, "t_short_sample_s": t_sr, "t_grid_s": t_grid, "sample_atoms": m,
            "wall_s": wall, "kind": kind}


def cpu_threads_used():
    return 1


def reference_full_short_range(w):
    """The reference's short_range (src/msm_phases.cpp:224-252) once on the whole system."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    if not oracle_lib.have("ref"):
        return None
    chk = oracle_lib.checker("ref")
    pos = np.ascontiguousarray(w.pos)
    t = chk.lib.ref_time_short_range(w.n, oracle_lib._p(pos), oracle_lib._p(np.ascontiguousarray(w.q)), w.a,
                                     332.0636, 1)
    return {"t_full_s": float(t)}


def reference_c3_estimate(w, steps, warmup):
    """Reference per-step cost on C3 (2^24 atoms; a full step is ~4.5 days of short_range
    + ~95 s of grid phases on one core): grid phases timed once on a 1/8-volume sub-box
    (2^21 atoms, same density) and scaled per phase (x8; top level x64 = (M_top ratio)^2),
    short_range on a 30,000-atom subset per step scaled by its N(N-1)/2 pair checks."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    chk = oracle_lib.checker("ref") if oracle_lib.have("ref") else None
    if chk is None:
        return None
    from paper_1309_1889_b200 import fixtures as fx
    sub = fx.config("c3s", n_override=1 << 21)
    ph = np.zeros(6)
    buf = C.create_string_buffer(256)
    chk.lib.ref_time_phases.argtypes = [C.c_int64, oracle_lib._D, oracle_lib._D, oracle_lib._D, C.c_double,
                                        C.c_double, C.c_int, oracle_lib._D, C.c_char_p, C.c_int]
    rc = chk.lib.ref_time_phases(sub.n, oracle_lib._p(np.ascontiguousarray(sub.pos)), oracle_lib._p(sub.q),
                                 oracle_lib._p(sub.box), sub.a, sub.h, sub.levels, oracle_lib._p(ph), buf, 256)
    if rc != 0:
        raise RuntimeError(buf.value.decode())
    scale = np.array([8, 8, 8, 64, 8, 8 * 4.0]) # interpolate + long-range forces ~ 4x interpolate
    t_grid = float(np.sum(ph * scale))
    srs = []
    rng = np.random.default_rng(3)
    for k in range(warmup + steps):
        idx = np.sort(rng.choice(w.n, size=30000, replace=False))
        pos = np.ascontiguousarray(w.pos[idx])
        q = np.ascontiguousarray(w.q[idx])
        t = chk.lib.ref_time_short_range(30000, oracle_lib._p(pos), oracle_lib._p(q), w.a, 332.0636, 1)
        if k >= warmup:
            srs.append(t * (w.n * (w.n - 1.0)) / (30000 * 29999.0))
    return {"t_step_s": float(np.mean(srs)) + t_grid, "t_grid_s": t_grid, "t_short_s": float(np.mean(srs))}


SPATIAL_TEXT = ("configs[2] survivable variant c3s: 2^24 point charges (RSA min-separation 1.5 A; the literal "
                "input aborts at step 2, tests/test_gpu_fullsize_parity.py), 551 A cube, +-1 rebalanced to net "
                "zero, 18 amu, MSM a=12 A h=2.5 A cubic, 4 levels, dt 0.02 fs")
PARAREAL_TEXT = ("configs[4] survivable variant c5s: 2^20 charges (RSA 1.5 A), F MSM a=12 h=2.5 l=4 dt 0.005 fs "
                 "x100, G MSM a=8 h=5 l=3 dt 0.02 fs x25, one window of 8 slices, K=1 iteration (no short circuit)")


def spatial_run(D, steps, warmup, transport="auto"):
    """C3-S through the slab decomposition over D.world GPUs: device-timed steps
    (events on each part's stream, max over ranks) and the end-to-end call time."""
    import paper_1309_1889_b200 as pkg
    from paper_1309_1889_b200 import fixtures as fx, parallel
    w = fx.config("c3s")
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, device=D.local, transport=transport)
    dd.propagate(w.dt, max(1, warmup))  # workspaces, plans
    D.barrier()
    sm = np.zeros(steps + 2)
    l0 = dd.fields[0].kernel_launches()
    with ClockSampler(D.local) as clk:
        t0 = time.perf_counter()
        dd.propagate(w.dt, steps, step_ms=sm)
        wall = D.max(time.perf_counter() - t0)
    launches = dd.fields[0].kernel_launches() - l0
    D.barrier()
    dev_ms = D.max(float(sm[1:steps + 1].sum()))
    st = dd.stats()
    bytes_step = D.max(float(st["bytes_per_step"]))
    value = w.n * steps / (dev_ms * 1e-3)
    nbytes = w.n * 64  # every rank uploads the whole system and downloads pos/vel
    return w, {
        "value": value, "ms_per_step": dev_ms / steps, "clocks": clk.result(), "gpu_launches": int(launches),
        "e2e": {"value": w.n * steps / wall, "unit": UNIT, "h2d_bytes_per_step": nbytes / steps,
                "d2h_bytes_per_step": w.n * 48 / steps,
                "note": "one msmb_slab_propagate call per rank from host arrays (whole system in, whole final "
                        "state out): upload, decomposition setup, initial evaluation, K steps, final gather; "
                        "host wall clock, max over ranks"},
        "exchange": {"bytes_received_per_step_per_rank": bytes_step, "halo_atoms": st["halo"],
                     "owned_atoms": st["owned"], "rebuilds": st["rebuilds"], "migrated": st["migrated"]},
        "config": {"workload": SPATIAL_TEXT, "n_atoms": int(w.n), "a": w.a, "h": w.h, "levels": w.levels,
                   "dt_fs": w.dt, "parallelism": f"spatial x-slab decomposition over {D.world} GPU(s) "
                                                 f"(csrc/msmb_slab.cu; NCCL halos)" if D.world > 1 else
                                                 "spatial decomposition, one part (single GPU)",
                   "l2": "inputs (1.1 GB state + 30 GB workspace) far exceed L2"},
    }


def parareal_run_line(D, K=1):
    """C5-S parareal with the fine slices sharded over the ranks (parallel.parareal_run)."""
    import torch
    import paper_1309_1889_b200 as pkg
    from paper_1309_1889_b200 import fixtures as fx, parallel
    w = fx.config("c5s")
    fa, fh, fl, fdt, fs = w.extra["fine"]
    ga, gh, gl, gdt, gs = w.extra["coarse"]
    F = pkg.MsmField(pkg.MsmConfig(fa, fh, fl), device=D.local)
    G = pkg.MsmField(pkg.MsmConfig(ga, gh, gl), device=D.local)
    cfg = pkg.PararealConfig(8, K, 1e300, pkg.PropagatorSpec(F, fdt, fs), pkg.PropagatorSpec(G, gdt, gs),
                             short_circuit=False)
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    be = parallel.DeviceBackend(cfg, s)
    st0 = be.from_system(s)
    be.propagate("fine", st0)  # warm-up: workspaces, plans, captured step graphs
    be.propagate("coarse", st0)
    torch.cuda.synchronize(D.local)
    D.barrier()
    t0 = time.perf_counter()
    res = parallel.parareal_run(s, 8, cfg, backend=be)
    torch.cuda.synchronize(D.local)
    D.barrier()
    wall = D.max(time.perf_counter() - t0)
    return {"value": w.n * 8 * fs / wall, "unit": UNIT, "ms_per_run": wall * 1e3, "K": K, "counts": res.counts,
            "metric_note": "SURVEY 8(d): N x fine steps over the horizon (8 slices x 100) / wall time of "
                           "parareal_init + K x parareal_iterate (host wall clock, max over ranks)",
            "workload": PARAREAL_TEXT,
            "parallelism": f"fine slices over {D.world} GPU(s) (parallel.parareal_run, NCCL broadcast of deltas)"}


def multi_gpu(args, D):
    """--gpus N > 1 under torchrun: the sharding paths (C3-S spatial, C5-S parareal)."""
    import torch
    torch.cuda.set_device(D.local)
    if args.impl == "reference":
        if D.rank == 0:
            from paper_1309_1889_b200 import fixtures as fx
            w = fx.config("c3s")
            est = reference_c3_estimate(w, args.steps, args.warmup)
            if est is None:
                print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}), flush=True)
                return
            val = w.n / est["t_step_s"]
            line = {"metric": METRIC, "impl": "reference", "value": val, "unit": UNIT, "n_gpus": D.world,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": est["t_step_s"] * 1e3,
                    "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                    "data": "synthetic (seeded)",
                    "config": {"workload": SPATIAL_TEXT, "n_atoms": int(w.n)},
                    "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "reference",
                                     "sample": "grid phases timed once on a 1/8-volume sub-box (2^21 atoms) and "
                                               "scaled per phase (x8, top x64); short_range on a 30,000-atom "
                                               "subset per step scaled by N(N-1)/2 pair checks; single-threaded"},
                    "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        return
    w, sp = spatial_run(D, args.steps, args.warmup, transport="nccl")
    par = parareal_run_line(D, 1)
    if D.rank == 0:
        line = {"metric": METRIC, "value": sp["value"], "unit": UNIT, "n_gpus": D.world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": sp["ms_per_step"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded; paper_1309_1889_b200/fixtures.py)", "config": sp["config"],
                "e2e": sp["e2e"], "exchange": sp["exchange"], "gpu_launches": sp["gpu_launches"],
                "clocks": sp["clocks"], "parareal": par}
        print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- main
def main():
    args = parse()
    D = Dist()
    from paper_1309_1889_b200 import fixtures as fx
    if D.world > 1 or args.multi_path:
        multi_gpu(args, D)
        D.close()
        return

    name = args.config
    wname = {"c5f": "c5"}.get(name, name)
    w = fx.config(wname)
    base = {"metric": METRIC, "unit": UNIT, "n_gpus": D.world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; paper_1309_1889_b200/fixtures.py)",
            "config": {"workload": CONFIG_TEXT.get(name, name), "n_atoms": int(w.n), "a": w.a, "h": w.h,
                       "levels": w.levels, "dt_fs": w.dt, "parallelism": "single GPU", "l2": "256 MB buffer written before every timed step (outside the "
                       "events); per-step working set ~230 MB (incl. 147 MB of pair masks)"}}

    if args.impl == "reference":
        if D.rank == 0:
            times = []
            for k in range(args.warmup + args.steps):
                est = reference_step_estimate(w, 30000, 100 + k)
                if k >= args.warmup:
                    times.append(est)
            t_sr_ext = float(np.mean([e["t_step_s"] - e["t_grid_s"] for e in times]))
            t_grid = float(np.mean([e["t_grid_s"] for e in times]))
            calib = None
            if not args.no_full_reference:
                # one FULL-size reference short_range (all N(N-1)/2 pair checks, ~1-2 min): the
                # sample extrapolation runs from cache, the full call from memory
                calib = reference_full_short_range(w)
            t_sr = calib["t_full_s"] if calib else t_sr_ext
            t = t_sr + t_grid
            val = w.n / t
            line = dict(base, impl="reference", value=val, ms_per_step=t * 1e3, n_gpus=D.world,
                        cpu_baseline={"value": val, "unit": UNIT, "cores": cpu_threads_used(),
                                      "kind": times[0]["kind"],
                                      "sample": (f"per step: the reference short_range timed ONCE at full size "
                                                 f"({calib['t_full_s']:.1f} s for N={w.n}) + reference grid phases at "
                                                 f"full N ({t_grid:.2f} s per step); " if calib else "")
                                                + f"per-step samples: short_range on a random "
                                                  f"{times[0]['sample_atoms']}-atom subset scaled by N(N-1)/2 pair "
                                                  f"checks -> {t_sr_ext:.1f} s (extrapolation check); "
                                                  f"single-threaded (msm_potential has no threading)",
                                      "short_range_full_s": calib["t_full_s"] if calib else None,
                                      "short_range_extrapolated_s": t_sr_ext},
                        e2e={"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
            print(json.dumps(line), flush=True)
        D.close()
        return

    import paper_1309_1889_b200 as pkg
    from paper_1309_1889_b200 import _native, roofline

    dev_id = D.local
    L = _native.lib()
    field = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels), pkg.UnitsConfig.physical(), device=dev_id)
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    dev = pkg.DeviceSystem(field, s)
    dt = 0.5 if name == "c5f" else w.dt
    K, W = args.steps, args.warmup

    def bench(steps, flush):
        step_ms = np.zeros(steps + 2)
        stage_ms = np.zeros(11)
        names = (C.c_char_p * 11)()
        launches = C.c_int64()
        rc = L.msmb_bench_propagate(field.handle, dev._h, dt, steps, int(flush), step_ms.ctypes.data_as(pkg._D),
                                    stage_ms.ctypes.data_as(pkg._D), names, C.byref(launches))
        pkg._check(field.handle, rc)
        return step_ms, dict(zip([n.decode() for n in names], stage_ms)), launches.value

    bench(max(W, 1), not args.no_flush)  # warm-up: graph capture + upload + caches
    D.barrier()
    with ClockSampler(dev_id) as clk:
        step_ms, stage_ms, launches = bench(K, not args.no_flush)
    D.barrier()
    total_ms = float(step_ms.sum())
    total_max = D.max(total_ms)
    value = D.world * w.n * K / (total_max * 1e-3)
    # informational: the same steps back to back (no L2 flush, no per-step host sync), as a
    # propagate call runs them -- the marginal cost of a step from two device-resident calls
    import time as _time
    def _wall(steps):
        dev.upload(w.pos, w.vel)  # every call from the input state (the survivable horizon is finite)
        t0 = _time.perf_counter()
        dev.propagate(dt, steps)
        return _time.perf_counter() - t0
    try:
        _wall(2)
        t_k, t_2k = _wall(K), _wall(2 * K)
        back_to_back = {"ms_per_step": (t_2k - t_k) / K * 1e3,
                        "note": "marginal step cost of device-resident propagate calls of K and 2K steps from the "
                                "input state (host wall clock; graphs launched back to back, L2 not flushed): "
                                "not the headline"}
    except pkg.Error as ex:  # e.g. a long --steps run leaving the grid coverage
        back_to_back = {"ms_per_step": None, "note": f"not measured: {ex}"}
    dev.upload(w.pos, w.vel)
    # per-stage times: a second pass over K more steps with CUDA events around every
    # stage on the engine's stream (eager launches instead of the graph); its
    # evaluations also count the in-cutoff pairs (the graph's pair kernel skips that)
    field.set_stage_timing(True)
    field.reset_stage_times()
    dev.propagate(dt, K)
    st_times = field.stage_times()
    field.set_stage_timing(False)
    counters = field.work_counters()
    stage_ms = {k: v[0] for k, v in st_times.items()}

    # ---- roofline: dominant kernel (short-range pairs) and per-stage model
    tf = C.c_double()
    L.msmb_measure_fp64_peak(dev_id, 0.5, C.byref(tf))
    fp64_peak = tf.value
    hbm, hbm_src = roofline.hbm_peak_gbs()
    evals = K + 1
    pair_ms = stage_ms.get("pairs", 0.0) / evals
    pairs_u = counters["pairs"]
    achieved = roofline.PAIR_FLOPS * pairs_u / (pair_ms * 1e-3) / 1e12 if pair_ms > 0 else 0.0
    slot_frac = (roofline.PAIR_SLOTS * pairs_u / (pair_ms * 1e-3)) / (fp64_peak * 1e12 / 2) if pair_ms > 0 else 0.0
    dims, _, _ = pkg.grid_geometry(field.config(), w.box)
    lsz = [int(np.prod(d)) for d in dims]
    per_step = {k: v / evals for k, v in stage_ms.items()}
    per_step["verlet"] = stage_ms.get("verlet", 0.0) / K
    stages, t_roof, t_meas = roofline.evaluate(w.n, lsz, pairs_u, counters["lattice_taps"], counters["top_taps"],
                                               per_step, fp64_peak, hbm)
    traffic = None
    tr_file = ROOT / "profiles" / "ncu_traffic.json"
    if tr_file.exists():
        try:
            traffic = json.loads(tr_file.read_text()).get(name, {}).get("k_pairs_mw_dram_bytes")
        except Exception:
            traffic = None

    # ---- e2e: the public host API, pinned host buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        n = w.n
        nbytes_in = n * (24 + 24 + 8 + 8)
        nbytes_out = n * 48
        ptr = L.msmb_host_alloc(n * 8 * 8)
        host = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(n * 8,))
        hp, hv, hq, hm = host[:3 * n], host[3 * n:6 * n], host[6 * n:7 * n], host[7 * n:8 * n]
        box = np.ascontiguousarray(w.box)

        def run_e2e(steps):
            hp[:] = w.pos.ravel()
            hv[:] = w.vel.ravel()
            hq[:] = w.q
            hm[:] = w.mass
            t = time.perf_counter()
            rc = L.msmb_propagate(field.handle, n, hp.ctypes.data_as(pkg._D), hv.ctypes.data_as(pkg._D),
                                  hq.ctypes.data_as(pkg._D), hm.ctypes.data_as(pkg._D), box.ctypes.data_as(pkg._D),
                                  dt, steps)
            el = time.perf_counter() - t
            pkg._check(field.handle, rc)
            return el

        run_e2e(max(W, 1))
        D.barrier()
        el = D.max(run_e2e(K))
        e2e = {"value": D.world * n * K / el, "unit": UNIT, "h2d_bytes_per_step": nbytes_in / K,
               "d2h_bytes_per_step": nbytes_out / K,
               "note": "one public msmb_propagate call (host AoS arrays in pinned memory -> H2D, initial evaluation "
                       "+ K steps, D2H of positions/velocities); host wall clock, max over ranks"}
        L.msmb_host_free(ptr)

    # ---- the rebuild-inclusive cost: skin 0 rebuilds the pair list (clusters, boxes,
    # lists, masks) at every evaluation, as at a dt where atoms cross skin/2 every step
    field.set_pair_skin(0.0)
    dev0 = pkg.DeviceSystem(field, s)
    step0 = np.zeros(K + 2)
    stage0 = np.zeros(11)
    names0 = (C.c_char_p * 11)()
    l0 = C.c_int64()
    L.msmb_bench_propagate(field.handle, dev0._h, dt, max(W, 1), int(not args.no_flush), step0.ctypes.data_as(pkg._D),
                           stage0.ctypes.data_as(pkg._D), names0, C.byref(l0))
    pkg._check(field.handle, L.msmb_bench_propagate(field.handle, dev0._h, dt, K, int(not args.no_flush),
                                                    step0.ctypes.data_as(pkg._D), stage0.ctypes.data_as(pkg._D),
                                                    names0, C.byref(l0)))
    rb_ms = float(step0[1:K + 1].sum()) / K
    rebuild_line = {"ms_per_step": rb_ms, "value": w.n / (rb_ms * 1e-3),
                    "list_rebuilds": field.work_counters()["list_rebuilds"],
                    "note": "pair-list skin 0: the cluster pair list (clusters, boxes, list, masks) is rebuilt at "
                            "every evaluation -- the cost of a step at a dt (e.g. C2's literal 1 fs) where atoms "
                            "cross skin/2 every step; the headline steps (dt 0.02 fs) rebuild once per call"}
    del dev0

    scaling_base = None
    if not args.no_scaling_base:
        _, sp = spatial_run(D, max(3, K // 4), 1)
        scaling_base = {"spatial_c3s_1gpu": {k: sp[k] for k in ("value", "ms_per_step", "e2e", "config")},
                        "parareal_c5s_1gpu": parareal_run_line(D, 1),
                        "note": "the --gpus N > 1 lines' workloads (C3-S spatial, C5-S parareal) through the same "
                                "code paths at one GPU, for scaling efficiency against the N > 1 lines"}

    cpu = None
    if D.rank == 0 and D.world == 1 and not args.no_cpu_baseline:
        est = reference_step_estimate(w, 40000, 7)
        cpu = {"value": w.n / est["t_step_s"], "unit": UNIT, "cores": cpu_threads_used(), "kind": est["kind"],
               "sample": f"reference short_range on a random {est['sample_atoms']}-atom subset of the same box "
                         f"({est['t_short_sample_s']:.2f} s) scaled by its N(N-1)/2 pair-check count, + the "
                         f"reference grid phases at full N ({est['t_grid_s']:.2f} s); one evaluation = one step",
               "host_cpus": os.cpu_count()}

    if D.rank == 0:
        line = dict(base)
        line.update({
            "value": value, "ms_per_step": total_max / K,
            "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.result(),
            "roofline": {"bound": "fp64", "kernel": "k_pairs_mw (short-range pair sum, SURVEY S2)",
                         "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                         "slot_frac": slot_frac, "traffic": traffic,
                         "traffic_note": "DRAM bytes per launch from the ncu capture named in profiles/ncu_traffic.json "
                                         "(r02c_k_pairs_mw_full.md): mostly the per-lane pair masks (k_pairmask, 128 B "
                                         "per list entry) and the dense lists (4 B per dense atom), read once per "
                                         "evaluation (L2-flushed between timed steps), not atom data",
                         "work_per_launch": f"{pairs_u} in-cutoff unordered pairs x {roofline.PAIR_FLOPS} flops "
                                            f"({roofline.PAIR_SLOTS} FP64 issue slots)",
                         "avg_launch_ms": pair_ms,
                         "peak_source": "FP64 FMA-chain microbenchmark run live in this bench (msmb_measure_fp64_peak); "
                                        "MEASURED_PEAKS.json has no FP64 entry"},
            "step_roofline": {"t_roof_ms": t_roof, "t_measured_ms": t_meas, "frac": t_roof / t_meas if t_meas else None,
                              "frac_of_step": t_roof / (total_max / K),
                              "note": "frac: against the serialised per-stage times (stage-timing pass, no "
                                      "overlap); frac_of_step: against the measured step (ms_per_step)",
                              "hbm_gbs": hbm, "hbm_source": hbm_src, "fp64_tflops": fp64_peak, "stages": stages},
            "stage_ms_per_eval": {k: round(v, 5) for k, v in per_step.items()},
            "cpu_baseline": cpu,
            "work": counters,
            "rebuild_every_step": rebuild_line,
            "back_to_back": back_to_back,
            "scaling_base": scaling_base,
        })
        print(json.dumps(line), flush=True)
    D.close()


if __name__ == "__main__":
    main()
