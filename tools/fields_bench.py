"""Throughput of the SURVEY.md 8(f) fields on one B200 (device-resident, CUDA-event timed).

* cutoff / wolf : C2-S (300,000 atoms, 144 A) propagated with SimpleCutoffField /
                  WolfField (a = 12 A, Wolf alpha 0.2), atom-steps/s, plus the pair
                  kernel's time from a stage-timing pass.
* direct        : DirectCoulombField evaluations at N = 8192 (C1) and 65536, in
                  ordered pair evaluations / s and FP64 issue-slot fraction
                  (18 DP instructions per ordered pair, the kernel's count).
* parareal      : C5-S parareal with the paper's pairing, MSM fine (a=12 h=2.5 l=4,
                  dt 0.005 x 100) + cutoff coarse (a=8, dt 0.02 x 25), 8 slices, K=1.
Prints one JSON object.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import _native, fixtures as fx
import ctypes as C


def timed_propagate(field, w, steps):
    dev = pkg.DeviceSystem(field, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
    dev.propagate(w.dt, 2)  # warm-up: workspace, list, graphs
    ms = np.zeros(steps + 2)
    names = (C.c_char_p * 16)()
    launches = np.zeros(1, dtype=np.int64)
    rc = _native.lib().msmb_bench_propagate(field.handle, dev._h, w.dt, steps, 1, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                            np.zeros(16).ctypes.data_as(C.POINTER(C.c_double)), names,
                                            launches.ctypes.data_as(C.POINTER(C.c_int64)))
    assert rc == 0
    step_ms = float(np.mean(ms[1:steps + 1]))
    field.set_stage_timing(True)
    field.reset_stage_times()
    dev.propagate(w.dt, 5)
    st = field.stage_times()
    field.set_stage_timing(False)
    pairs_ms = st["pairs"][0] / 6
    return step_ms, pairs_ms, field.work_counters()


def main():
    out = {}
    peak = C.c_double()
    _native.lib().msmb_measure_fp64_peak(0, 0.5, C.byref(peak))
    out["fp64_peak_tflops"] = peak.value
    w = fx.config("c2s")
    for name, f in [("cutoff", pkg.SimpleCutoffField(pkg.CutoffParams(12.0))),
                    ("wolf", pkg.WolfField(pkg.CutoffParams(12.0, 0.2)))]:
        step_ms, pairs_ms, wc = timed_propagate(f, w, 20)
        out[name] = dict(n=int(w.n), ms_per_step=step_ms, atom_steps_per_s=w.n / (step_ms * 1e-3),
                         pairs_ms=pairs_ms, pairs=wc["pairs"], launches_per_eval=wc["launches_per_eval"])
    for n in (8192, 65536):
        rng = np.random.default_rng(1)
        L = (n / 0.1) ** (1 / 3)
        s = pkg.ParticleSystem(rng.uniform(0, L, (n, 3)), None, rng.choice([-1.0, 1.0], n), None, np.array([L] * 3))
        f = pkg.DirectCoulombField()
        f.evaluate(s)
        dev = pkg.DeviceSystem(f, s)
        dev.evaluate()
        import torch
        torch.cuda.synchronize()
        reps = 20 if n <= 8192 else 5
        t0 = time.perf_counter()
        for _ in range(reps):
            dev.evaluate()
        dt = (time.perf_counter() - t0) / reps  # includes the D2H of the outputs
        f.set_stage_timing(True)
        f.reset_stage_times()
        dev.evaluate()
        kern_ms = f.stage_times()["pairs"][0]
        f.set_stage_timing(False)
        slots = 18.0 * n * (n - 1)
        out[f"direct_{n}"] = dict(eval_ms_host=dt * 1e3, kernel_ms=kern_ms,
                                  pair_evals_per_s=n * (n - 1) / (kern_ms * 1e-3),
                                  fp64_slot_frac=slots / (kern_ms * 1e-3) / (peak.value * 1e12 / 2))
    # parareal, paper pairing: MSM fine + cutoff coarse
    w = fx.config("c5s")
    fa, fh, fl, fdt, fs = w.extra["fine"]
    ga, gh, gl, gdt, gs = w.extra["coarse"]
    F = pkg.MsmField(pkg.MsmConfig(fa, fh, fl))
    G = pkg.SimpleCutoffField(pkg.CutoffParams(ga))
    cfg = pkg.PararealConfig(8, 1, 1e300, pkg.PropagatorSpec(F, fdt, fs), pkg.PropagatorSpec(G, gdt, gs),
                             short_circuit=False)
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    pkg.propagate(pkg.PropagatorSpec(F, fdt, 2), s)
    pkg.propagate(pkg.PropagatorSpec(G, gdt, 2), s)
    t0 = time.perf_counter()
    row, dr, counts = pkg.parareal_window(s, cfg, 8, 1)
    t = time.perf_counter() - t0
    out["parareal_msm_fine_cutoff_coarse_K1"] = dict(n=int(w.n), seconds=t, atom_steps_per_s=w.n * 800 / t,
                                                     counts=counts)
    # the reference's own CPU path for the same fields (oracle/_ref, 1 thread): an
    # O(N^2) i<j loop, timed on a random subset and scaled by the pair-check count
    try:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
        import oracle_lib
        if oracle_lib.have("ref"):
            ref = oracle_lib.checker("ref")
            w = fx.config("c2s")
            M = 20000
            idx = np.sort(np.random.default_rng(0).choice(w.n, M, replace=False))
            for name, spec in [("cutoff", oracle_lib.fspec("cutoff", 12.0)),
                               ("wolf", oracle_lib.fspec("wolf", 12.0, alpha=0.2)),
                               ("direct", oracle_lib.fspec("direct", 0.0))]:
                t0 = time.perf_counter()
                ref.field_evaluate(spec, w.pos[idx], w.q[idx], w.box)
                t = (time.perf_counter() - t0) * (w.n * (w.n - 1)) / (M * (M - 1))
                out.setdefault("cpu_reference_1thread", {})[name] = dict(
                    sample=f"{M}-atom random subset of C2-S, scaled by N(N-1)/(M(M-1))",
                    seconds_per_eval_at_300k=t, atom_steps_per_s=w.n / t)
    except Exception as e:  # the checker is optional on the box
        out["cpu_reference_1thread"] = f"unavailable: {e}"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
