"""Throughput of the multi-GPU paths; called by `bench.py --workload ...`.

spatial  : C3 (2^24 atoms, 551 A, a=12 h=2.5 l=4) propagated through
           parallel.SpatialDecomposition, one part per rank (torchrun), `steps`
           Verlet steps at dt 2 fs (C3's literal step; a few steps survive).
parareal : (parareal_cutoff: the same with the paper's simple-cutoff G, a=8)
           C5-S (2^20 atoms; RSA 1.5 A; F a=12 h=2.5 l=4 dt 0.005 fs x 100, G a=8 h=5
           l=3 dt 0.02 fs x 25; 8 slices) through parallel.parareal_run with the fine
           slices sharded over ranks, K = `steps` iterations (no short circuit).
           Metric: N x fine steps over the horizon (8 x 100) / time.
Wall-clock timing around a full call (host-driven phases), with a CUDA sync and a
barrier on both sides; max over ranks.
"""
from __future__ import annotations

import json
import time

import numpy as np


def run(args, d, metric, unit):
    import torch
    import paper_1309_1889_b200 as pkg
    from paper_1309_1889_b200 import fixtures as fx, parallel
    torch.cuda.set_device(d.local)
    dev = torch.device("cuda", d.local)
    if args.workload == "spatial":
        w = fx.config("c3s")
        s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
        dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, device=d.local)
        dd.propagate(w.dt, max(1, args.warmup), download=False)  # warm-up (workspaces, plans)
        torch.cuda.synchronize(dev)
        d.barrier()
        t0 = time.perf_counter()
        dd.propagate(w.dt, args.steps, download=False)
        torch.cuda.synchronize(dev)
        d.barrier()
        dt = d.max(time.perf_counter() - t0)
        steps = args.steps
        value = w.n * steps / dt
        cfg = {"workload": "configs[2] C3-S: 2^24 point charges (RSA 1.5 A; the literal input aborts at step 2), 551 A cube, a=12 A h=2.5 A l=4, dt 0.02 fs",
               "n_atoms": int(w.n), "parallelism": f"spatial decomposition over {d.world} GPU(s) (x-slabs)",
               "exchanged_bytes_per_step_per_rank": int(dd.exchanged_bytes / (args.steps + max(1, args.warmup) + 2))}
        extra = {"ms_per_step": 1e3 * dt / steps}
    else:
        w = fx.config("c5s")
        fa, fh, fl, fdt, fs = w.extra["fine"]
        ga, gh, gl, gdt, gs = w.extra["coarse"]
        F = pkg.MsmField(pkg.MsmConfig(fa, fh, fl), device=d.local)
        if args.workload == "parareal_cutoff":  # the paper's G: simple cutoff at the coarse a
            G = pkg.SimpleCutoffField(pkg.CutoffParams(ga), device=d.local)
        else:
            G = pkg.MsmField(pkg.MsmConfig(ga, gh, gl), device=d.local)
        K = max(1, args.steps)
        # one window of 8 slices, exactly K iterations: a tol every point meets, no short
        # circuit
        cfg_p = pkg.PararealConfig(8, K, 1e300, pkg.PropagatorSpec(F, fdt, fs), pkg.PropagatorSpec(G, gdt, gs),
                                   short_circuit=False)
        s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
        # warm-up: one fine and one coarse slice (graphs, plans)
        pkg.propagate(pkg.PropagatorSpec(F, fdt, 2), s)
        pkg.propagate(pkg.PropagatorSpec(G, gdt, 2), s)
        torch.cuda.synchronize(dev)
        d.barrier()
        t0 = time.perf_counter()
        res = parallel.parareal_run(s, 8, cfg_p)
        counts = res.counts
        torch.cuda.synchronize(dev)
        d.barrier()
        dt = d.max(time.perf_counter() - t0)
        value = w.n * 8 * fs / dt
        steps = K
        gtxt = ("G simple cutoff a=8 (the paper's coarse propagator)" if args.workload == "parareal_cutoff"
                else "G a=8 h=5 l=3")
        cfg = {"workload": "configs[4] C5-S parareal: 2^20 charges (RSA 1.5 A), F a=12 h=2.5 l=4 dt 0.005 fs x100, "
                           f"{gtxt} dt 0.02 fs x25, 8 slices, K iterations",
               "n_atoms": int(w.n), "K": K, "parallelism": f"parareal fine slices over {d.world} GPU(s)",
               "counts": counts}
        extra = {"ms_per_run": 1e3 * dt}
    if d.rank == 0:
        out = {"metric": metric, "value": value, "unit": unit, "n_gpus": d.world, "steps": steps,
               "warmup": args.warmup, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
               "config": cfg, "gpu_launches": None, "workload_path": args.workload}
        out.update(extra)
        print(json.dumps(out), flush=True)
