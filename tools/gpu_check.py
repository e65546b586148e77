"""Exploratory GPU check (not a test): parity vs the CPU oracle, stage bitwise
checks, error reproduction and first timings.  Prints one line per item."""
import sys
import time
import traceback
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1309_1889_b200 as pkg  # noqa: E402
from paper_1309_1889_b200 import fixtures as fx  # noqa: E402
import oracle_lib  # noqa: E402

port = oracle_lib.checker("port")
only = sys.argv[1:] or None


def section(name):
    def deco(fn):
        if only and name not in only:
            return fn
        t = time.time()
        try:
            fn()
            print(f"[{name}] done in {time.time() - t:.1f}s", flush=True)
        except Exception:
            print(f"[{name}] FAILED\n{traceback.format_exc()}", flush=True)
        return fn
    return deco


def rel(a, b):
    return float(np.sqrt(np.sum((a - b) ** 2) / max(np.sum(b ** 2), 1e-300)))


@section("smoke")
def _():
    import __graft_entry__ as g
    g.smoke()


@section("parity")
def _():
    for name, nov in [("c1", None), ("c1s", None), ("c2", 30000), ("c5", 20000), ("c3", 20000), ("c4", 30000)]:
        w = fx.config(name, n_override=nov)
        f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
        s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
        t = time.time()
        r = f.evaluate(s)
        tg = time.time() - t
        t = time.time()
        o = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels)
        to = time.time() - t
        r2 = f.evaluate(s)
        det = np.array_equal(r.per_particle_force, r2.per_particle_force) and r.total_energy == r2.total_energy
        print(f"  {name} N={w.n} E={r.total_energy:.10e} dE/E={abs(r.total_energy - o['energy']) / abs(o['energy']):.2e}"
              f" dF={rel(r.per_particle_force, o['force']):.2e} dphi={rel(r.per_particle_potential, o['phi']):.2e}"
              f" dphis={rel(r.short_part, o['phi_short']):.2e} dphil={rel(r.long_part, o['phi_long']):.2e}"
              f" det={det} gpu {tg:.3f}s port {to:.2f}s counters={f.work_counters()}", flush=True)


@section("stages")
def _():
    for name, nov in [("c1", None), ("c2", 30000), ("c5", 20000)]:
        w = fx.config(name, n_override=nov)
        cfg = pkg.MsmConfig(w.a, w.h, w.levels)
        f = pkg.MsmField(cfg)
        o = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels, diag=True)
        dims, _, _ = pkg.grid_geometry(cfg, w.box)
        sizes = [int(np.prod(d)) for d in dims]
        offs = np.concatenate([[0], np.cumsum(sizes)])
        lc = [o["level_charge"][offs[k]:offs[k + 1]] for k in range(w.levels)]
        lp = [o["level_potential"][offs[k]:offs[k + 1]] for k in range(w.levels)]
        # anterpolation (full evaluation on GPU, then compare level 0 charge)
        s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
        f.evaluate(s)
        gc, gp = f.debug_levels()
        q0 = gc[:sizes[0]]
        print(f"  {name} anterp max|dq|/max|q| = {np.max(np.abs(q0 - lc[0])) / np.max(np.abs(lc[0])):.2e}")
        for k in range(w.levels - 1):
            rq = f.debug_stage(0, k, w.box, lc[k])
            ref = port.restrict(w.box, w.a, w.h, w.levels, k, lc[k])
            print(f"  {name} restrict {k}->{k+1} bitwise={np.array_equal(rq, ref)} maxrel={np.max(np.abs(rq-ref))/np.max(np.abs(ref)):.2e}")
            lat = f.debug_stage(1, k, w.box, lc[k])
            ref = port.lattice_cutoff(w.box, w.a, w.h, w.levels, k, lc[k])
            print(f"  {name} lattice {k} maxrel={np.max(np.abs(lat-ref))/np.max(np.abs(ref)):.2e} bitwise={np.array_equal(lat, ref)}")
        t = w.levels - 1
        top = f.debug_stage(2, t, w.box, lc[t])
        ref = port.top_level(w.box, w.a, w.h, w.levels, lc[t])
        print(f"  {name} top maxrel={np.max(np.abs(top-ref))/np.max(np.abs(ref)):.2e} bitwise={np.array_equal(top, ref)}")
        for k in range(w.levels - 2, -1, -1):
            # fine potential before prolongation = lattice result of level k
            fine_in = port.lattice_cutoff(w.box, w.a, w.h, w.levels, k, lc[k])
            pr = f.debug_stage(3, k, w.box, lp[k + 1], out=fine_in)
            ref = port.prolongate(w.box, w.a, w.h, w.levels, k, lp[k + 1], fine_in)
            print(f"  {name} prolong {k+1}->{k} bitwise={np.array_equal(pr, ref)}")
        u = f.debug_stage(4, 0, w.box, lp[0], positions=w.pos)
        ref = port.interpolate(w.pos, w.box, w.a, w.h, w.levels, lp[0])
        print(f"  {name} interp bitwise={np.array_equal(u, ref)}")
        cells, cov = f.debug_cells(w.pos, w.box)
        dims0, _, org = pkg.grid_geometry(cfg, w.box)
        t = (w.pos - org[0]) * (1.0 / w.h)
        exp = np.floor(t).astype(np.int64)
        print(f"  {name} cells bitwise={np.array_equal(cells, exp)} covered_all={cov.all()}")


@section("errors")
def _():
    w = fx.config("c1s")
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    cases = []
    p = w.pos.copy(); p[100] = p[7]; p[50] = p[20]; cases.append(("coincident", p))
    p = w.pos.copy(); p[300, 1] = np.nan; p[200, 0] = -5; cases.append(("nan", p))
    p = w.pos.copy(); p[300, 1] = -2.6; p[200, 0] = 42.5; p[250, 2] = -2.5; cases.append(("coverage", p))
    p = w.pos.copy(); p[300, 1] = np.inf; p[200, 1] = np.inf; cases.append(("inf", p))
    for name, p in cases:
        try:
            port.msm_potential(p, w.q, w.box, w.a, w.h, w.levels)
            exp = "ok"
        except oracle_lib.OracleError as e:
            exp = f"{e.kind}: {e.msg}"
        try:
            f.evaluate(pkg.ParticleSystem(p, w.vel, w.q, w.mass, w.box))
            got = "ok"
        except pkg.Error as e:
            got = f"{type(e).__name__}: {e}"
        print(f"  {name}: oracle[{exp}] gpu[{got}] match={exp == got}")
    # literal c1 trajectory abort
    w = fx.config("c1")
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    try:
        pkg.propagate(pkg.PropagatorSpec(f, w.dt, 200), s)
        got = "ok"
    except pkg.Error as e:
        got = f"{type(e).__name__}: {e} step={e.step}"
    _, _, done, err = port.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, 200)
    print(f"  c1 literal: gpu[{got}] oracle[{err} after {done} steps]")


@section("trajectory")
def _():
    w = fx.config("c1s")
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    steps = 20
    t = time.time()
    out = pkg.propagate(pkg.PropagatorSpec(f, w.dt, steps), s)
    tg = time.time() - t
    t = time.time()
    p2, v2, done, err = port.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, steps)
    to = time.time() - t
    print(f"  c1s {steps} steps: dx={rel(out.positions, p2):.2e} dv={rel(out.velocities, v2):.2e} gpu {tg:.2f}s port {to:.2f}s")


@section("parareal")
def _():
    w = fx.config("c5", n_override=2048)
    # scaled survivable fixture: F a=12 h=2.5 l=3 dt .005 x100, G a=8 h=5 l=2 dt .02 x25
    p, q = fx.uniform(2048, w.box, "random_neutral", 1.5, 77)
    mass = np.full(2048, 18.0)
    vel = fx.maxwell_boltzmann(mass, 300.0, 78)
    fine = (12.0, 2.5, 3, 0.005, 100)
    coarse = (8.0, 5.0, 2, 0.02, 25)
    F = pkg.MsmField(pkg.MsmConfig(12.0, 2.5, 3))
    G = pkg.MsmField(pkg.MsmConfig(8.0, 5.0, 2))
    cfg = pkg.PararealConfig(8, 2, 1e300, pkg.PropagatorSpec(F, 0.005, 100), pkg.PropagatorSpec(G, 0.02, 25))
    s = pkg.ParticleSystem(p, vel, q, mass, w.box)
    t = time.time()
    row, dr, cnt = pkg.parareal_window(s, cfg, 8, 2)
    tg = time.time() - t
    t = time.time()
    rp, rv, drr, cnt2 = port.parareal_window(p, vel, q, mass, w.box, fine, coarse, 8, 2)
    to = time.time() - t
    gp = np.stack([r.positions for r in row])
    print(f"  parareal K=2: dx={rel(gp, rp):.2e} counts gpu={cnt} port={list(cnt2)} gpu {tg:.2f}s port {to:.2f}s")


@section("timing")
def _():
    for name in ["c2s", "c1s", "c5"]:
        w = fx.config(name)
        f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
        s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
        dev = pkg.DeviceSystem(f, s)
        dt = w.dt if name != "c5" else 0.5
        dev.propagate(dt, 2)  # warm-up + capture
        steps = 10
        t = time.time()
        dev.propagate(dt, steps)
        el = time.time() - t
        f.set_stage_timing(True)
        f.reset_stage_times()
        dev.propagate(dt, steps)
        st = f.stage_times()
        f.set_stage_timing(False)
        tot = sum(v[0] for v in st.values())
        print(f"  {name} N={w.n}: {1e3 * el / (steps + 1):.3f} ms/eval (graph, wall) -> "
              f"{w.n * steps / el:.3e} atom-steps/s; counters={f.work_counters()}")
        print("    stages(ms/eval): " + ", ".join(f"{k}={v[0] / (steps + 1):.3f}" for k, v in st.items())
              + f" total={tot / (steps + 1):.3f}")
