"""Command-line front end over the B200 fields: the reference CLI's
subcommands on this path -- gen, simulate, compare, parareal (tools/paramd_main.cpp) --
with its options, defaults, output files (CSV columns, extended-XYZ frames) and exit
codes (0 ok, 2 configuration/input error, 3 runtime error, 4 non-convergence), every
force evaluation on the GPU.  The cost-model and scheduler subcommands are not on the
path (out of scope).

    python -m paper_1309_1889_b200 simulate --input system.xyz --force-field msm ...

Differences by design: `simulate` propagates device-resident between the logging and
trajectory points (the reference calls verlet_step per step; the trajectory is the
same up to rounding) and checks finiteness at those points, rescanning the last
interval step by step to report the first non-finite step as the reference does.
"""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

from . import (ConfigError, CutoffParams, DeviceSystem, DirectCoulombField,
               MsmConfig, MsmField, NonConvergenceError, PairRepulsionOverlay, ParticleSystem,
               PararealConfig, PropagatorSpec, RuntimeFault, SimpleCutoffField, UnitsConfig, WolfField,
               energy_report)
from .xyz_io import CsvWriter, ParseError, TrajectoryWriter, csv_num, load_system, save_system


class _Common:
    def __init__(self, a):
        self.seed, self.threads, self.out_dir, self.units = a.seed, a.threads, a.out_dir, a.units

    def units_config(self) -> UnitsConfig:  # paramd_main.cpp:36-40
        if self.units == "physical":
            return UnitsConfig.physical()
        if self.units == "reduced":
            return UnitsConfig.reduced()
        raise ConfigError(f"unknown units preset '{self.units}'")

    def out(self, name: str) -> str:
        os.makedirs(self.out_dir, exist_ok=True)
        return os.path.join(self.out_dir, name)


def _field_flags(p):  # FieldOpts::add_flags, paramd_main.cpp:55-67
    p.add_argument("--cutoff", type=float, default=12.0)
    p.add_argument("--wolf-alpha", type=float, default=0.2)
    p.add_argument("--a", dest="msm_a", type=float, default=8.0)
    p.add_argument("--h", dest="msm_h", type=float, default=2.0)
    p.add_argument("--levels", dest="msm_levels", type=int, default=2)
    p.add_argument("--repulsion-eps", type=float, default=0.0)
    p.add_argument("--repulsion-sigma", type=float, default=1.0)


def build_field(a, kind: str, units: UnitsConfig):
    """FieldOpts::build (paramd_main.cpp:69-91), GPU fields."""
    if kind == "direct":
        ff = DirectCoulombField(units)
    elif kind == "cutoff":
        ff = SimpleCutoffField(CutoffParams(a.cutoff, None), units)
    elif kind == "wolf":
        ff = WolfField(CutoffParams(a.cutoff, a.wolf_alpha), units)
    elif kind == "msm":
        ff = MsmField(MsmConfig(a.msm_a, a.msm_h, a.msm_levels), units)
    else:
        raise ConfigError(f"unknown force field '{kind}'")
    if a.repulsion_eps > 0.0:
        ff = PairRepulsionOverlay(ff, a.repulsion_eps, a.repulsion_sigma)
    return ff


def _check_finite(s: ParticleSystem, step: int):  # paramd_main.cpp:94-99
    bad = ~(np.isfinite(s.positions).all(axis=1) & np.isfinite(s.velocities).all(axis=1))
    if bad.any():
        raise RuntimeFault(f"non-finite state at step {step}, particle {int(np.argmax(bad))}")


def cmd_gen(c: _Common, a) -> int:  # paramd_main.cpp:100-115
    from . import fixtures
    box = a.box
    if len(box) == 1:
        box = [box[0]] * 3
    elif len(box) != 3:
        raise ConfigError("--box takes 1 or 3 values")
    schemes = ("all_plus_one", "alternating", "random_neutral")
    if a.scheme not in schemes:
        raise ConfigError(f"unknown charge scheme '{a.scheme}'")
    if a.n < 1:
        raise ConfigError("generate_random_system: n must be >= 1")
    if a.min_sep < 0.0:
        raise ConfigError("generate_random_system: min_separation < 0")
    if not all(b > 0.0 for b in box):
        raise ConfigError("generate_random_system: box extents must be positive")
    pos, q = fixtures.uniform(a.n, np.array(box, dtype=np.float64), a.scheme, a.min_sep, c.seed)
    s = ParticleSystem(pos, np.zeros((a.n, 3)), q, np.ones(a.n), np.array(box, dtype=np.float64))
    save_system(s, a.out)
    print(f"wrote {s.size()} particles to {a.out}")
    return 0


def cmd_simulate(c: _Common, a) -> int:  # paramd_main.cpp:117-146
    units = c.units_config()
    ff = build_field(a, a.force_field, units)
    if a.steps < 0:
        raise ConfigError("--steps must be >= 0")
    if not (a.dt > 0.0):
        raise ConfigError("--dt must be > 0")
    if a.log_every < 1 or a.traj_every < 1:
        raise ConfigError("logging intervals must be >= 1")
    s = load_system(a.input)
    kind = a.force_field
    energy = CsvWriter(c.out(kind + "_energy.csv"))
    energy.row(["step", "time_fs", "kinetic", "potential", "total"])
    traj = TrajectoryWriter(c.out(kind + "_trajectory.xyz"))
    dev = DeviceSystem(ff, s)

    def log_state(step, st):
        rep = energy_report(st, ff, units)
        energy.row([str(step), csv_num(step * a.dt), csv_num(rep.kinetic), csv_num(rep.potential),
                    csv_num(rep.total)])

    log_state(0, s)
    traj.write_frame(s, 0, 0.0)
    step = 0
    while step < a.steps:
        # next step that logs or writes a frame (or the last step)
        nxt = min(a.steps, (step // a.log_every + 1) * a.log_every, (step // a.traj_every + 1) * a.traj_every)
        start = dev.download()
        dev.propagate(a.dt, nxt - step)
        pos, vel = dev.download()
        cur = ParticleSystem(pos, vel, s.charges, s.masses, s.box)
        if not (np.isfinite(pos).all() and np.isfinite(vel).all()):
            # first non-finite step of the interval, as the per-step check would report it
            dev.upload(*start)
            for k in range(step + 1, nxt + 1):
                dev.propagate(a.dt, 1)
                p2, v2 = dev.download()
                _check_finite(ParticleSystem(p2, v2, s.charges, s.masses, s.box), k)
        step = nxt
        if step % a.log_every == 0 or step == a.steps:
            log_state(step, cur)
        if step % a.traj_every == 0 or step == a.steps:
            traj.write_frame(cur, step, step * a.dt)
    print(f"simulated {a.steps} steps with {ff.name()}")
    return 0


def cmd_compare(c: _Common, a) -> int:  # paramd_main.cpp:148-212
    units = c.units_config()
    s = load_system(a.input)
    ref = DirectCoulombField(units).evaluate(s)
    per = CsvWriter(c.out("compare.csv"))
    per.row(["field", "index", "u_ref", "u_test", "u_rel_err", "f_rel_err"])
    summary = CsvWriter(c.out("compare_summary.csv"))
    summary.row(["field", "energy_ref", "energy_test", "energy_rel_err", "potential_rms_rel_err",
                 "force_rms_rel_err"])
    u_scale = float(np.max(np.abs(ref.per_particle_potential))) if s.size() else 0.0
    f_scale = float(np.max(np.sqrt((ref.per_particle_force ** 2).sum(axis=1)))) if s.size() else 0.0
    u_scale = u_scale or 1.0
    f_scale = f_scale or 1.0
    for kind in a.fields:
        ff = build_field(a, kind, units)
        got = ff.evaluate(s)
        if kind == "msm" and a.dump_grids and isinstance(ff, MsmField):
            from . import grid_geometry
            dims, _, _ = grid_geometry(ff.config(), s.box)
            qc, qp = ff.debug_levels()
            off = 0
            for lvl, d in enumerate(dims):
                size = int(np.prod(d))
                grid = CsvWriter(c.out(f"grid_level_{lvl}.csv"))
                grid.row(["i", "j", "k", "charge", "potential"])
                ch = qc[off:off + size].reshape(d)
                po = qp[off:off + size].reshape(d)
                for i in range(d[0]):
                    for j in range(d[1]):
                        for k in range(d[2]):
                            grid.row([str(i), str(j), str(k), csv_num(ch[i, j, k]), csv_num(po[i, j, k])])
                grid.close()
                off += size
        du = got.per_particle_potential - ref.per_particle_potential
        df = got.per_particle_force - ref.per_particle_force
        for i in range(s.size()):
            per.row([kind, str(i), csv_num(ref.per_particle_potential[i]), csv_num(got.per_particle_potential[i]),
                      csv_num(abs(du[i]) / u_scale), csv_num(math.sqrt(float(df[i] @ df[i])) / f_scale)])
        e_rel = abs(got.total_energy - ref.total_energy) / max(1e-300, abs(ref.total_energy))
        u2 = float(ref.per_particle_potential @ ref.per_particle_potential)
        f2 = float((ref.per_particle_force ** 2).sum())
        summary.row([kind, csv_num(ref.total_energy), csv_num(got.total_energy), csv_num(e_rel),
                     csv_num(math.sqrt(float(du @ du) / max(1e-300, u2))),
                     csv_num(math.sqrt(float((df ** 2).sum()) / max(1e-300, f2)))])
        print(f"{kind}: total energy rel err {e_rel:g}")
    return 0


def cmd_parareal(c: _Common, a) -> int:  # paramd_main.cpp:214-286
    from . import parallel
    units = c.units_config()
    v = load_system(a.input)
    cfg = PararealConfig(window_points=a.window, max_iter=a.max_iter, tol=a.tol,
                         fine=PropagatorSpec(build_field(a, a.fine, units), a.dt, a.steps_per_slice),
                         coarse=PropagatorSpec(build_field(a, a.coarse, units), a.dt, a.steps_per_slice),
                         units=units, skip_threshold=a.skip_threshold if a.skip_threshold >= 0.0 else None,
                         short_circuit=not a.no_short_circuit)

    def write_report(rows, counts, windows):
        conv = CsvWriter(c.out("convergence.csv"))
        conv.row(["window", "point", "iteration", "delta_rms", "converged"])
        for w, p, k, d, ok in rows:
            conv.row([str(w), str(p), str(k), csv_num(d), "1" if ok else "0"])
        ev = CsvWriter(c.out("evals.csv"))
        ev.row(["counter", "value"])
        for key in ("g_evals", "f_evals", "f_skipped"):
            ev.row([key, str(counts[key])])
        ev.row(["windows", str(windows)])

    try:
        r = parallel.parareal_run(v, a.points, cfg)
    except NonConvergenceError as e:
        rep = getattr(e, "report", None) or dict(rows=[], counts=dict(g_evals=0, f_evals=0, f_skipped=0), windows=0)
        write_report(rep["rows"], rep["counts"], rep["windows"])
        print(f"parareal: {e}", file=sys.stderr)
        return 4
    write_report(r.report_rows, r.counts, r.windows)
    traj = TrajectoryWriter(c.out("parareal_trajectory.xyz"))
    span = cfg.fine.slice_span()
    for n, st in enumerate(r.trajectory):
        traj.write_frame(st, n + 1, (n + 1) * span)
    if a.verify:
        from . import propagate
        ver = CsvWriter(c.out("verify.csv"))
        ver.row(["point", "rms_vs_fine"])
        ref = v
        worst = 0.0
        for n, st in enumerate(r.trajectory):
            ref = propagate(cfg.fine, ref, units)
            d = st.positions - ref.positions
            rms = math.sqrt(float((d ** 2).sum()) / (3.0 * v.size()))  # state_sub rms_pos
            ver.row([str(n + 1), csv_num(rms)])
            worst = max(worst, rms)
        print(f"verify: max RMS deviation from sequential fine run = {worst:g}")
    print(f"parareal: {a.points} points in {r.windows} windows, F evals {r.counts['f_evals']}, "
          f"G evals {r.counts['g_evals']}, skipped {r.counts['f_skipped']}")
    return 0


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1309_1889_b200",
                                 description="molecular dynamics with multilevel summation and parareal "
                                             "time stepping (B200 fields)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--out-dir", default=".")
    ap.add_argument("--units", default="physical")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen")
    g.add_argument("--n", type=int, default=32)
    g.add_argument("--box", type=float, nargs="+", default=[20.0])
    g.add_argument("--scheme", default="all_plus_one")
    g.add_argument("--min-sep", type=float, default=1.0)
    g.add_argument("--out", default="system.xyz")
    s = sub.add_parser("simulate")
    _field_flags(s)
    s.add_argument("--input", required=True)
    s.add_argument("--force-field", default="direct")
    s.add_argument("--steps", type=int, default=100)
    s.add_argument("--dt", type=float, default=0.5)
    s.add_argument("--log-every", type=int, default=1)
    s.add_argument("--traj-every", type=int, default=10)
    m = sub.add_parser("compare")
    _field_flags(m)
    m.add_argument("--input", required=True)
    m.add_argument("--fields", nargs="+", default=["msm", "cutoff", "wolf"])
    m.add_argument("--dump-grids", action="store_true")
    p = sub.add_parser("parareal")
    _field_flags(p)
    p.add_argument("--input", required=True)
    p.add_argument("--fine", default="msm")
    p.add_argument("--coarse", default="cutoff")
    p.add_argument("--dt", type=float, default=0.02)
    p.add_argument("--steps-per-slice", type=int, default=5)
    p.add_argument("--window", type=int, default=8)
    p.add_argument("--max-iter", type=int, default=5)
    p.add_argument("--tol", type=float, default=1e-6)
    p.add_argument("--points", type=int, default=8)
    p.add_argument("--verify", action="store_true")
    p.add_argument("--skip-threshold", type=float, default=-1.0)
    p.add_argument("--no-short-circuit", action="store_true")
    return ap


def main(argv=None) -> int:
    ap = parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # CLI11 parse errors exit 2 (paramd_main.cpp:470-478)
        return int(e.code or 0) and 2
    c = _Common(a)
    cmds = dict(gen=cmd_gen, simulate=cmd_simulate, compare=cmd_compare, parareal=cmd_parareal)
    try:
        return cmds[a.cmd](c, a)
    except ConfigError as e:  # paramd_main.cpp:490-500
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except ParseError as e:
        print(f"input error: {e}", file=sys.stderr)
        return 2
    except Exception as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
