"""Velocity Verlet and parareal on the GPU against the reference (P2 protocol,
SURVEY 8d): survivable variants, positions within 1e-8 relative RMS."""
import numpy as np
import pytest

from conftest import golden, rel_rms
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx

pytestmark = pytest.mark.gpu


def test_trajectory_vs_reference_golden():
    g = golden("c1s_traj10")
    f = pkg.MsmField(pkg.MsmConfig(float(g["a"]), float(g["h"]), int(g["levels"])))
    s = pkg.ParticleSystem(g["pos"], g["vel"], g["q"], g["mass"], g["box"])
    out = pkg.propagate(pkg.PropagatorSpec(f, float(g["dt"]), int(g["steps"])), s)
    assert rel_rms(out.positions, g["out_pos"]) <= 1e-8
    assert rel_rms(out.velocities, g["out_vel"]) <= 1e-8


def test_c1s_full_trajectory_vs_oracle(port):
    w = fx.config("c1s")
    steps = 60
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    out = pkg.propagate(pkg.PropagatorSpec(f, w.dt, steps), pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
    p, v, done, err = port.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, steps)
    assert err is None
    assert rel_rms(out.positions, p) <= 1e-8 and rel_rms(out.velocities, v) <= 1e-8


def test_water_trajectory_vs_oracle(port):
    w = fx.config("c2s", n_override=30000)
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    out = pkg.propagate(pkg.PropagatorSpec(f, w.dt, 8), s)
    p, v, done, err = port.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, 8)
    assert err is None
    assert rel_rms(out.positions, p) <= 1e-8 and rel_rms(out.velocities, v) <= 1e-8


def test_device_resident_equals_host_path_and_is_deterministic():
    w = fx.config("c2s", n_override=30000)
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    a = pkg.propagate(pkg.PropagatorSpec(f, w.dt, 5), s)
    dev = pkg.DeviceSystem(f, s)
    dev.propagate(w.dt, 5)
    p, v = dev.download()
    assert np.array_equal(p, a.positions) and np.array_equal(v, a.velocities)
    dev2 = pkg.DeviceSystem(f, s)
    dev2.propagate(w.dt, 2)
    dev2.propagate(w.dt, 3)
    # two calls = 5 steps with one extra initial evaluation.  The second call rebuilds
    # the pair list at step 2, the single call reuses it (skin), so the summation order
    # and the last bits differ ...
    p2, v2 = dev2.download()
    assert rel_rms(p2, p) <= 1e-14 and rel_rms(v2, v) <= 1e-12
    # ... and with skin 0 (rebuild every evaluation) forces are pure: bit-identical
    g = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    g.set_pair_skin(0.0)
    d1 = pkg.DeviceSystem(g, s)
    d1.propagate(w.dt, 5)
    d2 = pkg.DeviceSystem(g, s)
    d2.propagate(w.dt, 2)
    d2.propagate(w.dt, 3)
    (q1, u1), (q2, u2) = d1.download(), d2.download()
    assert np.array_equal(q1, q2) and np.array_equal(u1, u2)


def test_verlet_step_and_energy_report(port):
    w = fx.config("c1s", n_override=2000)
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    s1 = pkg.verlet_step(s, f, w.dt)
    p, v, _, _ = port.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, 1)
    assert rel_rms(s1.positions, p) <= 1e-12
    rep = pkg.energy_report(s, f)
    o = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels)
    assert abs(rep.potential - o["energy"]) <= 1e-10 * abs(o["energy"])
    ke = sum(0.5 * w.mass[i] * np.dot(w.vel[i], w.vel[i]) for i in range(w.n)) / 4.184e-4
    assert abs(rep.kinetic - ke) <= 1e-12 * ke


def test_parareal_window_vs_reference_golden():
    g = golden("parareal_w4k2")
    fa, fh, fl, fdt, fs = g["fine"]
    ga, gh, gl, gdt, gs = g["coarse"]
    F = pkg.MsmField(pkg.MsmConfig(fa, fh, int(fl)))
    G = pkg.MsmField(pkg.MsmConfig(ga, gh, int(gl)))
    cfg = pkg.PararealConfig(4, 2, 1e300, pkg.PropagatorSpec(F, fdt, int(fs)), pkg.PropagatorSpec(G, gdt, int(gs)))
    s = pkg.ParticleSystem(g["pos"], g["vel"], g["q"], g["mass"], g["box"])
    row, dr, cnt = pkg.parareal_window(s, cfg, 4, 2)
    gp = np.stack([r.positions for r in row])
    assert rel_rms(gp, g["row_pos"]) <= 1e-8
    assert [cnt["g_evals"], cnt["f_evals"], cnt["f_skipped"]] == list(g["counts"])


@pytest.mark.parametrize("k", [1, 2, 3])
def test_parareal_scaled_c5_vs_oracle(port, k):
    """SURVEY 6 scaled config-5 fixture: N=2048, 0.1 atoms/A^3, RSA 1.5 A, F a=12 h=2.5 l=3
    dt .005 x100, G a=8 h=5 l=2 dt .02 x25, T=8."""
    L = 27.4
    box = np.array([L, L, L])
    pos, q = fx.uniform(2048, box, "random_neutral", 1.5, 77)
    mass = np.full(2048, 18.0)
    vel = fx.maxwell_boltzmann(mass, 300.0, 78)
    fine, coarse = (12.0, 2.5, 3, 0.005, 100), (8.0, 5.0, 2, 0.02, 25)
    F = pkg.MsmField(pkg.MsmConfig(12.0, 2.5, 3))
    G = pkg.MsmField(pkg.MsmConfig(8.0, 5.0, 2))
    cfg = pkg.PararealConfig(8, k, 1e300, pkg.PropagatorSpec(F, 0.005, 100), pkg.PropagatorSpec(G, 0.02, 25))
    row, dr, cnt = pkg.parareal_window(pkg.ParticleSystem(pos, vel, q, mass, box), cfg, 8, k)
    rp, rv, drr, cnt2 = port.parareal_window(pos, vel, q, mass, box, fine, coarse, 8, k)
    gp = np.stack([r.positions for r in row])
    assert rel_rms(gp, rp) <= 1e-8
    assert [cnt["g_evals"], cnt["f_evals"], cnt["f_skipped"]] == list(cnt2)
    # counts: G = T(K+1)-1, F = T*K (src/parareal.cpp:167-168)
    assert cnt["g_evals"] == 8 * (k + 1) - 1 and cnt["f_evals"] == 8 * k


def test_parareal_run_convergence_vs_oracle(port):
    box = np.array([14.0, 14.0, 14.0])
    pos, q = fx.uniform(256, box, "random_neutral", 1.5, 5)
    mass = np.full(256, 18.0)
    vel = fx.maxwell_boltzmann(mass, 300.0, 6)
    fine, coarse = (8.0, 2.0, 2, 0.005, 8), (6.0, 3.0, 2, 0.02, 2)
    F = pkg.MsmField(pkg.MsmConfig(8.0, 2.0, 2))
    G = pkg.MsmField(pkg.MsmConfig(6.0, 3.0, 2))
    cfg = pkg.PararealConfig(3, 4, 1e-7, pkg.PropagatorSpec(F, 0.005, 8), pkg.PropagatorSpec(G, 0.02, 2),
                             skip_threshold=1e-9)
    res = pkg.parareal_run(pkg.ParticleSystem(pos, vel, q, mass, box), 7, cfg)
    tp, tv, cnt, err = port.parareal_run(pos, vel, q, mass, box, fine, coarse, 3, 4, 1e-7, 7, skip_threshold=1e-9)
    assert err is None and res.converged
    assert rel_rms(np.stack([t.positions for t in res.trajectory]), tp) <= 1e-8
    assert [res.counts["g_evals"], res.counts["f_evals"], res.counts["f_skipped"], res.windows] == list(cnt[:4])


def test_parareal_config_validation():
    F = pkg.MsmField(pkg.MsmConfig(8.0, 2.0, 2))
    s = pkg.ParticleSystem([[1.0, 1, 1], [4.0, 4, 4]], None, [1.0, -1.0], [1.0, 1.0], [10.0] * 3)
    cfg = pkg.PararealConfig(2, 1, 1e-6, pkg.PropagatorSpec(F, 0.5, 4), pkg.PropagatorSpec(F, 1.0, 3))
    with pytest.raises(pkg.ConfigError, match="span different slice lengths"):
        pkg.parareal_window(s, cfg, 2, 1)


def test_pair_list_rebuilds_mid_trajectory(port):
    # a tiny skin makes the displacement check trigger several rebuilds inside one
    # propagate (graph-captured steps); the trajectory must still match the oracle,
    # and a skin-0 run (rebuild every evaluation) to rounding
    w = fx.config("c1s", n_override=2000)
    dt, steps = 0.05, 40
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    runs = {}
    for skin in (0.002, 0.0):
        f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
        f.set_pair_skin(skin)
        ds = pkg.DeviceSystem(f, s)
        ds.propagate(dt, steps)
        runs[skin] = (ds.download(), f.work_counters()["list_rebuilds"])
    (p1, v1), nreb = runs[0.002]
    (p0, v0), nreb0 = runs[0.0]
    assert 2 < nreb < steps + 1       # rebuilt more than once, but not at every evaluation
    assert nreb0 == steps + 1         # skin 0: every evaluation
    assert rel_rms(p1, p0) <= 1e-13 and rel_rms(v1, v0) <= 1e-11
    pp, vv, done, err = port.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, dt, steps)
    assert err is None and done == steps
    assert rel_rms(p1, pp) <= 1e-8 and rel_rms(v1, vv) <= 1e-8


def test_pair_list_per_call_and_reuse_opt_in(port):
    """Every evaluate / propagate call starts from a fresh pair list, so its results are
    a pure function of its input (bitwise repeatable, whatever ran before on the field);
    msmb_set_list_reuse opts into carrying a still-valid list across calls."""
    w = fx.config("c1s", n_override=3000)
    cfg = pkg.MsmConfig(w.a, w.h, w.levels)
    a = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    far = w.pos.copy()
    far[:, 0] = w.box[0] - far[:, 0]          # mirrored copy: every atom moved
    b = pkg.ParticleSystem(far, w.vel, w.q, w.mass, w.box)
    f = pkg.MsmField(cfg)
    ra = f.evaluate(a)
    assert f.work_counters()["list_rebuilds"] == 1
    rb = f.evaluate(b)
    ra2 = f.evaluate(a)
    assert f.work_counters()["list_rebuilds"] == 3
    assert np.array_equal(ra2.per_particle_force, ra.per_particle_force)   # bit-identical
    assert ra2.total_energy == ra.total_energy
    fb = pkg.MsmField(cfg).evaluate(b)        # a fresh field agrees bit for bit
    assert np.array_equal(fb.per_particle_force, rb.per_particle_force)
    o = port.msm_potential(far, w.q, w.box, w.a, w.h, w.levels)
    assert abs(rb.total_energy - o["energy"]) <= 1e-10 * abs(o["energy"])
    # opt-in reuse: same positions, no rebuild; a propagate call continues from the list
    f.set_list_reuse(True)
    f.evaluate(a)
    n0 = f.work_counters()["list_rebuilds"]
    f.evaluate(a)
    assert f.work_counters()["list_rebuilds"] == n0
    ds = pkg.DeviceSystem(f, a)
    ds.propagate(w.dt, 3)
    n1 = f.work_counters()["list_rebuilds"]
    ds.propagate(w.dt, 3)
    assert f.work_counters()["list_rebuilds"] == n1


def test_pair_list_invalidated_by_failed_evaluation():
    # a failed evaluation (coverage error) invalidates the list: the next one rebuilds
    w = fx.config("c1s", n_override=2000)
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    f.set_list_reuse(True)                    # (without reuse every call rebuilds anyway)
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    r0 = f.evaluate(s)
    bad = w.pos.copy()
    bad[7] = [1e3, 1e3, 1e3]                  # outside grid coverage
    with pytest.raises(pkg.CoverageError):
        f.evaluate(pkg.ParticleSystem(bad, w.vel, w.q, w.mass, w.box))
    r1 = f.evaluate(s)                        # rebuilt from s: the first result, bit for bit
    assert np.array_equal(r1.per_particle_force, r0.per_particle_force)
    n1 = f.work_counters()["list_rebuilds"]
    f.evaluate(s)                             # and valid again afterwards
    assert f.work_counters()["list_rebuilds"] == n1
