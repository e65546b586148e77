"""Pair-only GPU fields: SimpleCutoffField and WolfField on
the sm_100a pair path (msmb_create_cutoff), against the reference's goldens
(tests/golden/fields*.npz, written by the reference itself) and the bitwise C
restatement (oracle/).  Tolerances are BASELINE.json's: energy 1e-10 relative,
RMS force 1e-8 relative; per-atom potentials 1e-12 RMS relative."""
import numpy as np
import pytest

from conftest import golden, rel_e, rel_rms
from oracle_lib import fspec
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx

pytestmark = pytest.mark.gpu

E_TOL, F_TOL, P_TOL = 1e-10, 1e-8, 1e-12


def gpu_field(spec, units=None):
    kind, a, alpha = int(spec[0]), float(spec[1]), (float(spec[5]) if spec[4] else None)
    cls = {1: pkg.SimpleCutoffField, 2: pkg.WolfField}[kind]
    return cls(pkg.CutoffParams(a, alpha), units or pkg.UnitsConfig.physical())


def check(r, o):
    assert rel_e(r.total_energy, o["energy"]) <= E_TOL
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL
    assert rel_rms(r.per_particle_potential, o["phi"]) <= P_TOL


@pytest.mark.parametrize("name", ["cutoff10", "cutoff7", "wolf10", "wolf8_a0"])
def test_golden(name):
    g = golden("fields")
    spec = g["specs"][list(g["names"]).index(name)]
    f = gpu_field(spec)
    r = f.evaluate(pkg.ParticleSystem(g["pos"], None, g["q"], None, g["box"]))
    check(r, dict(energy=float(g[f"{name}_energy"]), force=g[f"{name}_force"], phi=g[f"{name}_phi"]))
    assert r.short_part is None and r.long_part is None  # as the reference's make_result


@pytest.mark.parametrize("name,n,spec", [
    ("c1", None, fspec("cutoff", 10.0)), ("c1", None, fspec("wolf", 10.0, alpha=0.2)),
    ("c2", 20000, fspec("cutoff", 12.0)), ("c2", 20000, fspec("wolf", 12.0, alpha=0.25)),
    ("c5", 20000, fspec("cutoff", 8.0)), ("c4", 20000, fspec("wolf", 9.0, alpha=0.3)),
])
def test_config_shapes_vs_oracle(port, name, n, spec):
    w = fx.config(name, n_override=n)
    f = gpu_field(spec)
    r = f.evaluate(pkg.ParticleSystem(w.pos, None, w.q, None, w.box))
    check(r, port.field_evaluate(spec, w.pos, w.q, w.box))
    wc = f.work_counters()
    assert wc["pairs"] > 0 and wc["lattice_taps"] == 0


@pytest.mark.parametrize("spec", [fspec("cutoff", 6.0), fspec("wolf", 6.0, alpha=0.3)])
def test_atoms_outside_the_box(port, spec):
    # the reference's cutoff fields ignore the box; here it only sets the binning
    # extent and atoms outside it are clamped into the boundary cells
    rng = np.random.default_rng(3)
    n, L = 6000, 30.0
    pos = rng.uniform(0, L, (n, 3))
    pos[:300] = rng.uniform(-40.0, L + 40.0, (300, 3))          # near and far outside
    pos[300:310] = np.array([L + 100.0, -50.0, 7.0]) + rng.uniform(0, 3.0, (10, 3))  # a far cluster
    q = rng.choice([-1.0, 1.0], n)
    box = np.array([L, L, L])
    r = gpu_field(spec).evaluate(pkg.ParticleSystem(pos, None, q, None, box))
    check(r, port.field_evaluate(spec, pos, q, box))


def test_coincident_pair_error():
    w = fx.config("c1", n_override=4000)
    pos = w.pos.copy()
    pos[2999] = pos[41]
    for spec in (fspec("cutoff", 10.0), fspec("wolf", 10.0, alpha=0.2)):
        with pytest.raises(pkg.CoincidentParticlesError) as ei:
            gpu_field(spec).evaluate(pkg.ParticleSystem(pos, None, w.q, None, w.box))
        assert str(ei.value) == "particles 41 and 2999 coincide"


def test_nan_and_inf_positions():
    w = fx.config("c1", n_override=2000)
    pos = w.pos.copy()
    pos[7, 1] = np.nan  # the reference: every pair with particle 7 is NaN -> all outputs NaN
    f = gpu_field(fspec("cutoff", 10.0))
    r = f.evaluate(pkg.ParticleSystem(pos, None, w.q, None, w.box))
    assert np.isnan(r.per_particle_potential).all() and np.isnan(r.per_particle_force).all()
    assert np.isnan(r.total_energy)
    pos = w.pos.copy()
    pos[11, 2] = np.inf
    with pytest.raises(pkg.DomainError, match="particle 11 has a non-finite position"):
        f.evaluate(pkg.ParticleSystem(pos, None, w.q, None, w.box))
    r = f.evaluate(pkg.ParticleSystem(w.pos, None, w.q, None, w.box))  # recovers
    assert np.isfinite(r.total_energy)


def test_trajectory_vs_reference_golden():
    g = golden("fields_traj10")
    f = gpu_field(g["spec"])
    s = pkg.ParticleSystem(g["pos"], g["vel"], g["q"], g["mass"], g["box"])
    out = pkg.propagate(pkg.PropagatorSpec(f, float(g["dt"]), int(g["steps"])), s)
    assert rel_rms(out.positions, g["out_pos"]) <= 1e-12
    assert rel_rms(out.velocities, g["out_vel"]) <= 1e-9


@pytest.mark.parametrize("spec", [fspec("cutoff", 10.0), fspec("wolf", 9.0, alpha=0.2)])
def test_trajectory_vs_oracle_with_list_reuse(port, spec):
    # 40 steps through the device-resident graph engine (Verlet-skin list reused
    # across steps and rebuilt after skin/2 moves) against the restatement
    w = fx.config("c1s", n_override=6000)
    f = gpu_field(spec)
    f.set_pair_skin(0.004)  # rebuilds every few steps at this dt
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    out = pkg.propagate(pkg.PropagatorSpec(f, 0.05, 40), s)
    assert f.work_counters()["list_rebuilds"] >= 3
    p2, v2, done, err = port.field_propagate(spec, w.pos, w.vel, w.q, w.mass, w.box, 0.05, 40)
    assert err is None and done == 40
    assert rel_rms(out.positions, p2) <= 1e-12
    assert rel_rms(out.velocities, v2) <= 1e-8


def test_parareal_msm_fine_cutoff_coarse_vs_reference_golden():
    # the CLI's default pairing (tools/paramd_main.cpp:417): fine MSM, coarse cutoff
    g = golden("fields_parareal_w4k2")
    fs, gs = g["fine"], g["coarse"]
    fine = pkg.MsmField(pkg.MsmConfig(float(fs[1]), float(fs[2]), int(fs[3])))
    coarse = gpu_field(gs)
    cfg = pkg.PararealConfig(window_points=int(g["t_points"]), max_iter=int(g["k_iters"]), tol=1e300,
                             fine=pkg.PropagatorSpec(fine, float(g["fdt"]), int(g["fsteps"])),
                             coarse=pkg.PropagatorSpec(coarse, float(g["gdt"]), int(g["gsteps"])),
                             short_circuit=False)
    v = pkg.ParticleSystem(g["pos"], g["vel"], g["q"], g["mass"], g["box"])
    row, dr, counts = pkg.parareal_window(v, cfg, int(g["t_points"]), int(g["k_iters"]))
    rp = np.stack([s.positions for s in row])
    assert rel_rms(rp, g["row_pos"]) <= 1e-8
    assert [counts["g_evals"], counts["f_evals"], counts["f_skipped"]] == list(g["counts"])


def test_cost_model_and_names(ref):
    import oracle_lib as ol
    for spec, cls, name in [(fspec("cutoff", 10.0), pkg.SimpleCutoffField, "cutoff"),
                            (fspec("wolf", 10.0, alpha=0.2), pkg.WolfField, "wolf")]:
        f = gpu_field(spec)
        assert isinstance(f, cls) and f.name() == name
        for n in (1, 8192, 300000):
            assert f.cost_flops_per_step(n) == ref.lib.ref_field_cost(ol._p(spec), 332.0636, 4.184e-4, n)
    f = pkg.SimpleCutoffField(pkg.CutoffParams(10.0), flops_per_particle=123.0)
    assert f.cost_flops_per_step(1000) == 123000.0


def test_msm_only_entry_points_refuse_pair_fields():
    f = gpu_field(fspec("cutoff", 10.0))
    with pytest.raises(pkg.ConfigError, match="needs an MSM field"):
        pkg.MsmField.set_lattice_method(f, True)


# ---- all-pairs fields: DirectCoulombField, PairRepulsionOverlay
def test_direct_golden_and_spec500():
    g = golden("fields")
    r = pkg.DirectCoulombField().evaluate(pkg.ParticleSystem(g["pos"], None, g["q"], None, g["box"]))
    check(r, dict(energy=float(g["direct_energy"]), force=g["direct_force"], phi=g["direct_phi"]))
    s5, d5 = golden("spec500"), golden("spec500_direct")
    r = pkg.direct_coulomb(pkg.ParticleSystem(s5["pos"], None, s5["q"], None, s5["box"]))
    check(r, dict(energy=float(d5["energy"]), force=d5["force"], phi=d5["phi"]))


@pytest.mark.parametrize("name", ["cutoff10_rep", "direct_rep"])
def test_overlay_golden(name):
    g = golden("fields")
    spec = g["specs"][list(g["names"]).index(name)]
    base = pkg.DirectCoulombField() if spec[0] == 3 else gpu_field(spec)
    f = pkg.PairRepulsionOverlay(base, float(spec[6]), float(spec[7]))
    s = pkg.ParticleSystem(g["pos"], None, g["q"], None, g["box"])
    r = f.evaluate(s)
    check(r, dict(energy=float(g[f"{name}_energy"]), force=g[f"{name}_force"], phi=g[f"{name}_phi"]))
    assert f.name() == base.name() + "+rep"
    assert f.cost_flops_per_step(1000) == base.cost_flops_per_step(1000) + 30000.0
    # the base field is unchanged by the overlay
    rb = base.evaluate(s)
    base_name = name.replace("_rep", "")
    assert rel_e(rb.total_energy, float(g[f"{base_name}_energy"])) <= E_TOL


@pytest.mark.parametrize("n", [1, 2, 37, 1000, 20000])
def test_direct_vs_oracle_sizes(port, n):
    rng = np.random.default_rng(n)
    L = max(5.0, (n / 0.1) ** (1 / 3))
    pos = rng.uniform(0, L, (n, 3))
    q = rng.choice([-1.0, 1.0], n)
    r = pkg.DirectCoulombField().evaluate(pkg.ParticleSystem(pos, None, q, None, np.array([L, L, L])))
    o = port.field_evaluate(fspec("direct", 0.0), pos, q, np.array([L, L, L]))
    if n == 1:
        assert r.total_energy == 0.0 and not r.per_particle_force.any()
        return
    check(r, o)


def test_overlay_on_msm_vs_reference(ref):
    # MsmField + PairRepulsionOverlay: the restatement has no MSM overlay, so check the
    # reference directly
    w = fx.config("c1s", n_override=3000)
    spec = fspec("msm", w.a, w.h, w.levels, rep_eps=0.1, rep_sigma=2.0)
    base = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    f = pkg.PairRepulsionOverlay(base, 0.1, 2.0)
    r = f.evaluate(pkg.ParticleSystem(w.pos, None, w.q, None, w.box))
    check(r, ref.field_evaluate(spec, w.pos, w.q, w.box))
    assert r.short_part is not None and r.long_part is not None


def test_direct_and_overlay_errors_and_dynamics(port):
    w = fx.config("c1", n_override=3000)
    pos = w.pos.copy()
    pos[1234] = pos[99]
    with pytest.raises(pkg.CoincidentParticlesError, match="particles 99 and 1234 coincide"):
        pkg.DirectCoulombField().evaluate(pkg.ParticleSystem(pos, None, w.q, None, w.box))
    f = pkg.PairRepulsionOverlay(gpu_field(fspec("cutoff", 10.0)), 0.1, 2.0)
    with pytest.raises(pkg.CoincidentParticlesError, match="particles 99 and 1234 coincide"):
        f.evaluate(pkg.ParticleSystem(pos, None, w.q, None, w.box))
    # 10 Verlet steps with the overlay on the cutoff field (device-resident) vs the restatement
    w = fx.config("c1s", n_override=2500)
    spec = fspec("cutoff", 10.0, rep_eps=0.1, rep_sigma=2.0)
    out = pkg.propagate(pkg.PropagatorSpec(f, 0.05, 10), pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
    p2, v2, done, err = port.field_propagate(spec, w.pos, w.vel, w.q, w.mass, w.box, 0.05, 10)
    assert err is None
    assert rel_rms(out.positions, p2) <= 1e-12 and rel_rms(out.velocities, v2) <= 1e-8
    # direct field propagate
    spec = fspec("direct", 0.0)
    out = pkg.propagate(pkg.PropagatorSpec(pkg.DirectCoulombField(), 0.05, 5),
                        pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
    p2, v2, done, err = port.field_propagate(spec, w.pos, w.vel, w.q, w.mass, w.box, 0.05, 5)
    assert err is None
    assert rel_rms(out.positions, p2) <= 1e-12 and rel_rms(out.velocities, v2) <= 1e-8


@pytest.mark.parametrize("n", [0, 1, 2, 31, 33, 65])
@pytest.mark.parametrize("spec", [fspec("cutoff", 8.0), fspec("wolf", 8.0, alpha=0.25), fspec("direct", 0.0),
                                  fspec("cutoff", 8.0, rep_eps=0.1, rep_sigma=1.5)])
def test_tiny_and_ragged_systems(port, n, spec):
    box = np.array([20.0, 20.0, 20.0])
    if n == 0:
        pos, q = np.zeros((0, 3)), np.zeros(0)
    else:
        pos, q = fx.uniform(n, box, "alternating", 0.5, 31)
    base = pkg.DirectCoulombField() if spec[0] == 3 else gpu_field(spec)
    f = pkg.PairRepulsionOverlay(base, float(spec[6]), float(spec[7])) if spec[6] > 0 else base
    r = f.evaluate(pkg.ParticleSystem(pos, None, q, None, box))
    if n == 0:
        assert r.total_energy == 0.0 and r.per_particle_potential.size == 0
        return
    o = port.field_evaluate(spec, pos, q, box)
    assert abs(r.total_energy - o["energy"]) <= E_TOL * max(1.0, abs(o["energy"]))
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL or np.allclose(r.per_particle_force, o["force"], atol=1e-12)
    assert np.allclose(r.per_particle_potential, o["phi"], rtol=1e-12, atol=1e-14)
