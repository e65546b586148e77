"""Whole-evaluation parity of the sm_100a path (through the C ABI) with the
reference: golden vectors written by the reference itself, and the bitwise C
restatement (oracle/) on seeded inputs of every BASELINE config shape.
Tolerances are BASELINE.json's: energy 1e-10 relative, RMS force 1e-8 relative."""
import numpy as np
import pytest

from conftest import golden, rel_e, rel_rms
from gpu_util import field, system
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx

pytestmark = pytest.mark.gpu

E_TOL, F_TOL = 1e-10, 1e-8


@pytest.mark.parametrize("name", ["spec500", "c1_small", "c2_small", "c5_small", "c3_small"])
def test_golden(name):
    g = golden(name)
    f = pkg.MsmField(pkg.MsmConfig(float(g["a"]), float(g["h"]), int(g["levels"])))
    s = pkg.ParticleSystem(g["pos"], None, g["q"], None, g["box"])
    r = f.evaluate(s)
    assert rel_e(r.total_energy, float(g["energy"])) <= E_TOL
    assert rel_rms(r.per_particle_force, g["force"]) <= F_TOL
    assert rel_rms(r.per_particle_potential, g["phi"]) <= 1e-12
    assert rel_rms(r.short_part, g["phi_short"]) <= 1e-12
    assert rel_rms(r.long_part, g["phi_long"]) <= 1e-12
    # level lattices (MsmDiagnostics, msm.hpp:11-13)
    qc, qp = f.debug_levels()
    assert rel_rms(qc, g["level_charge"]) <= 1e-13
    assert rel_rms(qp, g["level_potential"]) <= 1e-12


@pytest.mark.parametrize("name,n", [("c1", None), ("c1s", None), ("c2", 30000), ("c2s", 30000),
                                    ("c3", 40000), ("c4", 45000), ("c5", 40000)])
def test_config_shapes_vs_oracle(port, name, n):
    w = fx.config(name, n_override=n)
    f = field(w)
    r = f.evaluate(system(w))
    o = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels)
    assert rel_e(r.total_energy, o["energy"]) <= E_TOL
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL
    assert rel_rms(r.short_part, o["phi_short"]) <= 1e-12
    assert rel_rms(r.long_part, o["phi_long"]) <= 1e-12
    wc = f.work_counters()
    assert wc["pairs"] > 0 and wc["candidates"] >= 2 * wc["pairs"]


def test_c5_coarse_propagator_field(port):
    # config 5's G: a=8 h=5 l=3 (coarser grid, 5 A columns)
    w = fx.config("c5", n_override=30000)
    f = pkg.MsmField(pkg.MsmConfig(8.0, 5.0, 3))
    r = f.evaluate(system(w))
    o = port.msm_potential(w.pos, w.q, w.box, 8.0, 5.0, 3)
    assert rel_e(r.total_energy, o["energy"]) <= E_TOL
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL


@pytest.mark.parametrize("a,h,l,box", [(8.0, 2.0, 1, (20.0, 20.0, 20.0)), (6.0, 1.5, 3, (15.0, 31.0, 9.0)),
                                       (12.0, 3.0, 2, (50.0, 20.0, 35.0)), (9.0, 2.0, 4, (33.0, 33.0, 33.0))])
def test_odd_configs_vs_oracle(port, a, h, l, box):
    box = np.array(box)
    pos, q = fx.uniform(1500, box, "random_neutral", 0.8, 17)
    f = pkg.MsmField(pkg.MsmConfig(a, h, l))
    r = f.evaluate(pkg.ParticleSystem(pos, None, q, None, box))
    o = port.msm_potential(pos, q, box, a, h, l)
    assert rel_e(r.total_energy, o["energy"]) <= E_TOL
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL


def test_reduced_units_and_odd_charges(port):
    box = np.array([25.0, 25.0, 25.0])
    pos, _ = fx.uniform(2000, box, "all_plus_one", 1.0, 23)
    q = np.random.default_rng(3).normal(size=2000)
    f = pkg.MsmField(pkg.MsmConfig(7.0, 2.0, 3), pkg.UnitsConfig.reduced())
    r = f.evaluate(pkg.ParticleSystem(pos, None, q, None, box))
    o = port.msm_potential(pos, q, box, 7.0, 2.0, 3, kc=1.0, conv=1.0)
    assert rel_e(r.total_energy, o["energy"]) <= E_TOL
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL


@pytest.mark.parametrize("n", [0, 1, 2, 31, 33])
def test_tiny_and_ragged_systems(port, n):
    box = np.array([20.0, 20.0, 20.0])
    if n == 0:
        pos, q = np.zeros((0, 3)), np.zeros(0)
    else:
        pos, q = fx.uniform(n, box, "alternating", 0.5, 31)
    f = pkg.MsmField(pkg.MsmConfig(8.0, 2.0, 2))
    r = f.evaluate(pkg.ParticleSystem(pos, None, q, None, box))
    o = port.msm_potential(pos, q, box, 8.0, 2.0, 2)
    if n == 0:
        assert r.total_energy == 0.0
        return
    assert abs(r.total_energy - o["energy"]) <= E_TOL * max(1.0, abs(o["energy"]))
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL or np.allclose(r.per_particle_force, o["force"], atol=1e-12)


def test_clustered_dense_cell(port):
    # many atoms in a few cells (long cell lists, uneven clusters)
    box = np.array([30.0, 30.0, 30.0])
    rng = np.random.default_rng(5)
    pos = np.concatenate([rng.uniform(14.0, 16.0, size=(600, 3)), rng.uniform(0.0, 30.0, size=(900, 3))])
    q = np.where(np.arange(1500) % 2 == 0, 1.0, -1.0)
    f = pkg.MsmField(pkg.MsmConfig(9.0, 2.0, 3))
    r = f.evaluate(pkg.ParticleSystem(pos, None, q, None, box))
    o = port.msm_potential(pos, q, box, 9.0, 2.0, 3)
    assert rel_e(r.total_energy, o["energy"]) <= E_TOL
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL


def test_coverage_edges_accepted(port):
    # x = -h is covered, x just below (ceil(L/h)+1)h is covered
    box = np.array([40.0, 40.0, 40.0])
    pos, q = fx.uniform(400, box, "alternating", 1.0, 3)
    pos[0] = [-2.5, -2.5, -2.5]
    pos[1] = [np.nextafter(42.5, 0), 20.0, 20.0]
    f = pkg.MsmField(pkg.MsmConfig(10.0, 2.5, 2))
    r = f.evaluate(pkg.ParticleSystem(pos, None, q, None, box))
    o = port.msm_potential(pos, q, box, 10.0, 2.5, 2)
    assert rel_e(r.total_energy, o["energy"]) <= E_TOL


def test_determinism_bitwise():
    w = fx.config("c2s", n_override=60000)
    f = field(w)
    s = system(w)
    r1 = f.evaluate(s)
    r2 = f.evaluate(s)
    f2 = field(w)
    r3 = f2.evaluate(s)
    for a, b in [(r1, r2), (r1, r3)]:
        assert a.total_energy == b.total_energy
        assert np.array_equal(a.per_particle_force, b.per_particle_force)
        assert np.array_equal(a.per_particle_potential, b.per_particle_potential)


def test_msm_potential_free_function(port):
    g = golden("spec500")
    r = pkg.msm_potential(pkg.ParticleSystem(g["pos"], None, g["q"], None, g["box"]), pkg.MsmConfig(8.0, 2.0, 3))
    assert rel_e(r.total_energy, float(g["energy"])) <= E_TOL


@pytest.mark.parametrize("name,n", [("c2s", 30000), ("c4", 45000), ("c5", 40000)])
def test_fft_and_direct_lattice_agree(name, n):
    w = fx.config(name, n_override=n)
    a = field(w)
    b = field(w)
    b.set_lattice_method(direct=True)
    ra, rb = a.evaluate(system(w)), b.evaluate(system(w))
    assert rel_e(ra.total_energy, rb.total_energy) <= 1e-13
    assert rel_rms(ra.long_part, rb.long_part) <= 1e-13
    assert np.array_equal(ra.short_part, rb.short_part)


def test_propagate_bitwise_across_fresh_fields():
    # two independently built fields (own spectra, own workspaces) and the graph vs
    # eager paths give bit-identical trajectories (C2 shape with small levels where
    # the FFT padding M < 2R + 1)
    w = fx.config("c2s", n_override=30000)
    out = []
    for eager in (False, False, True):
        f = field(w)
        ds = pkg.DeviceSystem(f, system(w))
        if eager:
            f.set_stage_timing(True)
        ds.propagate(w.dt, 2)
        out.append(ds.download())
    for p, v in out[1:]:
        assert np.array_equal(p, out[0][0]) and np.array_equal(v, out[0][1])


def test_fields_with_different_fft_sizes_coexist(port):
    # the dynamic shared-memory limit of the FFT kernels is process-wide; a field with
    # a small plan created after one with a large plan must not break the large one
    box = np.array([219.0, 219.0, 219.0])
    pos, q = fx.uniform(4000, box, "random_neutral", 1.5, 21)
    s = pkg.ParticleSystem(pos, None, q, None, box)
    big = pkg.MsmField(pkg.MsmConfig(12.0, 2.5, 4))
    e1 = big.evaluate(s).total_energy
    small = pkg.MsmField(pkg.MsmConfig(8.0, 5.0, 3))
    small.evaluate(s)
    r = big.evaluate(s)
    assert r.total_energy == e1
    ds = pkg.DeviceSystem(big, s)
    ds.propagate(0.005, 2)  # graph capture path
    o = port.msm_potential(pos, q, box, 12.0, 2.5, 4)
    assert rel_e(e1, o["energy"]) <= 1e-10


@pytest.mark.parametrize("env", [{"MSMB_DENSE_T": "0"}, {"MSMB_DENSE_T": "16"}, {"MSMB_DENSE_T": "32"},
                                 {"MSMB_DENSE_CAP": "64"}, {"MSMB_DENSE_T": "12", "MSMB_DENSE_CAP": "96"}])
def test_dense_phase_settings_vs_oracle(port, env, monkeypatch):
    # the pair kernel's dense phase (k_pairmask's dense lists): off, other thresholds, and
    # dense lists that overflow their capacity (the excess stays in the per-lane masks) --
    # every setting sums the same pairs; the knobs are read when the field's geometry is built
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    w = fx.config("c2s", n_override=30000)
    f = field(w)
    r = f.evaluate(system(w))
    o = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels)
    assert rel_e(r.total_energy, o["energy"]) <= E_TOL
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL
    assert rel_rms(r.short_part, o["phi_short"]) <= 1e-12
    wc = f.work_counters()
    assert wc["pairs"] > 0
    # the same set of in-cutoff pairs whatever the split between the phases
    monkeypatch.undo()
    f0 = field(w)
    f0.evaluate(system(w))
    assert f0.work_counters()["pairs"] == wc["pairs"]
