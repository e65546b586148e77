"""Parity at the BASELINE sizes the bench and the multi-GPU paths run.

* C2 / C2-S (300,000 water atoms, 6 levels): the benchmarked configuration.  At
  this size the pair sum runs the large-system instance of the pair kernel (one
  warp per i-cluster, `pair_split == 1`), on water geometry (O-H at 0.957 A, H
  atoms outside the box): checked against the C oracle (cell lists; bitwise with
  the reference on every fixture, tests/test_oracle.py), energy 1e-10, RMS force
  1e-8 (BASELINE.json north_star), potentials 1e-12.
* C3 (2^24 atoms) and C4 (12.7M atoms): the whole evaluation against the same
  oracle (per-atom results equal to the reference's `short_range` restricted to
  cell neighbourhoods, the survey's blocked oracle) -- energy,
  forces, and phi_short / phi_long.
* P1 literal aborts for C3, C4 and C5: the literal inputs abort in
  the reference; the GPU aborts at the same Verlet step with the same exception
  type, message and particle index.
Reference: msm_potential src/msm.cpp:52-90, short_range src/msm_phases.cpp:224-252,
propagate src/integrate.cpp:13-36.
"""
import numpy as np
import pytest

from conftest import rel_e, rel_rms
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

E_TOL, F_TOL, PHI_TOL = 1e-10, 1e-8, 1e-12
EXC = {1: pkg.ConfigError, 2: pkg.DomainError, 3: pkg.CoverageError, 4: pkg.CoincidentParticlesError}


def _check(w, r, o):
    assert rel_e(r.total_energy, o["energy"]) <= E_TOL
    assert rel_rms(r.per_particle_force, o["force"]) <= F_TOL
    assert rel_rms(r.short_part, o["phi_short"]) <= PHI_TOL
    assert rel_rms(r.long_part, o["phi_long"]) <= PHI_TOL
    assert rel_rms(r.per_particle_potential, o["phi"]) <= PHI_TOL


@pytest.mark.parametrize("name", ["c2s", "c2"])
def test_c2_full_size_vs_oracle(port, name):
    w = fx.config(name)
    assert w.n == 300_000
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    r = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)).evaluate()
    wc = f.work_counters()
    assert wc["pair_split"] == 1          # the production large-system pair kernel
    assert wc["pairs"] > 9e7              # ~9.7e7 unordered in-cutoff pairs
    # water geometry: some H atoms sit outside the box, inside MSM coverage
    assert np.any(w.pos < 0.0) or np.any(w.pos > w.box)
    _check(w, r, port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels))


@pytest.mark.parametrize("name", ["c4", "c3"])
def test_c3_c4_full_size_vs_oracle(port, name):
    w = fx.config(name)
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    r = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)).evaluate()
    assert f.work_counters()["pair_split"] == 1
    _check(w, r, port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels))


@pytest.mark.parametrize("name", ["c5", "c4", "c3"])
def test_literal_abort_full_size(port, name):
    """P1 at full size: same abort step, exception type, message and particle."""
    w = fx.config(name)
    _, _, done, err = port.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, 4)
    assert err is not None, "the literal input is expected to abort in the reference"
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    with pytest.raises(EXC[err.code]) as ei:
        pkg.DeviceSystem(f, s).propagate(w.dt, 4)
    assert str(ei.value) == err.msg and ei.value.step == done + 1
