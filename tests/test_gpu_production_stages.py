"""Stage parity of the PRODUCTION kernels -- the ones every evaluation runs -- as
opposed to the bit-exact stage variants of tests/test_gpu_stages.py:

* binning: the production k_bin's sort keys decode to the reference's level-0
  cell triple floor((x - origin) * (1/h)) bit for bit, coverage included
  (src/msm_phases.cpp:21-29,42);
* restriction chain (k_restrict_tile<false>, separable FMA sums) vs the
  reference's restrict_charges per level (src/msm_phases.cpp:63-91), 1e-13 of the
  level scale;
* top level as evaluations run it (warp kernel / FFT job) vs top_level
  (src/msm_phases.cpp:136-162), 1e-13;
* prolongation chain vs prolongate (src/msm_phases.cpp:164-193), bit for bit;
* interpolation + long-range forces (k_interp) on the GPU's own level-0
  potential vs the reference's interpolate_to_atoms + self term +
  add_long_range_forces (src/msm_phases.cpp:195-222, src/msm.cpp:16-48,70-73),
  1e-13 for u_long and the long-range forces.
"""
import numpy as np
import pytest

from conftest import rel_rms
from gpu_util import level_slices
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx

pytestmark = pytest.mark.gpu

CASES = [("c1", None), ("c2", 30000), ("c5", 20000), ("c4", 30000), ("c2s", 120000)]


def _scale_err(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name,n", CASES)
def test_production_binning_bit_exact(name, n):
    w = fx.config(name, n_override=n)
    cfg = pkg.MsmConfig(w.a, w.h, w.levels)
    pos = w.pos.copy()
    # grid lines and coverage edges (x = -h accepted, x >= (ceil(L/h)+1) h rejected)
    _, _, org = pkg.grid_geometry(cfg, w.box)
    dims, _, _ = pkg.grid_geometry(cfg, w.box)
    pos[:17, 0] = org[0][0] + np.arange(17) * w.h + w.h
    pos[17] = [-w.h, -w.h, -w.h]
    hi = org[0] + (dims[0] - 2) * w.h
    pos[18] = np.nextafter(hi, -1e9)
    pos[19] = [hi[0], 1.0, 1.0]                 # just outside
    pos[20] = [np.nextafter(-w.h, -1e9), 1.0, 1.0]
    cells, cov = pkg.MsmField(cfg).debug_bin_keys(pos, w.box)
    t = (pos - org[0]) * (1.0 / w.h)            # IEEE sub, then mul by 1/h (msm_phases.cpp:42)
    exp_cov = np.all((np.floor(t) >= 1) & (np.floor(t) <= dims[0] - 3), axis=1)
    assert np.array_equal(cov, exp_cov)
    assert cov[17] and not cov[20]              # x = -h accepted, just below rejected
    assert not (cov[18] and cov[19])            # the upper edge: [hi - ulp, hi] straddles it
    assert np.array_equal(cells[cov], np.floor(t[cov]).astype(np.int64))


def _levels(port, name, n):
    w = fx.config(name, n_override=n)
    cfg = pkg.MsmConfig(w.a, w.h, w.levels)
    o = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels, diag=True)
    sl, _ = level_slices(cfg, w.box)
    return w, cfg, o, sl


@pytest.mark.parametrize("name,n", CASES)
def test_production_restriction_chain(port, name, n):
    w, cfg, o, sl = _levels(port, name, n)
    got = pkg.MsmField(cfg).debug_stage(5, 0, w.box, o["level_charge"][sl[0]])
    for k in range(1, w.levels):
        assert _scale_err(got[sl[k]], o["level_charge"][sl[k]]) <= 1e-13, k


@pytest.mark.parametrize("name,n", CASES)
def test_production_top_level(port, name, n):
    w, cfg, o, sl = _levels(port, name, n)
    t = w.levels - 1
    q = o["level_charge"][sl[t]]
    got = pkg.MsmField(cfg).debug_stage(6, t, w.box, q)
    assert _scale_err(got, port.top_level(w.box, w.a, w.h, w.levels, q)) <= 1e-13


@pytest.mark.parametrize("name,n", CASES)
def test_production_prolongation_chain(port, name, n):
    w, cfg, o, sl = _levels(port, name, n)
    # potentials before prolongation: lattice cutoff per level, top level on top
    pre = np.zeros_like(o["level_potential"])
    for k in range(w.levels - 1):
        pre[sl[k]] = port.lattice_cutoff(w.box, w.a, w.h, w.levels, k, o["level_charge"][sl[k]])
    t = w.levels - 1
    pre[sl[t]] = port.top_level(w.box, w.a, w.h, w.levels, o["level_charge"][sl[t]])
    got = pkg.MsmField(cfg).debug_stage(7, 0, w.box, pre)
    exp = pre.copy()
    for k in range(w.levels - 2, -1, -1):
        exp[sl[k]] = port.prolongate(w.box, w.a, w.h, w.levels, k, exp[sl[k + 1]], exp[sl[k]])
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("name,n", CASES)
def test_production_interpolation_and_forces(port, name, n):
    w = fx.config(name, n_override=n)
    cfg = pkg.MsmConfig(w.a, w.h, w.levels)
    f = pkg.MsmField(cfg)
    r = f.evaluate(pkg.ParticleSystem(w.pos, None, w.q, None, w.box))
    _, qp = f.debug_levels()
    sl, _ = level_slices(cfg, w.box)
    u, flong = port.long_range(w.pos, w.q, w.box, w.a, w.h, w.levels, qp[sl[0]])
    assert rel_rms(r.long_part, u) <= 1e-13
    _, fshort = port.short_range(w.pos, w.q, w.a)
    assert rel_rms(r.per_particle_force - fshort, flong) <= 1e-12
