"""Per-stage parity: each sm_100a stage kernel against the reference phase
function on identical inputs (test plan item 1).  Binning,
restriction, prolongation and interpolation reproduce the reference bit for
bit; anterpolation, the lattice-cutoff stencil and the top level sum in a
different (deterministic) order and are held to 1e-13 of the lattice scale."""
import numpy as np
import pytest

from conftest import golden
from gpu_util import level_slices
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx

pytestmark = pytest.mark.gpu

CASES = [("c1", None), ("c2", 30000), ("c5", 20000), ("c4", 30000)]


def _setup(port, name, n):
    w = fx.config(name, n_override=n)
    cfg = pkg.MsmConfig(w.a, w.h, w.levels)
    o = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels, diag=True)
    sl, dims = level_slices(cfg, w.box)
    return w, cfg, o, sl


def _scale_err(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name,n", CASES)
def test_restriction_bitwise(port, name, n):
    w, cfg, o, sl = _setup(port, name, n)
    f = pkg.MsmField(cfg)
    for k in range(w.levels - 1):
        fine = o["level_charge"][sl[k]]
        got = f.debug_stage(0, k, w.box, fine)
        assert np.array_equal(got, port.restrict(w.box, w.a, w.h, w.levels, k, fine))
        assert np.array_equal(got, o["level_charge"][sl[k + 1]])


@pytest.mark.parametrize("name,n", CASES)
def test_prolongation_bitwise(port, name, n):
    w, cfg, o, sl = _setup(port, name, n)
    f = pkg.MsmField(cfg)
    for k in range(w.levels - 2, -1, -1):
        fine_in = port.lattice_cutoff(w.box, w.a, w.h, w.levels, k, o["level_charge"][sl[k]])
        coarse = o["level_potential"][sl[k + 1]]
        got = f.debug_stage(3, k, w.box, coarse, out=fine_in)
        exp = port.prolongate(w.box, w.a, w.h, w.levels, k, coarse, fine_in)
        bad = np.flatnonzero(got != exp)
        assert bad.size == 0, (f"level {k}: {bad.size}/{got.size} differ, first {bad[:5]}, "
                               f"unchanged={np.array_equal(got, fine_in)}, maxdiff={np.max(np.abs(got - exp))}")
        assert np.array_equal(got, o["level_potential"][sl[k]])


@pytest.mark.parametrize("name,n", CASES)
def test_interpolation_bitwise(port, name, n):
    w, cfg, o, sl = _setup(port, name, n)
    f = pkg.MsmField(cfg)
    pot0 = o["level_potential"][sl[0]]
    got = f.debug_stage(4, 0, w.box, pot0, positions=w.pos)
    assert np.array_equal(got, port.interpolate(w.pos, w.box, w.a, w.h, w.levels, pot0))


@pytest.mark.parametrize("method", ["fft", "direct"])
@pytest.mark.parametrize("name,n", CASES)
def test_lattice_cutoff(port, name, n, method):
    # fft: zero-padded FFT convolution (default); direct: the stencil sum (k_lattice)
    w, cfg, o, sl = _setup(port, name, n)
    f = pkg.MsmField(cfg)
    f.set_lattice_method(direct=method == "direct")
    for k in range(w.levels - 1):
        q = o["level_charge"][sl[k]]
        got = f.debug_stage(1, k, w.box, q)
        assert _scale_err(got, port.lattice_cutoff(w.box, w.a, w.h, w.levels, k, q)) <= 1e-13


@pytest.mark.parametrize("name,n", CASES)
def test_top_level(port, name, n):
    w, cfg, o, sl = _setup(port, name, n)
    f = pkg.MsmField(cfg)
    t = w.levels - 1
    q = o["level_charge"][sl[t]]
    got = f.debug_stage(2, t, w.box, q)
    ref = port.top_level(w.box, w.a, w.h, w.levels, q)
    assert _scale_err(got, ref) <= 1e-13
    # small top levels use the direct gather in the reference's order with exact grid
    # coordinates (h = 2.5 * 2^k): bit-for-bit the reference's top_level
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("name,n", CASES)
def test_anterpolation(port, name, n):
    w, cfg, o, sl = _setup(port, name, n)
    f = pkg.MsmField(cfg)
    f.evaluate(pkg.ParticleSystem(w.pos, None, w.q, None, w.box))
    qc, _ = f.debug_levels()
    assert _scale_err(qc[sl[0]], o["level_charge"][sl[0]]) <= 1e-14
    # charge conservation (SPEC acceptance 3): the cubic basis is a partition of unity
    assert abs(qc[sl[0]].sum() - w.q.sum()) <= 1e-12 * np.abs(w.q).sum()


def test_cells_bit_exact_including_grid_lines():
    """Level-0 cell triple floor((x - origin) * (1/h)) (src/msm_phases.cpp:23,42) for every
    particle, including positions exactly on grid lines and at the coverage edges."""
    box = np.array([40.0, 40.0, 40.0])
    cfg = pkg.MsmConfig(10.0, 2.5, 2)
    f = pkg.MsmField(cfg)
    pos, _ = fx.uniform(3000, box, "alternating", 0.0, 9)
    grid = np.arange(-1, 18) * 2.5
    pos[:len(grid), 0] = grid
    pos[:len(grid), 1] = grid[::-1]
    pos[100] = [-2.5, -2.5, -2.5]
    pos[101] = [np.nextafter(42.5, 0), np.nextafter(42.5, 0), 0.0]
    pos[102] = [np.nextafter(-2.5, -10), 5.0, 5.0]  # just outside
    pos[103] = [42.5, 5.0, 5.0]                     # just outside
    pos[104] = [1e-300, -1e-300, 0.0]
    cells, cov = f.debug_cells(pos, box)
    _, _, org = pkg.grid_geometry(cfg, box)
    t = (pos - org[0]) * (1.0 / 2.5)  # numpy: IEEE sub then mul, like the reference
    assert np.array_equal(cells, np.floor(t).astype(np.int64))
    dims, _, _ = pkg.grid_geometry(cfg, box)
    exp_cov = np.all((np.floor(t) >= 1) & (np.floor(t) <= dims[0] - 3), axis=1)
    assert np.array_equal(cov, exp_cov)
    assert cov[100] and cov[101] and not cov[102] and not cov[103]


@pytest.mark.parametrize("box,levels", [((219.0, 219.0, 219.0), 4),      # C5 fine: top 17^3 = 4913
                                        ((120.0, 180.0, 150.0), 3)])     # ragged top
def test_top_level_fft_large(port, box, levels):
    # top levels above kTopFftMin points run as a dense FFT convolution (M >= 2d - 1)
    cfg = pkg.MsmConfig(12.0, 2.5, levels)
    box = np.array(box)
    _, dims = level_slices(cfg, box)
    t = levels - 1
    m = int(np.prod(dims[t]))
    assert m > 4096
    q = np.random.default_rng(3).standard_normal(m)
    got = pkg.MsmField(cfg).debug_stage(2, t, box, q)
    ref = port.top_level(box, 12.0, 2.5, levels, q)
    assert _scale_err(got, ref) <= 1e-13


def test_anterpolation_streaming_kernel(port):
    # the layer-streaming anterpolation runs for level-0 lattices above 4M points: a
    # C3-sized box (226^3 points) with few atoms exercises it against the reference
    box = np.array([551.0, 551.0, 551.0])
    pos, q = fx.uniform(20000, box, "random_neutral", 1.5, 31)
    cfg = pkg.MsmConfig(12.0, 2.5, 4)
    f = pkg.MsmField(cfg)
    f.evaluate(pkg.ParticleSystem(pos, None, q, None, box))
    qc, _ = f.debug_levels()
    o = port.msm_potential(pos, q, box, 12.0, 2.5, 4, diag=True)
    sl, _ = level_slices(cfg, box)
    assert _scale_err(qc[sl[0]], o["level_charge"][sl[0]]) <= 1e-14
