"""Failure semantics: the GPU path raises the reference's exception type with
the reference's message and particle indices, with the reference's precedence
(short-range pair errors in i<j order before coverage, minimum particle index),
and reproduces literal-input trajectory aborts at the same step."""
import numpy as np
import pytest

from conftest import golden
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx

pytestmark = pytest.mark.gpu

EXC = {1: pkg.ConfigError, 2: pkg.DomainError, 3: pkg.CoverageError, 4: pkg.CoincidentParticlesError}


@pytest.mark.parametrize("case", ["coincident", "nan", "coverage", "inf_pair", "coincident_vs_nan"])
def test_error_vs_reference_golden(case):
    g = golden("errors")
    f = pkg.MsmField(pkg.MsmConfig(8.0, 2.0, 3))
    with pytest.raises(EXC[int(g[f"code_{case}"])]) as ei:
        f.evaluate(pkg.ParticleSystem(g[f"pos_{case}"], None, g["q"], None, g["box"]))
    assert str(ei.value) == str(g[f"msg_{case}"])


def _random_cases():
    rng = np.random.default_rng(11)
    box = np.array([30.0, 30.0, 30.0])
    pos, q = fx.uniform(2500, box, "random_neutral", 0.5, 12)
    out = []
    for t in range(8):
        p = pos.copy()
        k = rng.integers(1, 5)
        for _ in range(k):
            kind = rng.integers(0, 4)
            i, j = rng.integers(0, 2500, size=2)
            if kind == 0:
                p[i] = p[j]
            elif kind == 1:
                p[i, rng.integers(0, 3)] = np.nan
            elif kind == 2:
                p[i, rng.integers(0, 3)] = rng.choice([-3.0, 33.5, 40.0])
            else:
                p[i, rng.integers(0, 3)] = rng.choice([np.inf, -np.inf])
        out.append((p, q, box))
    return out


@pytest.mark.parametrize("idx", range(8))
def test_error_precedence_random(port, idx):
    import oracle_lib
    p, q, box = _random_cases()[idx]
    try:
        port.msm_potential(p, q, box, 8.0, 2.0, 2)
        expect = None
    except oracle_lib.OracleError as e:
        expect = e
    f = pkg.MsmField(pkg.MsmConfig(8.0, 2.0, 2))
    if expect is None:
        f.evaluate(pkg.ParticleSystem(p, None, q, None, box))
        return
    with pytest.raises(EXC[expect.code]) as ei:
        f.evaluate(pkg.ParticleSystem(p, None, q, None, box))
    assert str(ei.value) == expect.msg


def test_box_error_after_pair_error(port):
    # short_range runs before build_grid_hierarchy (src/msm.cpp:58-60): a coincident
    # pair wins over an invalid box -- but an invalid box is a ConfigError otherwise.
    box = np.array([30.0, 30.0, 30.0])
    pos, q = fx.uniform(200, box, "alternating", 1.0, 2)
    f = pkg.MsmField(pkg.MsmConfig(8.0, 2.0, 2))
    with pytest.raises(pkg.ConfigError, match="msm: box extents must be positive"):
        f.evaluate(pkg.ParticleSystem(pos, None, q, None, [30.0, 0.0, 30.0]))


def test_literal_trajectory_abort_vs_reference_golden():
    g = golden("c1_abort")
    f = pkg.MsmField(pkg.MsmConfig(float(g["a"]), float(g["h"]), int(g["levels"])))
    s = pkg.ParticleSystem(g["pos"], g["vel"], g["q"], g["mass"], g["box"])
    with pytest.raises(EXC[int(g["err_code"])]) as ei:
        pkg.propagate(pkg.PropagatorSpec(f, float(g["dt"]), int(g["steps"])), s)
    assert str(ei.value) == str(g["err_msg"])
    assert ei.value.step == int(g["steps_done"]) + 1


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_literal_config_abort_vs_oracle(port, name):
    """P1: the literal BASELINE inputs abort in the reference; the GPU aborts at the
    same step with the same exception and particle index."""
    w = fx.config(name)
    _, _, done, err = port.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, 5)
    assert err is not None
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    with pytest.raises(EXC[err.code]) as ei:
        pkg.propagate(pkg.PropagatorSpec(f, w.dt, 5), s)
    assert str(ei.value) == err.msg and ei.value.step == done + 1
    # the device-resident system is left untouched on error
    dev = pkg.DeviceSystem(f, s)
    with pytest.raises(EXC[err.code]):
        dev.propagate(w.dt, 5)
    p, v = dev.download()
    assert np.array_equal(p, w.pos) and np.array_equal(v, w.vel)


def test_propagate_validation():
    f = pkg.MsmField(pkg.MsmConfig(8.0, 2.0, 2))
    s = pkg.ParticleSystem(np.zeros((2, 3)) + [[1, 1, 1], [5, 5, 5]], None, [1.0, -1.0], None, [10.0] * 3)
    with pytest.raises(pkg.ConfigError, match="dt must be > 0"):
        pkg.propagate(pkg.PropagatorSpec(f, -1.0, 2), s)
    with pytest.raises(pkg.ConfigError, match="steps_per_slice must be >= 1"):
        pkg.propagate(pkg.PropagatorSpec(f, 1.0, 0), s)
