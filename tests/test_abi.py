"""The C-ABI library loads, exports every symbol include/msmb.h declares, and
its host-side logic (validation, level geometry) matches the reference --
all without a GPU.  Compute entry points must fail loudly without one."""
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "msmb.h"


def declared_symbols():
    txt = HEADER.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(msmb_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_all_exported():
    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.exported_symbols())


def test_abi_version():
    assert _native.lib().msmb_abi_version() == 2


@pytest.mark.parametrize("box,a,h,l", [([40, 40, 40], 10, 2.5, 2), ([144, 144, 144], 12, 2.5, 6),
                                       ([551, 551, 551], 12, 2.5, 4), ([300, 650, 650], 12, 2.5, 5),
                                       ([219, 219, 219], 8, 5, 3), ([7.3, 19.1, 3.3], 3, 1.1, 4)])
def test_grid_geometry_matches_reference(port, box, a, h, l):
    d1, s1, o1 = pkg.grid_geometry(pkg.MsmConfig(a, h, l), np.array(box, float))
    d2, s2, o2 = port.grid_geometry(np.array(box, float), a, h, l)
    assert np.array_equal(d1, d2) and np.array_equal(s1, s2) and np.array_equal(o1, o2)


def test_level_sizes_from_survey():
    # SURVEY 8 level sizes (reference build_grid_hierarchy probe output)
    d, _, _ = pkg.grid_geometry(pkg.MsmConfig(12, 2.5, 4), [551.0] * 3)
    assert [tuple(x) for x in d] == [(226,) * 3, (116,) * 3, (61,) * 3, (34,) * 3]
    d, _, _ = pkg.grid_geometry(pkg.MsmConfig(12, 2.5, 6), [144.0] * 3)
    assert [x[0] for x in d] == [63, 35, 21, 14, 10, 8]
    d, _, _ = pkg.grid_geometry(pkg.MsmConfig(12, 2.5, 5), [300.0, 650.0, 650.0])
    assert tuple(d[0]) == (125, 265, 265) and tuple(d[4]) == (14, 23, 23)


@pytest.mark.parametrize("cfg,msg", [
    (pkg.MsmConfig(0.0, 2.0, 2), "msm: cutoff_a must be > 0"),
    (pkg.MsmConfig(8.0, -1.0, 2), "msm: spacing_h must be > 0"),
    (pkg.MsmConfig(8.0, 2.0, 0), "msm: levels_l must be >= 1"),
    (pkg.MsmConfig(8.0, 2.0, 2, 5), "msm: unsupported interpolation order p=5"),
    (pkg.MsmConfig(8.0, 2.0, 2, 3, 4), "msm: unsupported smoothing order m=4"),
    (pkg.MsmConfig(1.0, 2.0, 2), "msm: cutoff_a / spacing_h must be >= 1"),
])
def test_config_validation_messages(cfg, msg):
    # validation happens before any GPU work (MsmConfig::validate, src/msm_grid.cpp:11-22)
    with pytest.raises(pkg.ConfigError) as ei:
        pkg.MsmField(cfg)
    assert str(ei.value) == msg


def test_units_validation():
    with pytest.raises(pkg.ConfigError, match="coulomb_constant must be > 0"):
        pkg.MsmField(pkg.MsmConfig(8, 2, 2), pkg.UnitsConfig(0.0, 1.0))


def test_propagator_spec_validation():
    with pytest.raises(pkg.ConfigError, match="propagator has no force field"):
        pkg.PropagatorSpec(None, 1.0, 1).validate()
    with pytest.raises(pkg.ConfigError, match="dt must be > 0"):
        pkg.PropagatorSpec(object(), 0.0, 1).validate()


def test_no_cpu_fallback_without_gpu():
    if pkg.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(pkg.CudaUnavailableError):
        pkg.MsmField(pkg.MsmConfig(10.0, 2.5, 2))


def test_cost_model_is_reference_formula(ref):
    # MsmField::cost_flops_per_step = msm_flops_simplified (src/force_field.cpp:41-43)
    from paper_1309_1889_b200 import _native
    import ctypes as C
    for a, h, n in [(12, 2, 1e5), (10, 2.5, 8192)]:
        assert ref.lib.ref_msm_flops_simplified(a, h, n) == pytest.approx(
            77.7 * a ** 3 * n + 566 * n + 73 * a ** 3 / h ** 6 * n + 80 / h ** 3 * n, rel=1e-15)


@pytest.mark.parametrize("cls,params,msg", [
    (pkg.SimpleCutoffField, pkg.CutoffParams(0.0), "cutoff must be > 0"),
    (pkg.SimpleCutoffField, pkg.CutoffParams(float("nan")), "cutoff must be > 0"),
    (pkg.WolfField, pkg.CutoffParams(10.0), "wolf_alpha is required"),
    (pkg.WolfField, pkg.CutoffParams(10.0, -0.1), "wolf_alpha must be >= 0"),
    (pkg.SimpleCutoffField, pkg.CutoffParams(10.0, -0.1), "wolf_alpha must be >= 0"),
])
def test_pair_field_validation_messages(cls, params, msg):
    # CutoffParams::validate (src/electrostatics.cpp:38-42), before any GPU work
    with pytest.raises(pkg.ConfigError) as ei:
        cls(params)
    assert str(ei.value) == msg
    with pytest.raises(pkg.ConfigError) as ei:
        params.validate(cls is pkg.WolfField)
    assert str(ei.value) == msg


def test_pair_field_no_cpu_fallback_without_gpu():
    if pkg.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(pkg.CudaUnavailableError):
        pkg.SimpleCutoffField(pkg.CutoffParams(10.0))
    with pytest.raises(pkg.CudaUnavailableError):
        pkg.WolfField(pkg.CutoffParams(10.0, 0.2))
