"""The CPU oracle (oracle/msm_oracle.c) pinned against the reference itself:
golden vectors written by the compiled reference (tests/golden/make_golden.py),
the SPEC known-answer values, and -- when oracle/_ref is built -- bitwise
agreement with the reference on fresh seeded inputs."""
import numpy as np
import pytest

from conftest import golden, rel_e
from paper_1309_1889_b200 import fixtures as fx


def _eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


# SPEC.md:201-253 examples (verified against the compiled reference)
KATS = [(0, 0.0, 1.0, 1.875), (0, 1.0, 1.0, 1.0), (0, 2.0, 1.0, 0.5), (2, 0.5, 1.0, 0.4140625),
        (5, 0.5, 1.0, 0.5625), (5, 1.5, 1.0, -0.0625)]


@pytest.mark.parametrize("which,x,a,expect", KATS)
def test_spec_kats(port, which, x, a, expect):
    assert port.kernel(which, x, a) == expect


def test_kernel_kats_vs_reference_golden(port):
    g = golden("kats")
    args = {"gamma0": (0, 0.0, 1, 0, 1), "gamma1": (0, 1.0, 1, 0, 1), "gamma2": (0, 2.0, 1, 0, 1),
            "gstar_half": (2, 0.5, 1.0, 0, 1), "phi_half": (5, 0.5, 1, 0, 1), "phi_1p5": (5, 1.5, 1, 0, 1),
            "glevel_0_2": (4, 3.0, 8.0, 0, 2), "glevel_top": (4, 3.0, 8.0, 1, 2),
            "dphi_m03": (6, -0.3, 1, 0, 1), "dgstar": (3, 2.0, 5.0, 0, 1)}
    for k, (w, x, a, kk, l) in args.items():
        assert port.kernel(w, x, a, kk, l) == float(g[k]), k


@pytest.mark.parametrize("name", ["spec500", "c1_small", "c2_small", "c5_small", "c3_small"])
def test_port_bitwise_vs_reference_golden(port, name):
    g = golden(name)
    r = port.msm_potential(g["pos"], g["q"], g["box"], float(g["a"]), float(g["h"]), int(g["levels"]), diag=True)
    for k in ["phi", "phi_short", "phi_long", "force", "level_charge", "level_potential"]:
        assert _eq(r[k], g[k]), k
    assert r["energy"] == float(g["energy"])


def test_spec500_energy_value(port):
    # the reference gives U_msm = -597.6718 on the SPEC fixture (10.5% off direct)
    g = golden("spec500")
    assert abs(float(g["energy"]) - (-597.6718)) < 1e-4
    d = golden("spec500_direct")
    assert abs(rel_e(float(g["energy"]), float(d["energy"])) - 0.10537) < 1e-4


def test_port_trajectory_vs_reference_golden(port):
    g = golden("c1s_traj10")
    p, v, done, err = port.propagate(g["pos"], g["vel"], g["q"], g["mass"], g["box"], float(g["a"]),
                                     float(g["h"]), int(g["levels"]), float(g["dt"]), int(g["steps"]))
    assert err is None and done == 10
    assert _eq(p, g["out_pos"]) and _eq(v, g["out_vel"])


def test_port_abort_vs_reference_golden(port):
    g = golden("c1_abort")
    p, v, done, err = port.propagate(g["pos"], g["vel"], g["q"], g["mass"], g["box"], float(g["a"]),
                                     float(g["h"]), int(g["levels"]), float(g["dt"]), int(g["steps"]))
    assert done == int(g["steps_done"])
    assert err is not None and err.code == int(g["err_code"]) and err.msg == str(g["err_msg"])


@pytest.mark.parametrize("case", ["coincident", "nan", "coverage", "inf_pair", "coincident_vs_nan"])
def test_port_error_precedence_vs_reference_golden(port, case):
    import oracle_lib
    g = golden("errors")
    with pytest.raises(oracle_lib.OracleError) as ei:
        port.msm_potential(g[f"pos_{case}"], g["q"], g["box"], 8.0, 2.0, 3)
    assert ei.value.code == int(g[f"code_{case}"])
    assert ei.value.msg == str(g[f"msg_{case}"])


def test_port_parareal_vs_reference_golden(port):
    g = golden("parareal_w4k2")
    fine = tuple(g["fine"]); coarse = tuple(g["coarse"])
    fine = (fine[0], fine[1], int(fine[2]), fine[3], int(fine[4]))
    coarse = (coarse[0], coarse[1], int(coarse[2]), coarse[3], int(coarse[4]))
    rp, rv, dr, cnt = port.parareal_window(g["pos"], g["vel"], g["q"], g["mass"], g["box"], fine, coarse, 4, 2)
    assert _eq(rp, g["row_pos"]) and _eq(rv, g["row_vel"])
    assert _eq(cnt, g["counts"])
    assert np.allclose(dr[1:], g["delta_rms"][1:], rtol=1e-12)


# ---- live comparison with the compiled reference (when oracle/_ref exists) ------
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_bitwise_vs_reference_live(port, ref, seed):
    w = fx.config("c1", seed=seed, n_override=1500)
    a = ref.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels, diag=True)
    b = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels, diag=True)
    for k in a:
        assert _eq(a[k], b[k]), k


def test_port_grid_geometry_vs_reference(port, ref):
    for box, a, h, l in [([40, 40, 40], 10, 2.5, 2), ([144, 144, 144], 12, 2.5, 6),
                         ([300, 650, 650], 12, 2.5, 5), ([219, 219, 219], 8, 5, 3), ([7.3, 19.1, 3.3], 3, 1.1, 4)]:
        r1 = ref.grid_geometry(np.array(box, float), a, h, l)
        r2 = port.grid_geometry(np.array(box, float), a, h, l)
        for x, y in zip(r1, r2):
            assert _eq(x, y)


def test_port_parareal_run_vs_reference_live(port, ref):
    box = np.array([12.0, 12.0, 12.0])
    pos, q = fx.uniform(128, box, "random_neutral", 1.5, 5)
    mass = np.full(128, 18.0)
    vel = fx.maxwell_boltzmann(mass, 300.0, 6)
    fine, coarse = (8.0, 2.0, 2, 0.005, 8), (6.0, 3.0, 2, 0.02, 2)
    a = ref.parareal_run(pos, vel, q, mass, box, fine, coarse, 3, 4, 1e-7, 7)
    b = port.parareal_run(pos, vel, q, mass, box, fine, coarse, 3, 4, 1e-7, 7)
    assert (a[3] is None) == (b[3] is None)
    assert _eq(a[0], b[0]) and _eq(a[1], b[1]) and _eq(a[2], b[2])


# ---- pair-only fields: the restatement is bitwise the reference
def test_port_fields_bitwise_vs_reference_golden(port):
    g = golden("fields")
    for name, spec in zip(g["names"], g["specs"]):
        r = port.field_evaluate(spec, g["pos"], g["q"], g["box"])
        assert np.array_equal(r["phi"], g[f"{name}_phi"]), name
        assert np.array_equal(r["force"], g[f"{name}_force"]), name
        assert r["energy"] == float(g[f"{name}_energy"]), name


def test_port_field_trajectory_vs_reference_golden(port):
    g = golden("fields_traj10")
    p2, v2, done, err = port.field_propagate(g["spec"], g["pos"], g["vel"], g["q"], g["mass"], g["box"],
                                             float(g["dt"]), int(g["steps"]))
    assert err is None and done == int(g["steps"])
    assert np.array_equal(p2, g["out_pos"]) and np.array_equal(v2, g["out_vel"])


def test_port_field_parareal_vs_reference_golden(port):
    g = golden("fields_parareal_w4k2")
    rp, rv, dr, cnt = port.field_parareal_window(g["pos"], g["vel"], g["q"], g["mass"], g["box"], g["fine"],
                                                 float(g["fdt"]), int(g["fsteps"]), g["coarse"], float(g["gdt"]),
                                                 int(g["gsteps"]), int(g["t_points"]), int(g["k_iters"]))
    assert np.array_equal(rp, g["row_pos"]) and np.array_equal(rv, g["row_vel"])
    assert np.array_equal(dr[1:], g["delta_rms"][1:]) and np.array_equal(cnt, g["counts"])


@pytest.mark.parametrize("spec_args", [("cutoff", 9.0), ("wolf", 9.0, 0.0, 0, 0.3), ("direct", 0.0),
                                       ("wolf", 6.0, 0.0, 0, 0.25, 0.5, 1.5)])
def test_port_fields_bitwise_vs_reference_live(port, ref, spec_args):
    import oracle_lib
    spec = oracle_lib.fspec(*spec_args)
    rng = np.random.default_rng(11)
    n, L = 900, 22.0
    pos = rng.uniform(-2.0, L + 2.0, (n, 3))  # also outside the box: the fields ignore it
    q = rng.choice([-1.0, 0.5, 1.0], n)
    box = np.array([L, L, L])
    a = ref.field_evaluate(spec, pos, q, box)
    b = port.field_evaluate(spec, pos, q, box)
    assert np.array_equal(a["phi"], b["phi"]) and np.array_equal(a["force"], b["force"])
    assert a["energy"] == b["energy"]
    pos[17] = pos[5]
    import oracle_lib as ol
    for k in (ref, port):
        with pytest.raises(ol.OracleError, match="particles 5 and 17 coincide"):
            k.field_evaluate(spec, pos, q, box)
