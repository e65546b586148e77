"""The command-line front end (tools/paramd_main.cpp): CPU checks of
`gen` (byte-identical to the reference generator + writer), option errors and exit
codes; GPU runs of simulate / compare / parareal checked against the reference library."""
import csv
import ctypes as C

import numpy as np
import pytest

import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import cli, xyz_io
import oracle_lib

_D = C.POINTER(C.c_double)


def run(tmp_path, *args):
    return cli.main(["--out-dir", str(tmp_path), *args])


def rows(path):
    with open(path) as f:
        return list(csv.reader(f))


def test_gen_matches_reference_generator(ref, tmp_path):
    out = tmp_path / "sys.xyz"
    assert cli.main(["--seed", "42", "gen", "--n", "500", "--box", "40", "--scheme", "random_neutral",
                     "--min-sep", "1.5", "--out", str(out)]) == 0
    n, box = 500, np.array([40.0, 40.0, 40.0])
    pos, q = np.zeros((n, 3)), np.zeros(n)
    buf = C.create_string_buffer(256)
    assert ref.lib.ref_generate_random_system(n, oracle_lib._p(box), 2, 1.5, 42, oracle_lib._p(pos),
                                              oracle_lib._p(q), buf, 256) == 0
    s = xyz_io.load_system(str(out))
    assert np.array_equal(s.positions, pos) and np.array_equal(s.charges, q)
    assert not s.velocities.any() and (s.masses == 1.0).all()


@pytest.mark.parametrize("args,code", [
    (["gen", "--box", "1", "2"], 2),                       # --box takes 1 or 3 values
    (["gen", "--scheme", "nope"], 2),
    (["simulate", "--input", "x.xyz", "--force-field", "nope"], 2),
    (["--units", "weird", "simulate", "--input", "x.xyz"], 2),
    (["simulate"], 2),                                      # --input is required
])
def test_exit_codes(tmp_path, args, code):
    assert run(tmp_path, *args) == code


def test_input_errors_exit_2(tmp_path):
    bad = tmp_path / "bad.xyz"
    bad.write_text("2\nbox 5 5 5\nX 0 0 0 1 0 0 0 1\n")
    if pkg.device_count() == 0:
        pytest.skip("field construction needs the GPU before the input is read")
    assert run(tmp_path, "simulate", "--input", str(bad), "--force-field", "cutoff") == 2


@pytest.mark.gpu
def test_simulate_and_compare_vs_reference(ref, tmp_path):
    from paper_1309_1889_b200 import fixtures as fx
    w = fx.config("c1s", n_override=1200)
    inp = tmp_path / "in.xyz"
    xyz_io.save_system(pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box), str(inp))
    for kind, extra, spec in [("msm", ["--a", "10", "--h", "2.5", "--levels", "2"], oracle_lib.fspec("msm", 10.0, 2.5, 2)),
                              ("cutoff", ["--cutoff", "9"], oracle_lib.fspec("cutoff", 9.0))]:
        assert run(tmp_path, "simulate", "--input", str(inp), "--force-field", kind, "--steps", "6", "--dt", "0.02",
                   "--log-every", "2", "--traj-every", "3", *extra) == 0
        e = rows(tmp_path / f"{kind}_energy.csv")
        assert e[0] == ["step", "time_fs", "kinetic", "potential", "total"]
        assert [r[0] for r in e[1:]] == ["0", "2", "4", "6"]
        p6, v6, done, err = ref.field_propagate(spec, w.pos, w.vel, w.q, w.mass, w.box, 0.02, 6)
        assert err is None
        pot6 = ref.field_evaluate(spec, p6, w.q, w.box)["energy"]
        assert abs(float(e[-1][3]) - pot6) <= 1e-10 * abs(pot6)
        # last trajectory frame = step 6
        txt = (tmp_path / f"{kind}_trajectory.xyz").read_text().split("\n")
        frames = [i for i, l in enumerate(txt) if l.startswith("box ")]
        assert len(frames) == 3 and "step=6" in txt[frames[-1]]
        last = np.array([[float(x) for x in l.split()[1:4]] for l in txt[frames[-1] + 1:frames[-1] + 1 + len(w.q)]])
        assert np.sqrt(((last - p6) ** 2).sum() / (p6 ** 2).sum()) <= 1e-12
    assert run(tmp_path, "compare", "--input", str(inp), "--fields", "msm", "cutoff", "wolf",
               "--a", "10", "--h", "2.5", "--levels", "2", "--cutoff", "9") == 0
    summ = {r[0]: r for r in rows(tmp_path / "compare_summary.csv")[1:]}
    direct = ref.field_evaluate(oracle_lib.fspec("direct", 0.0), w.pos, w.q, w.box)["energy"]
    for kind, spec in [("msm", oracle_lib.fspec("msm", 10.0, 2.5, 2)), ("cutoff", oracle_lib.fspec("cutoff", 9.0)),
                       ("wolf", oracle_lib.fspec("wolf", 9.0, alpha=0.2))]:
        e_ref = float(summ[kind][1])
        assert abs(e_ref - direct) <= 1e-10 * abs(direct)
        got = ref.field_evaluate(spec, w.pos, w.q, w.box)["energy"]
        assert abs(float(summ[kind][2]) - got) <= 1e-10 * abs(got)
    assert len(rows(tmp_path / "compare.csv")) == 1 + 3 * len(w.q)


@pytest.mark.gpu
def test_parareal_cli(tmp_path):
    from paper_1309_1889_b200 import fixtures as fx
    w = fx.config("c1s", n_override=600)
    inp = tmp_path / "in.xyz"
    xyz_io.save_system(pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box), str(inp))
    rc = run(tmp_path, "parareal", "--input", str(inp), "--a", "10", "--h", "2.5", "--levels", "2", "--cutoff", "8",
             "--dt", "0.01", "--steps-per-slice", "4", "--window", "4", "--points", "6", "--max-iter", "6",
             "--tol", "1e-9", "--verify")
    assert rc == 0
    ev = dict((r[0], r[1]) for r in rows(tmp_path / "evals.csv")[1:])
    assert int(ev["windows"]) >= 2 and int(ev["f_evals"]) > 0
    ver = rows(tmp_path / "verify.csv")[1:]
    assert len(ver) == 6 and max(float(r[1]) for r in ver) <= 1e-8
    conv = rows(tmp_path / "convergence.csv")
    assert conv[0] == ["window", "point", "iteration", "delta_rms", "converged"] and len(conv) > 1
