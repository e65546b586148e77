"""Writes tests/golden/*.npz from the REFERENCE library itself.

Runs the unmodified reference (`paramd`, compiled from /root/reference/proj/src
by oracle/Makefile into oracle/_ref/libparamd_ref.so) on small seeded inputs and
stores inputs + outputs.  The reference ships no golden files or tests
(SURVEY.md 4), so these are the pins for the oracle restatement and for the GPU
path.  Re-run with:  python tests/golden/make_golden.py   (needs /root/reference).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_lib  # noqa: E402
from paper_1309_1889_b200 import fixtures as fx  # noqa: E402


def main():
    ref = oracle_lib.checker("ref")
    out = {}

    # SPEC acceptance-1 fixture: 500 atoms, random_neutral, seed 42,
    # 40 A box, min-sep 1.5, a=8 h=2 l=3 -- the reference gives U=-597.6718.
    box = np.array([40.0, 40.0, 40.0])
    pos, q = fx.uniform(500, box, "random_neutral", 1.5, 42)
    r = ref.msm_potential(pos, q, box, 8.0, 2.0, 3, diag=True)
    np.savez_compressed(HERE / "spec500.npz", pos=pos, q=q, box=box, a=8.0, h=2.0, levels=3, **r)
    out["spec500"] = r["energy"]

    # direct Coulomb on the same fixture (the reference's accuracy oracle)
    import ctypes as C
    n = len(q)
    phi, f, e = np.zeros(n), np.zeros((n, 3)), np.zeros(1)
    buf = C.create_string_buffer(256)
    ref.lib.ref_direct_coulomb(n, oracle_lib._p(pos), oracle_lib._p(q), 332.0636, oracle_lib._p(phi),
                               oracle_lib._p(f), oracle_lib._p(e), buf, 256)
    np.savez_compressed(HERE / "spec500_direct.npz", phi=phi, force=f, energy=e[0])

    # config-shaped small systems
    for name, nov, levels in [("c1", 1024, None), ("c2", 1500, 3), ("c5", 1200, None), ("c3", 1000, None)]:
        w = fx.config(name, n_override=nov)
        L = levels or w.levels
        r = ref.msm_potential(w.pos, w.q, w.box, w.a, w.h, L, diag=True)
        np.savez_compressed(HERE / f"{name}_small.npz", pos=w.pos, q=w.q, box=w.box, a=w.a, h=w.h,
                            levels=L, **r)
        out[name] = r["energy"]

    # trajectory (survivable variant) and a literal-input abort
    w = fx.config("c1s", n_override=512)
    p2, v2, done, err = ref.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, 10)
    assert err is None
    np.savez_compressed(HERE / "c1s_traj10.npz", pos=w.pos, vel=w.vel, q=w.q, mass=w.mass, box=w.box,
                        a=w.a, h=w.h, levels=w.levels, dt=w.dt, steps=10, out_pos=p2, out_vel=v2)
    w = fx.config("c1", n_override=1024)
    p2, v2, done, err = ref.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, 50)
    np.savez_compressed(HERE / "c1_abort.npz", pos=w.pos, vel=w.vel, q=w.q, mass=w.mass, box=w.box,
                        a=w.a, h=w.h, levels=w.levels, dt=w.dt, steps=50, steps_done=done,
                        err_code=err.code if err else 0, err_msg=str(err.msg if err else ""))
    out["c1_abort"] = (done, str(err))

    # error precedence cases on the SPEC fixture
    cases = {}
    p = pos.copy(); p[100] = p[7]; p[50] = p[20]; cases["coincident"] = p
    p = pos.copy(); p[300, 1] = np.nan; p[200, 0] = -5; cases["nan"] = p
    p = pos.copy(); p[300, 1] = -2.1; p[200, 0] = 42.0; p[250, 2] = -2.0; cases["coverage"] = p
    p = pos.copy(); p[300, 1] = np.inf; p[200, 1] = np.inf; cases["inf_pair"] = p
    p = pos.copy(); p[10] = p[400]; p[400, 0] = np.nan; cases["coincident_vs_nan"] = p
    err_rows = {}
    for k, p in cases.items():
        try:
            ref.msm_potential(p, q, box, 8.0, 2.0, 3)
            err_rows[k] = (0, "")
        except oracle_lib.OracleError as e:
            err_rows[k] = (e.code, e.msg)
    np.savez_compressed(HERE / "errors.npz", q=q, box=box,
                        **{f"pos_{k}": v for k, v in cases.items()},
                        **{f"code_{k}": np.int64(v[0]) for k, v in err_rows.items()},
                        **{f"msg_{k}": np.array(v[1]) for k, v in err_rows.items()})
    out["errors"] = err_rows

    # parareal: one window, T=4, K=2, scaled survivable fixture
    pos_p, q_p = fx.uniform(256, np.array([13.7, 13.7, 13.7]), "random_neutral", 1.5, 77)
    mass_p = np.full(256, 18.0)
    vel_p = fx.maxwell_boltzmann(mass_p, 300.0, 78)
    box_p = np.array([13.7, 13.7, 13.7])
    fine = (12.0, 2.5, 3, 0.005, 20)
    coarse = (8.0, 5.0, 2, 0.02, 5)
    rp, rv, dr, cnt = ref.parareal_window(pos_p, vel_p, q_p, mass_p, box_p, fine, coarse, 4, 2)
    np.savez_compressed(HERE / "parareal_w4k2.npz", pos=pos_p, vel=vel_p, q=q_p, mass=mass_p, box=box_p,
                        fine=np.array(fine), coarse=np.array(coarse), row_pos=rp, row_vel=rv,
                        delta_rms=dr, counts=cnt)
    out["parareal"] = list(cnt)

    # kernel-math KATs from the reference
    kat = {}
    for name, (which, x, a, k, l) in {"gamma0": (0, 0.0, 1, 0, 1), "gamma1": (0, 1.0, 1, 0, 1),
                                      "gamma2": (0, 2.0, 1, 0, 1), "gstar_half": (2, 0.5, 1.0, 0, 1),
                                      "phi_half": (5, 0.5, 1, 0, 1), "phi_1p5": (5, 1.5, 1, 0, 1),
                                      "glevel_0_2": (4, 3.0, 8.0, 0, 2), "glevel_top": (4, 3.0, 8.0, 1, 2),
                                      "dphi_m03": (6, -0.3, 1, 0, 1), "dgstar": (3, 2.0, 5.0, 0, 1)}.items():
        kat[name] = ref.kernel(which, x, a, k, l)
    np.savez_compressed(HERE / "kats.npz", **{k: np.float64(v) for k, v in kat.items()})
    for k, v in out.items():
        print(k, v)


if __name__ == "__main__":
    main()
