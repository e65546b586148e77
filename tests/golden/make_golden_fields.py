"""Writes tests/golden/fields*.npz from the REFERENCE library itself.

The pair-only fields (SimpleCutoffField, WolfField, DirectCoulombField, and the
PairRepulsionOverlay around them; src/electrostatics.cpp, src/force_field.cpp:45-68)
evaluated by the unmodified reference (oracle/_ref/libparamd_ref.so) on seeded
inputs, plus a cutoff-field trajectory and a parareal window with an MSM fine
and a cutoff coarse propagator (the CLI's default pairing, tools/paramd_main.cpp:417).
Re-run with:  python tests/golden/make_golden_fields.py   (needs /root/reference).
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
from oracle_lib import fspec  # noqa: E402
from paper_1309_1889_b200 import fixtures as fx  # noqa: E402

# (name, fspec) of the evaluated fields
FIELDS = [
    ("cutoff10", fspec("cutoff", 10.0)),
    ("cutoff7", fspec("cutoff", 7.0)),
    ("wolf10", fspec("wolf", 10.0, alpha=0.2)),
    ("wolf8_a0", fspec("wolf", 8.0, alpha=0.0)),
    ("direct", fspec("direct", 0.0)),
    ("cutoff10_rep", fspec("cutoff", 10.0, rep_eps=0.1, rep_sigma=2.0)),
    ("direct_rep", fspec("direct", 0.0, rep_eps=1.0, rep_sigma=2.5)),
]


def main():
    ref = oracle_lib.checker("ref")
    w = fx.config("c1s", n_override=1536)
    out = dict(pos=w.pos, q=w.q, box=w.box, names=np.array([n for n, _ in FIELDS]),
               specs=np.stack([s for _, s in FIELDS]))
    for name, spec in FIELDS:
        r = ref.field_evaluate(spec, w.pos, w.q, w.box)
        out[f"{name}_phi"], out[f"{name}_force"], out[f"{name}_energy"] = r["phi"], r["force"], r["energy"]
        print(name, r["energy"])
    np.savez_compressed(HERE / "fields.npz", **out)

    # cutoff-field trajectory: 10 Verlet steps of the survivable C1 variant
    w = fx.config("c1s", n_override=768)
    spec = fspec("cutoff", 10.0)
    p2, v2, done, err = ref.field_propagate(spec, w.pos, w.vel, w.q, w.mass, w.box, w.dt, 10)
    assert err is None and done == 10
    np.savez_compressed(HERE / "fields_traj10.npz", spec=spec, pos=w.pos, vel=w.vel, q=w.q, mass=w.mass,
                        box=w.box, dt=w.dt, steps=10, out_pos=p2, out_vel=v2)

    # parareal window: F = MSM a=10 h=2.5 l=2 (dt 0.005 x 8), G = cutoff 8 A (dt 0.02 x 2)
    w = fx.config("c1s", n_override=384)
    fs, gs = fspec("msm", 10.0, 2.5, 2), fspec("cutoff", 8.0)
    rp, rv, dr, cnt = ref.field_parareal_window(w.pos, w.vel, w.q, w.mass, w.box, fs, 0.005, 8, gs, 0.02, 2,
                                                4, 2)
    np.savez_compressed(HERE / "fields_parareal_w4k2.npz", pos=w.pos, vel=w.vel, q=w.q, mass=w.mass, box=w.box,
                        fine=fs, fdt=0.005, fsteps=8, coarse=gs, gdt=0.02, gsteps=2, t_points=4, k_iters=2,
                        row_pos=rp, row_vel=rv, delta_rms=dr, counts=cnt)


if __name__ == "__main__":
    main()
