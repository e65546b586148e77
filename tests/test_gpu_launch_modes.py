"""Launch-mode independence of the results: programmatic dependent launch on or off, any
dense threshold and the stream priorities only change WHEN kernels run, never what they
compute -- a propagated trajectory must be bit for bit the same.  The knobs are read once per
process, so every variant runs in its own interpreter."""
import hashlib
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, %r)
import numpy as np
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
out = []
for name, n, steps in (("c1s", None, 6), ("c2s", 30000, 4)):
    w = fx.config(name, n_override=n)
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels), pkg.UnitsConfig.physical(), device=0)
    r = f.evaluate(s)
    p = pkg.propagate(pkg.PropagatorSpec(f, w.dt, steps), s)
    h = hashlib.sha256()
    for a in (np.float64(r.total_energy), r.per_particle_force, p.positions, p.velocities):
        h.update(np.ascontiguousarray(a).tobytes())
    out.append(h.hexdigest())
print(" ".join(out))
""" % str(ROOT)


def _run(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


def test_pdl_and_priorities_do_not_change_results():
    base = _run({})
    assert _run({"MSMB_PDL": "0"}) == base
    assert _run({"MSMB_SIDE_PRIO": "equal"}) == base
    assert _run({"MSMB_FFT_LINES": "2"}) == base


def test_repeatable_across_processes():
    assert _run({}) == _run({})
