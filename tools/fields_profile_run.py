"""One small run per field for ncu captures (tools/ncu_summary.py): `cutoff` / `wolf`
propagate C2-S for 3 steps, `direct` evaluates N = 65536 twice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx

which = sys.argv[1]
if which in ("cutoff", "wolf"):
    w = fx.config("c2s")
    f = pkg.SimpleCutoffField(pkg.CutoffParams(12.0)) if which == "cutoff" else pkg.WolfField(pkg.CutoffParams(12.0, 0.2))
    dev = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
    dev.propagate(w.dt, 3)
else:
    n = 65536
    rng = np.random.default_rng(1)
    L = (n / 0.1) ** (1 / 3)
    s = pkg.ParticleSystem(rng.uniform(0, L, (n, 3)), None, rng.choice([-1.0, 1.0], n), None, np.array([L] * 3))
    f = pkg.DirectCoulombField()
    dev = pkg.DeviceSystem(f, s)
    dev.evaluate()
    dev.evaluate()
