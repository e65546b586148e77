import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx, parallel
w = fx.config("c2s", n_override=30000)
cfg = pkg.MsmConfig(w.a, w.h, w.levels)
s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
def single(steps, eager=False):
    f = pkg.MsmField(cfg)
    ds = pkg.DeviceSystem(f, s)
    if eager: f.set_stage_timing(True)
    ds.propagate(w.dt, steps)
    return ds.download()
a = single(2); b = single(2); c = single(2, eager=True)
print("graph run-to-run", np.array_equal(a[1], b[1]), " graph vs eager", np.array_equal(a[1], c[1]), np.max(np.abs(a[1]-c[1])))
for parts in (1, 2):
    r1 = parallel.SpatialDecomposition(cfg, s, local_parts=parts).propagate(w.dt, 2)[0]
    r2 = parallel.SpatialDecomposition(cfg, s, local_parts=parts).propagate(w.dt, 2)[0]
    print("dd", parts, "run-to-run", np.array_equal(r1.velocities, r2.velocities), "vs graph", np.array_equal(r1.velocities, a[1]), "vs eager", np.array_equal(r1.velocities, c[1]))
