import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx, parallel
w = fx.config("c2s", n_override=30000)
cfg = pkg.MsmConfig(w.a, w.h, w.levels)
s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
for direct in (False, True):
    for steps in (0, 1, 2, 3):
        f = pkg.MsmField(cfg); f.set_lattice_method(direct)
        ds = pkg.DeviceSystem(f, s); ds.propagate(w.dt, steps) if steps else None
        p1, v1 = ds.download()
        e1 = ds.evaluate().total_energy
        dd = parallel.SpatialDecomposition(cfg, s, local_parts=2)
        for _, _, _ in []: pass
        if direct:
            for fld, dsx, _ in dd.parts: fld.set_lattice_method(True)
        out, e = dd.propagate(w.dt, steps)
        print("direct" if direct else "fft", steps, "pos", np.array_equal(out.positions, p1), "vel", np.array_equal(out.velocities, v1),
              "maxdv %.3e" % np.max(np.abs(out.velocities - v1)), "dE %.2e" % ((e - e1) / e1))
    # single-GPU evaluate vs eval-only DD
    f = pkg.MsmField(cfg); f.set_lattice_method(direct)
    r = f.evaluate(s)
    ds = pkg.DeviceSystem(f, s); r2 = ds.evaluate()
    print("evaluate vs system evaluate forces equal:", np.array_equal(r.per_particle_force, r2.per_particle_force))
