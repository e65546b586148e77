"""Full-size BASELINE configs on one GPU: evaluation + propagate timing and exact checks."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
for name in sys.argv[1:] or ["c5", "c4", "c3"]:
    t0 = time.time()
    w = fx.config(name)
    t1 = time.time()
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    ds = pkg.DeviceSystem(f, s)
    r = ds.evaluate()
    import ctypes
    t2 = time.time()
    r = ds.evaluate()
    t3 = time.time()
    wc = f.work_counters()
    f.set_stage_timing(True); f.reset_stage_times()
    ds.evaluate()
    st = {k: round(v[0], 3) for k, v in f.stage_times().items()}
    f.set_stage_timing(False)
    s2 = pkg.ParticleSystem(w.pos, w.vel, 2.0 * w.q, w.mass, w.box)
    r2 = pkg.DeviceSystem(f, s2).evaluate()
    lin = (np.array_equal(r2.per_particle_potential, 2 * r.per_particle_potential),
           np.array_equal(r2.per_particle_force, 4 * r.per_particle_force), r2.total_energy == 4 * r.total_energy)
    print(f"{name}: n={w.n} gen {t1-t0:.1f}s eval {1e3*(t3-t2):.1f} ms E={r.total_energy:.10e} pairs={wc['pairs']} "
          f"linear={lin} stages={st}", flush=True)
