import sys, time, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
import oracle_lib
port = oracle_lib.checker('port')
def rel(a,b): return float(np.sqrt(np.sum((a-b)**2)/np.sum(b**2)))
w = fx.config('c2s')
for trial in range(3):
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    dev = pkg.DeviceSystem(f, s)
    try:
        dev.propagate(w.dt, 2); print(trial, 'dev propagate 2 ok', f.work_counters(), flush=True)
        p, v = dev.download()
    except pkg.Error as e:
        print(trial, 'dev propagate 2 FAILED', type(e).__name__, e, 'step', e.step, flush=True)
        p = None
    if trial == 0 and p is not None:
        p2, v2, done, err = port.propagate(w.pos, w.vel, w.q, w.mass, w.box, w.a, w.h, w.levels, w.dt, 2)
        print('  vs port dx', rel(p, p2), 'dv', rel(v, v2), flush=True)
    try:
        dev.propagate(w.dt, 10); print(trial, 'dev propagate 10 more ok', flush=True)
    except pkg.Error as e:
        print(trial, 'dev propagate 10 FAILED', type(e).__name__, e, 'step', e.step, flush=True)
    del dev, f
