import sys, time, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
import oracle_lib
port = oracle_lib.checker('port')
def rel(a,b): return float(np.sqrt(np.sum((a-b)**2)/np.sum(b**2)))
for name, nov in [('c2s', None), ('c2', None), ('c2s', 100000)]:
    w = fx.config(name, n_override=nov)
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
    r = f.evaluate(s)
    o = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels, diag=True)
    print(name, w.n, 'dE', abs(r.total_energy-o['energy'])/abs(o['energy']), 'dF', rel(r.per_particle_force, o['force']),
          'dphis', rel(r.short_part, o['phi_short']), 'dphil', rel(r.long_part, o['phi_long']), f.work_counters(), flush=True)
    d = np.abs(r.short_part - o['phi_short'])
    bad = np.argsort(d)[-5:]
    print('  worst phis', bad, d[bad], o['phi_short'][bad])
    gc, gp = f.debug_levels()
    print('  levels charge rel', rel(gc, o['level_charge']), 'pot rel', rel(gp, o['level_potential']))
    dev = pkg.DeviceSystem(f, s)
    r2 = dev.evaluate()
    print('  device evaluate same', np.array_equal(r2.per_particle_force, r.per_particle_force))
    try:
        dev.propagate(w.dt, 1); print('  dev propagate 1 ok')
    except pkg.Error as e:
        print('  dev propagate 1 FAILED', type(e).__name__, e, e.step)
    try:
        out = pkg.propagate(pkg.PropagatorSpec(f, w.dt, 1), s); print('  host propagate 1 ok')
    except pkg.Error as e:
        print('  host propagate 1 FAILED', type(e).__name__, e, e.step)
