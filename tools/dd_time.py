import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx, parallel
w = fx.config("c3s")
s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
dd = parallel.SpatialDecomposition(pkg.MsmConfig(w.a, w.h, w.levels), s, device=0)
dd.propagate(w.dt, 2, download=False)
T = {}
orig_phase, orig_ex = dd._phase, dd._exchange
def tp(phase, *a, **k):
    t0 = time.perf_counter(); r = orig_phase(phase, *a, **k); torch.cuda.synchronize()
    T["phase%d" % phase] = T.get("phase%d" % phase, 0) + time.perf_counter() - t0; return r
def te(which, *a, **k):
    t0 = time.perf_counter(); r = orig_ex(which, *a, **k); torch.cuda.synchronize()
    T["ex%d" % which] = T.get("ex%d" % which, 0) + time.perf_counter() - t0; return r
dd._phase, dd._exchange = tp, te
t0 = time.perf_counter()
dd.propagate(w.dt, 4, download=False)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print("total ms/step", 1e3 * tot / 5, {k: round(1e3 * v / 5, 2) for k, v in T.items()})
