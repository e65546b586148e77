"""One C3 evaluation (for ncu captures of the full-size kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
w = fx.config(sys.argv[1] if len(sys.argv) > 1 else "c3")
f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
ds = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
ds.evaluate(outputs=False)
print("ok")
