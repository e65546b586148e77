"""Prints one C2-S evaluation's work counters with the library selected by MSMB_LIB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
w = fx.config(sys.argv[1] if len(sys.argv) > 1 else "c2s")
f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
dev = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
dev.propagate(w.dt, 1)
print(os.environ.get("MSMB_LIB", "default"), f.work_counters())
