import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, ctypes as C
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import _native, fixtures as fx
for name in ["c1s", "c2s"]:
    w = fx.config(name)
    for direct in (0, 1):
        f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
        f.set_lattice_method(bool(direct))
        dev = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
        dev.propagate(w.dt, 3)
        steps = 100 if name == "c1s" else 20
        ms = np.zeros(steps + 2); names = (C.c_char_p * 16)(); l = np.zeros(1, dtype=np.int64)
        _native.lib().msmb_bench_propagate(f.handle, dev._h, w.dt, steps, 1, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                           np.zeros(16).ctypes.data_as(C.POINTER(C.c_double)), names, l.ctypes.data_as(C.POINTER(C.c_int64)))
        f.set_stage_timing(True); f.reset_stage_times(); dev.propagate(w.dt, 5)
        st = f.stage_times()
        print(name, "direct" if direct else "fft", "ms/step %.4f" % np.mean(ms[1:steps + 1]), "lattice %.4f" % (st["lattice"][0] / 6))
