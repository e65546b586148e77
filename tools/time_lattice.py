"""Stage times of one C2-S evaluation with the FFT and the direct lattice cutoff."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
name = sys.argv[1] if len(sys.argv) > 1 else "c2s"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = fx.config(name, n_override=n)
for direct in (False, True):
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    f.set_lattice_method(direct)
    dev = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
    dev.propagate(w.dt, 1)
    f.set_stage_timing(True); f.reset_stage_times()
    dev.propagate(w.dt, 4)
    st = f.stage_times()
    print(name, "direct" if direct else "fft", " ".join(f"{k}={v[0]/5:.4f}" for k, v in st.items()))
