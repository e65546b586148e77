"""Times one C2-S evaluation's stages with the library selected by MSMB_LIB."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
w = fx.config(sys.argv[1] if len(sys.argv) > 1 else "c2s")
f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
dev = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
dev.propagate(w.dt, 2)
f.set_stage_timing(True); f.reset_stage_times()
dev.propagate(w.dt, 10)
st = f.stage_times()
print(os.environ.get("MSMB_LIB", "default"), " ".join(f"{k}={v[0]/11:.4f}" for k, v in st.items() if k in ("pairs", "clusters", "lattice", "anterp", "restrict", "top", "prolong", "sort", "interp")))
