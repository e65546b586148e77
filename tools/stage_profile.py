"""Per-stage times of propagate steps (stage-timing pass: stages serialised, list reused)
for a fixture: python tools/stage_profile.py c3s [steps]."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
name = sys.argv[1] if len(sys.argv) > 1 else "c3s"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t0 = time.time()
w = fx.config(name)
f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
dev = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
dev.propagate(w.dt, 2)
f.set_stage_timing(True)
f.reset_stage_times()
dev.propagate(w.dt, steps)
st = f.stage_times()
print(name, f"n={w.n} setup {time.time() - t0:.1f}s", {k: round(v[0] / (steps + 1), 3) for k, v in st.items()})
