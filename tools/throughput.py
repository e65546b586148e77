"""Single-GPU propagate throughput of the full-size BASELINE configs (survivable
variants): atom-steps/s = N x steps / wall time of one device-resident propagate
call of `steps` steps (its initial evaluation included), after a
2-step warm-up call (graphs, pair list).  Usage: python tools/throughput.py c3s c4s"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx

for name in sys.argv[1:] or ["c3s", "c4s"]:
    t0 = time.time()
    w = fx.config(name)
    gen = time.time() - t0
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    ds = pkg.DeviceSystem(f, pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
    ds.propagate(w.dt, 2)
    steps = w.steps
    t0 = time.perf_counter()
    ds.propagate(w.dt, steps)
    t = time.perf_counter() - t0
    wc = f.work_counters()
    print(json.dumps({"config": name, "n_atoms": int(w.n), "steps": steps, "dt_fs": w.dt, "seconds": t,
                      "ms_per_step": 1e3 * t / steps, "atom_steps_per_s": w.n * steps / t,
                      "pairs_per_eval": wc["pairs"], "list_rebuilds": wc["list_rebuilds"],
                      "generate_s": round(gen, 1)}), flush=True)
