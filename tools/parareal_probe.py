"""C5-S parareal (K=1) timing with and without pair-list reuse across propagate calls:
python tools/parareal_probe.py"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1309_1889_b200 as pkg  # noqa: E402
from paper_1309_1889_b200 import fixtures as fx, parallel  # noqa: E402

w = fx.config("c5s")
fa, fh, fl, fdt, fs = w.extra["fine"]
ga, gh, gl, gdt, gs = w.extra["coarse"]
s = pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)
for reuse in (False, True, False):
    F = pkg.MsmField(pkg.MsmConfig(fa, fh, fl))
    G = pkg.MsmField(pkg.MsmConfig(ga, gh, gl))
    F.set_list_reuse(reuse)
    G.set_list_reuse(reuse)
    cfg = pkg.PararealConfig(8, 1, 1e300, pkg.PropagatorSpec(F, fdt, fs), pkg.PropagatorSpec(G, gdt, gs),
                             short_circuit=False)
    pkg.propagate(pkg.PropagatorSpec(F, fdt, 2), s)
    pkg.propagate(pkg.PropagatorSpec(G, gdt, 2), s)
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = parallel.parareal_run(s, 8, cfg)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    t = time.perf_counter()
    pkg.propagate(pkg.PropagatorSpec(F, fdt, fs), s)
    one_f = time.perf_counter() - t
    t = time.perf_counter()
    pkg.propagate(pkg.PropagatorSpec(G, gdt, gs), s)
    one_g = time.perf_counter() - t
    print(f"reuse={reuse}: parareal {el:.3f} s, rebuilds F {F.work_counters()['list_rebuilds']} "
          f"G {G.work_counters()['list_rebuilds']}; one F slice {one_f*1e3:.1f} ms, one G slice {one_g*1e3:.1f} ms",
          flush=True)
