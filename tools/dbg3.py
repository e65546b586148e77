import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1309_1889_b200 as pkg
from conftest import golden
g = golden("spec500")
f = pkg.MsmField(pkg.MsmConfig(8.0, 2.0, 3))
s = pkg.ParticleSystem(g["pos"], None, g["q"], None, g["box"])
try:
    r = f.evaluate(s); print("ok", r.total_energy, g["energy"])
except pkg.Error as e:
    print(type(e).__name__, e, e.i, e.j, e.step)
    if e.i >= 0: print(g["pos"][e.i], g["pos"][e.j] if e.j >= 0 else None)
