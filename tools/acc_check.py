"""Prints the parity errors of one config shape (library chosen by MSMB_LIB)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import oracle_lib
import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx
from conftest import rel_rms, rel_e
port = oracle_lib.checker("port")
for name, n in [("c2s", 30000), ("c2", 30000), ("c4", 45000), ("c5", 40000)]:
    w = fx.config(name, n_override=n)
    f = pkg.MsmField(pkg.MsmConfig(w.a, w.h, w.levels))
    r = f.evaluate(pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box))
    o = port.msm_potential(w.pos, w.q, w.box, w.a, w.h, w.levels)
    print(os.environ.get("MSMB_LIB", "default")[-20:], name, "E %.2e F %.2e phis %.2e phil %.2e" % (
        rel_e(r.total_energy, o["energy"]), rel_rms(r.per_particle_force, o["force"]),
        rel_rms(r.short_part, o["phi_short"]), rel_rms(r.long_part, o["phi_long"])))
