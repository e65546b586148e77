"""Helpers for the GPU parity tests."""
import numpy as np

import paper_1309_1889_b200 as pkg
from paper_1309_1889_b200 import fixtures as fx


def system(w):
    return pkg.ParticleSystem(w.pos, w.vel, w.q, w.mass, w.box)


def field(w, levels=None):
    return pkg.MsmField(pkg.MsmConfig(w.a, w.h, levels or w.levels), pkg.UnitsConfig.physical())


def level_slices(cfg, box):
    dims, _, _ = pkg.grid_geometry(cfg, box)
    sizes = [int(np.prod(d)) for d in dims]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    return [slice(offs[k], offs[k + 1]) for k in range(len(sizes))], dims
