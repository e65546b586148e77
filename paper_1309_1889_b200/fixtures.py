"""Seeded synthetic inputs for the BASELINE.json configurations.

Thin ctypes layer over csrc/fixtures.c (libmsmb_fixtures.so).  Not on the hot
path; used by bench.py and tests/ to build systems in-process.  See
SURVEY.md Appendix B and DESIGN.md "Synthetic inputs" for every choice made
where BASELINE.json leaves a field unspecified.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libmsmb_fixtures.so"
_lib = None
_D = C.POINTER(C.c_double)


def _load():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build()")
        lib = C.CDLL(str(_LIB_PATH))
        lib.fx_uniform.argtypes = [C.c_int64, _D, C.c_int, C.c_double, C.c_uint64, _D, _D]
        lib.fx_rebalanced_charges.argtypes = [C.c_int64, C.c_uint64, _D]
        lib.fx_maxwell_boltzmann.argtypes = [C.c_int64, _D, C.c_double, C.c_double, C.c_uint64, _D]
        lib.fx_water.argtypes = [C.c_int64, _D, C.c_double, C.c_uint64, _D, _D, _D]
        for f in (lib.fx_uniform, lib.fx_rebalanced_charges, lib.fx_maxwell_boltzmann, lib.fx_water):
            f.restype = C.c_int
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(_D)


SCHEMES = {"all_plus_one": 0, "alternating": 1, "random_neutral": 2}


def uniform(n, box, scheme="alternating", min_sep=0.0, seed=1):
    """The reference's generate_random_system (src/generate.cpp:40-93): positions, charges."""
    lib = _load()
    box = np.asarray(box, dtype=np.float64)
    pos = np.zeros((n, 3))
    q = np.zeros(n)
    rc = lib.fx_uniform(n, _p(box), SCHEMES[scheme], float(min_sep), seed, _p(pos), _p(q))
    if rc:
        raise RuntimeError(f"fx_uniform failed rc={rc}")
    return pos, q


def rebalanced_charges(n, seed):
    q = np.zeros(n)
    _load().fx_rebalanced_charges(n, seed, _p(q))
    return q


def maxwell_boltzmann(mass, temperature=300.0, seed=7, energy_to_native=4.184e-4):
    mass = np.ascontiguousarray(mass, dtype=np.float64)
    vel = np.zeros((len(mass), 3))
    _load().fx_maxwell_boltzmann(len(mass), _p(mass), temperature, energy_to_native, seed, _p(vel))
    return vel


def water(n_mol, box, min_oo=0.0, seed=1):
    lib = _load()
    box = np.asarray(box, dtype=np.float64)
    pos = np.zeros((3 * n_mol, 3))
    q = np.zeros(3 * n_mol)
    m = np.zeros(3 * n_mol)
    rc = lib.fx_water(n_mol, _p(box), float(min_oo), seed, _p(pos), _p(q), _p(m))
    if rc:
        raise RuntimeError(f"fx_water failed rc={rc}")
    return pos, q, m


@dataclass
class Workload:
    """A BASELINE.json configuration resolved to concrete arrays + MSM/integrator parameters."""
    name: str
    pos: np.ndarray
    vel: np.ndarray
    q: np.ndarray
    mass: np.ndarray
    box: np.ndarray
    a: float
    h: float
    levels: int
    dt: float
    steps: int
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def n(self):
        return len(self.q)


def config(name: str, seed: int | None = None, n_override: int | None = None) -> Workload:
    """Build one BASELINE.json config by name.

    c1    : configs[0] literal (8,192 atoms, 40 A, alternating, a=10 h=2.5 l=2, dt 2 fs x 200)
    c1s   : c1 survivable variant (RSA min-sep 1.5 A, dt 0.02 fs)  [SURVEY.md 8(d)]
    c2    : configs[1] literal (100,000 waters in a 144 A cube, a=12 h=2.5 l=6, dt 1 fs x 100)
    c2s   : c2 survivable variant (O-O min-sep 2.5 A, dt 0.02 fs)
    c3    : configs[2] (2^24 atoms, 551 A, rebalanced +-1, a=12 h=2.5 l=4, dt 2 fs x 20)
    c3s   : c3 survivable variant (RSA min-sep 1.5 A, dt 0.02 fs)
    c4    : configs[3] (water slab 300x650x650 A, a=12 h=2.5 l=5, dt 2 fs x 20)
    c4s   : c4 survivable variant (O-O min-sep 2.5 A, dt 0.02 fs)
    c5    : configs[4] (2^20 atoms, 219 A, random_neutral; F a=12 h=2.5 l=4 dt .5 x100,
            G a=8 h=5 l=3 dt 2 x25; 8 slices)
    c5s   : c5 survivable parareal variant (RSA min-sep 1.5 A, F dt 0.005 x100, G dt 0.02 x25)
    n_override scales N down at fixed density (for parity tests at oracle-friendly sizes).
    """
    base = name.rstrip("s") if name.endswith("s") and name[:-1] in ("c1", "c2") else name
    surv = name in ("c1s", "c2s")
    if base == "c1":
        seed = 1309 if seed is None else seed
        n = 8192 if n_override is None else n_override
        L = 40.0 * (n / 8192) ** (1 / 3)
        box = np.array([L, L, L])
        pos, q = uniform(n, box, "alternating", 1.5 if surv else 0.0, seed)
        mass = np.full(n, 18.0)
        vel = maxwell_boltzmann(mass, 300.0, seed + 1)
        return Workload(name, pos, vel, q, mass, box, 10.0, 2.5, 2, 0.02 if surv else 2.0, 200)
    if base == "c2":
        seed = 2309 if seed is None else seed
        nm = 100_000 if n_override is None else max(1, n_override // 3)
        L = 144.0 * (nm / 100_000) ** (1 / 3)
        box = np.array([L, L, L])
        pos, q, mass = water(nm, box, 2.5 if surv else 0.0, seed)
        vel = maxwell_boltzmann(mass, 300.0, seed + 1)
        return Workload(name, pos, vel, q, mass, box, 12.0, 2.5, 6, 0.02 if surv else 1.0, 100)
    if base in ("c3", "c3s"):
        # c3s: survivable variant (RSA min-sep 1.5 A, dt 0.02 fs) for multi-step runs
        surv = base == "c3s"
        seed = 3309 if seed is None else seed
        n = 1 << 24 if n_override is None else n_override
        L = 551.0 * (n / (1 << 24)) ** (1 / 3)
        box = np.array([L, L, L])
        pos, _ = uniform(n, box, "all_plus_one", 1.5 if surv else 0.0, seed)
        q = rebalanced_charges(n, seed + 2)
        mass = np.full(n, 18.0)
        vel = maxwell_boltzmann(mass, 300.0, seed + 1)
        return Workload(name, pos, vel, q, mass, box, 12.0, 2.5, 4, 0.02 if surv else 2.0, 20)
    if base in ("c4", "c4s"):
        surv = base == "c4s"
        seed = 4309 if seed is None else seed
        nm = 4_225_000 if n_override is None else max(1, n_override // 3)
        s = (nm / 4_225_000) ** (1 / 3)
        box = np.array([300.0 * s, 650.0 * s, 650.0 * s])
        pos, q, mass = water(nm, box, 2.5 if surv else 0.0, seed)
        vel = maxwell_boltzmann(mass, 300.0, seed + 1)
        return Workload(name, pos, vel, q, mass, box, 12.0, 2.5, 5, 0.02 if surv else 2.0, 20)
    if base in ("c5", "c5s"):
        # c5s: survivable variant for parareal runs: RSA min-sep 1.5 A,
        # fine dt 0.005 fs x 100, coarse dt 0.02 fs x 25 (slice span 0.5 fs, 8 slices)
        surv = base == "c5s"
        seed = 5309 if seed is None else seed
        n = 1 << 20 if n_override is None else n_override
        L = 219.0 * (n / (1 << 20)) ** (1 / 3)
        box = np.array([L, L, L])
        pos, q = uniform(n, box, "random_neutral", 1.5 if surv else 0.0, seed)
        mass = np.full(n, 18.0)
        vel = maxwell_boltzmann(mass, 300.0, seed + 1)
        fdt, gdt = (0.005, 0.02) if surv else (0.5, 2.0)
        w = Workload(name, pos, vel, q, mass, box, 12.0, 2.5, 4, fdt, 100)
        w.extra = dict(coarse=(8.0, 5.0, 3, gdt, 25), fine=(12.0, 2.5, 4, fdt, 100), slices=8)
        return w
    raise ValueError(name)
