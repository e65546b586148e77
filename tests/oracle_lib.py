"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``ref``  -- oracle/_ref/libparamd_ref.so: the unmodified reference library
  (compiled from /root/reference/proj/src by oracle/Makefile) behind
  oracle/ref_shim.cpp.
* ``port`` -- oracle/liboracle.so: the plain-C restatement (oracle/msm_oracle.c).

Both expose the same functions (``ref_*`` / ``orc_*``) with identical
signatures, wrapped here by :class:`Checker` so tests can run either.
Only tests/, bench.py (cpu_baseline / --impl reference) and
__graft_entry__.smoke() import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libparamd_ref.so"
PORT_SO = ROOT / "oracle" / "liboracle.so"

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_L = C.POINTER(C.c_int64)
_S = C.c_char_p
i64, i32, f64 = C.c_int64, C.c_int, C.c_double

ERR_NAMES = {0: "ok", 1: "ConfigError", 2: "DomainError", 3: "CoverageError",
             4: "CoincidentParticlesError", 5: "HierarchyError", 6: "RuntimeFault",
             7: "NonConvergenceError", 9: "Error"}

_SIGS = {
    "msm_potential": [i64, _D, _D, _D, f64, f64, i32, i32, i32, f64, f64, _D, _D, _D, _D, _D, _D, _D, _S, i32],
    "grid_geometry": [_D, f64, f64, i32, i32, i32, _I, _D, _D, _S, i32],
    "short_range": [i64, _D, _D, f64, f64, _D, _D, _S, i32],
    "anterpolate": [i64, _D, _D, _D, f64, f64, i32, _D, _S, i32],
    "restrict": [_D, f64, f64, i32, i32, _D, _D, _S, i32],
    "lattice_cutoff": [_D, f64, f64, i32, i32, _D, _D, _S, i32],
    "top_level": [_D, f64, f64, i32, _D, _D, _S, i32],
    "prolongate": [_D, f64, f64, i32, i32, _D, _D, _S, i32],
    "interpolate": [i64, _D, _D, f64, f64, i32, _D, _D, _S, i32],
    "parareal_window": [i64, _D, _D, _D, _D, _D, f64, f64, i32, f64, i32, f64, f64, i32, f64, i32,
                        f64, f64, i32, i32, i32, _D, _D, _D, _L, _S, i32],
    "parareal_run": [i64, _D, _D, _D, _D, _D, f64, f64, i32, f64, i32, f64, f64, i32, f64, i32,
                     f64, f64, i32, i32, f64, i32, f64, i32, i32, _D, _D, _L, _S, i32],
    # any ForceField, described by fspec() below
    "field_evaluate": [_D, i64, _D, _D, _D, f64, f64, _D, _D, _D, _S, i32],
    "field_parareal_window": [i64, _D, _D, _D, _D, _D, _D, f64, i32, _D, f64, i32, f64, f64, i32, i32,
                              _D, _D, _D, _L, _S, i32],
}


def fspec(kind: str, a: float, h: float = 0.0, levels: int = 0, alpha=None, rep_eps: float = 0.0,
          rep_sigma: float = 1.0) -> np.ndarray:
    """Field description shared by ref_field_* / orc_field_*: kind 'msm' | 'cutoff' | 'wolf' |
    'direct'; a = MsmConfig::cutoff_a or CutoffParams::cutoff; rep_eps > 0 wraps the field in
    PairRepulsionOverlay(rep_eps, rep_sigma)."""
    k = {"msm": 0, "cutoff": 1, "wolf": 2, "direct": 3}[kind]
    return np.array([k, a, h, levels, 0.0 if alpha is None else 1.0, alpha or 0.0, rep_eps, rep_sigma],
                    dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, str(code))
        self.msg = msg


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(_D)


def _pl(a):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_L)


class Checker:
    """One CPU checker library (``kind`` = 'ref' or 'port')."""

    def __init__(self, kind: str):
        self.kind = kind
        path = REF_SO if kind == "ref" else PORT_SO
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(str(path))
        pre = "ref_" if kind == "ref" else "orc_"
        self.f = {}
        for name, args in _SIGS.items():
            fn = getattr(self.lib, pre + name)
            fn.argtypes = args
            fn.restype = C.c_int
            self.f[name] = fn
        if kind == "ref":
            k = self.lib.ref_kernel_eval
            k.argtypes = [i32, f64, f64, i32, i32, _D, _S, i32]
            k.restype = C.c_int
            self.lib.ref_msm_flops_general.argtypes = [f64, f64, f64, f64, f64]
            self.lib.ref_msm_flops_general.restype = f64
            self.lib.ref_msm_flops_simplified.argtypes = [f64, f64, f64]
            self.lib.ref_msm_flops_simplified.restype = f64
            self.lib.ref_time_short_range.argtypes = [i64, _D, _D, f64, f64, i32]
            self.lib.ref_time_short_range.restype = f64
            g = self.lib.ref_generate_random_system
            g.argtypes = [i64, _D, i32, f64, C.c_uint64, _D, _D, _S, i32]
            g.restype = C.c_int
            pt = self.lib.ref_propagate_trace
            pt.argtypes = [i64, _D, _D, _D, _D, _D, f64, f64, i32, f64, f64, f64, i32, _I, _S, i32]
            pt.restype = C.c_int
            fp = self.lib.ref_field_propagate_trace
            fp.argtypes = [_D, i64, _D, _D, _D, _D, _D, f64, f64, f64, i32, _I, _S, i32]
            fp.restype = C.c_int
            self.lib.ref_field_cost.argtypes = [_D, f64, f64, i64]
            self.lib.ref_field_cost.restype = f64
            dc = self.lib.ref_direct_coulomb
            dc.argtypes = [i64, _D, _D, f64, _D, _D, _D, _S, i32]
            dc.restype = C.c_int
        else:
            k = self.lib.orc_kernel
            k.argtypes = [i32, f64, f64, i32, i32]
            k.restype = f64
            pp = self.lib.orc_propagate
            pp.argtypes = [i64, _D, _D, _D, _D, _D, f64, f64, i32, f64, f64, f64, i32, _I, _S, i32]
            pp.restype = C.c_int
            self.lib.orc_num_threads.restype = C.c_int
            fp = self.lib.orc_field_propagate
            fp.argtypes = [_D, i64, _D, _D, _D, _D, _D, f64, f64, f64, i32, _I, _S, i32]
            fp.restype = C.c_int
            lr = self.lib.orc_long_range
            lr.argtypes = [i64, _D, _D, _D, f64, f64, i32, f64, _D, _D, _D, _S, i32]
            lr.restype = C.c_int

    # -------------------------------------------------------------- helpers
    @staticmethod
    def _call(fn, *args):
        buf = C.create_string_buffer(512)
        rc = fn(*args, buf, 512)
        if rc != 0:
            raise OracleError(rc, buf.value.decode())

    def kernel(self, which: int, x: float, a: float = 1.0, k: int = 0, l: int = 1) -> float:
        if self.kind == "port":
            return self.lib.orc_kernel(which, x, a, k, l)
        out = C.c_double()
        self._call(self.lib.ref_kernel_eval, which, x, a, k, l, C.byref(out))
        return out.value

    def grid_geometry(self, box, a, h, levels, p=3, m=2):
        dims = (C.c_int * (3 * levels))()
        sp = np.zeros(levels)
        org = np.zeros(3 * levels)
        self._call(self.f["grid_geometry"], _p(np.asarray(box, dtype=np.float64)), a, h, levels, p, m,
                   dims, _p(sp), _p(org))
        return np.array(list(dims)).reshape(levels, 3), sp, org.reshape(levels, 3)

    def msm_potential(self, pos, q, box, a, h, levels, kc=332.0636, conv=4.184e-4, p=3, m=2,
                      diag=False):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64)
        n = len(q)
        box = np.asarray(box, dtype=np.float64)
        phi, ps, pl = np.zeros(n), np.zeros(n), np.zeros(n)
        f = np.zeros((n, 3))
        e = np.zeros(1)
        lc = lp = None
        if diag:
            dims, _, _ = self.grid_geometry(box, a, h, levels, p, m)
            tot = int(sum(int(np.prod(d)) for d in dims))
            lc, lp = np.zeros(tot), np.zeros(tot)
        self._call(self.f["msm_potential"], n, _p(pos), _p(q), _p(box), a, h, levels, p, m, kc, conv,
                   _p(phi), _p(ps), _p(pl), _p(f), _p(e), _p(lc), _p(lp))
        out = dict(phi=phi, phi_short=ps, phi_long=pl, force=f, energy=float(e[0]))
        if diag:
            out["level_charge"], out["level_potential"] = lc, lp
        return out

    def short_range(self, pos, q, a, kc=332.0636):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64)
        phi, f = np.zeros(len(q)), np.zeros((len(q), 3))
        self._call(self.f["short_range"], len(q), _p(pos), _p(q), a, kc, _p(phi), _p(f))
        return phi, f

    def anterpolate(self, pos, q, box, a, h, levels):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64)
        box = np.asarray(box, dtype=np.float64)
        dims, _, _ = self.grid_geometry(box, a, h, levels)
        out = np.zeros(int(np.prod(dims[0])))
        self._call(self.f["anterpolate"], len(q), _p(pos), _p(q), _p(box), a, h, levels, _p(out))
        return out

    def restrict(self, box, a, h, levels, k, fine):
        box = np.asarray(box, dtype=np.float64)
        dims, _, _ = self.grid_geometry(box, a, h, levels)
        out = np.zeros(int(np.prod(dims[k + 1])))
        self._call(self.f["restrict"], _p(box), a, h, levels, k, _p(np.ascontiguousarray(fine)), _p(out))
        return out

    def lattice_cutoff(self, box, a, h, levels, k, charge):
        box = np.asarray(box, dtype=np.float64)
        out = np.zeros(len(charge))
        self._call(self.f["lattice_cutoff"], _p(box), a, h, levels, k, _p(np.ascontiguousarray(charge)), _p(out))
        return out

    def top_level(self, box, a, h, levels, charge):
        box = np.asarray(box, dtype=np.float64)
        out = np.zeros(len(charge))
        self._call(self.f["top_level"], _p(box), a, h, levels, _p(np.ascontiguousarray(charge)), _p(out))
        return out

    def prolongate(self, box, a, h, levels, k, coarse_pot, fine_pot):
        box = np.asarray(box, dtype=np.float64)
        fine = np.array(fine_pot, dtype=np.float64, copy=True)
        self._call(self.f["prolongate"], _p(box), a, h, levels, k, _p(np.ascontiguousarray(coarse_pot)), _p(fine))
        return fine

    def interpolate(self, pos, box, a, h, levels, pot0):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        box = np.asarray(box, dtype=np.float64)
        out = np.zeros(len(pos))
        self._call(self.f["interpolate"], len(pos), _p(pos), _p(box), a, h, levels, _p(np.ascontiguousarray(pot0)), _p(out))
        return out

    def long_range(self, pos, q, box, a, h, levels, pot0, kc=332.0636):
        """(port only) u_long and the long-range forces of msm_potential (src/msm.cpp:16-48,
        69-78) from a given level-0 potential."""
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64)
        box = np.asarray(box, dtype=np.float64)
        u, f = np.zeros(len(q)), np.zeros((len(q), 3))
        self._call(self.lib.orc_long_range, len(q), _p(pos), _p(q), _p(box), a, h, levels, kc,
                   _p(np.ascontiguousarray(pot0, dtype=np.float64)), _p(u), _p(f))
        return u, f

    def propagate(self, pos, vel, q, mass, box, a, h, levels, dt, steps, kc=332.0636, conv=4.184e-4):
        """Returns (pos, vel, steps_done, error-or-None)."""
        pos = np.array(pos, dtype=np.float64, copy=True).reshape(-1, 3)
        vel = np.array(vel, dtype=np.float64, copy=True).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64)
        mass = np.ascontiguousarray(mass, dtype=np.float64)
        box = np.asarray(box, dtype=np.float64)
        done = C.c_int(0)
        buf = C.create_string_buffer(512)
        fn = self.lib.ref_propagate_trace if self.kind == "ref" else self.lib.orc_propagate
        rc = fn(len(q), _p(pos), _p(vel), _p(q), _p(mass), _p(box), a, h, levels, kc, conv, dt, steps,
                C.byref(done), buf, 512)
        err = None if rc == 0 else OracleError(rc, buf.value.decode())
        return pos, vel, done.value, err

    def parareal_window(self, pos, vel, q, mass, box, fine, coarse, t_points, k_iters,
                        kc=332.0636, conv=4.184e-4, threads=1):
        """fine/coarse = (a, h, levels, dt, steps). Returns (row_pos[t+1,n,3], row_vel, delta_rms, counts)."""
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        vel = np.ascontiguousarray(vel, dtype=np.float64).reshape(-1, 3)
        n = len(pos)
        rp = np.zeros((t_points + 1, n, 3))
        rv = np.zeros((t_points + 1, n, 3))
        dr = np.zeros(t_points + 1)
        cnt = np.zeros(3, dtype=np.int64)
        fa, fh, fl, fdt, fs = fine
        ga, gh, gl, gdt, gs = coarse
        self._call(self.f["parareal_window"], n, _p(pos), _p(vel), _p(np.ascontiguousarray(q, dtype=np.float64)),
                   _p(np.ascontiguousarray(mass, dtype=np.float64)), _p(np.asarray(box, dtype=np.float64)),
                   fa, fh, fl, fdt, fs, ga, gh, gl, gdt, gs, kc, conv, t_points, k_iters, threads,
                   _p(rp), _p(rv), _p(dr), _pl(cnt))
        return rp, rv, dr, cnt

    def parareal_run(self, pos, vel, q, mass, box, fine, coarse, window, max_iter, tol,
                     total_points, short_circuit=True, skip_threshold=-1.0, kc=332.0636,
                     conv=4.184e-4, threads=1):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        vel = np.ascontiguousarray(vel, dtype=np.float64).reshape(-1, 3)
        n = len(pos)
        tp = np.zeros((total_points, n, 3))
        tv = np.zeros((total_points, n, 3))
        cnt = np.zeros(5, dtype=np.int64)
        fa, fh, fl, fdt, fs = fine
        ga, gh, gl, gdt, gs = coarse
        buf = C.create_string_buffer(512)
        rc = self.f["parareal_run"](n, _p(pos), _p(vel), _p(np.ascontiguousarray(q, dtype=np.float64)),
                                    _p(np.ascontiguousarray(mass, dtype=np.float64)),
                                    _p(np.asarray(box, dtype=np.float64)), fa, fh, fl, fdt, fs, ga, gh,
                                    gl, gdt, gs, kc, conv, window, max_iter, tol, int(short_circuit),
                                    skip_threshold, total_points, threads, _p(tp), _p(tv), _pl(cnt),
                                    buf, 512)
        err = None if rc == 0 else OracleError(rc, buf.value.decode())
        return tp, tv, cnt, err


    # ---------------------------------------------------------- any ForceField
    def field_evaluate(self, spec, pos, q, box, kc=332.0636, conv=4.184e-4):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64)
        n = len(q)
        phi, f, e = np.zeros(n), np.zeros((n, 3)), np.zeros(1)
        self._call(self.f["field_evaluate"], _p(np.ascontiguousarray(spec, dtype=np.float64)), n, _p(pos), _p(q),
                   _p(np.asarray(box, dtype=np.float64)), kc, conv, _p(phi), _p(f), _p(e))
        return dict(phi=phi, force=f, energy=float(e[0]))

    def field_propagate(self, spec, pos, vel, q, mass, box, dt, steps, kc=332.0636, conv=4.184e-4):
        """Returns (pos, vel, steps_done, error-or-None)."""
        pos = np.array(pos, dtype=np.float64, copy=True).reshape(-1, 3)
        vel = np.array(vel, dtype=np.float64, copy=True).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64)
        mass = np.ascontiguousarray(mass, dtype=np.float64)
        done = C.c_int(0)
        buf = C.create_string_buffer(512)
        fn = self.lib.ref_field_propagate_trace if self.kind == "ref" else self.lib.orc_field_propagate
        rc = fn(_p(np.ascontiguousarray(spec, dtype=np.float64)), len(q), _p(pos), _p(vel), _p(q), _p(mass),
                _p(np.asarray(box, dtype=np.float64)), kc, conv, dt, steps, C.byref(done), buf, 512)
        err = None if rc == 0 else OracleError(rc, buf.value.decode())
        return pos, vel, done.value, err

    def field_parareal_window(self, pos, vel, q, mass, box, fine_spec, fdt, fsteps, coarse_spec, gdt, gsteps,
                              t_points, k_iters, kc=332.0636, conv=4.184e-4):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        vel = np.ascontiguousarray(vel, dtype=np.float64).reshape(-1, 3)
        n = len(pos)
        rp = np.zeros((t_points + 1, n, 3))
        rv = np.zeros((t_points + 1, n, 3))
        dr = np.zeros(t_points + 1)
        cnt = np.zeros(3, dtype=np.int64)
        self._call(self.f["field_parareal_window"], n, _p(pos), _p(vel), _p(np.ascontiguousarray(q, dtype=np.float64)),
                   _p(np.ascontiguousarray(mass, dtype=np.float64)), _p(np.asarray(box, dtype=np.float64)),
                   _p(np.ascontiguousarray(fine_spec, dtype=np.float64)), fdt, fsteps,
                   _p(np.ascontiguousarray(coarse_spec, dtype=np.float64)), gdt, gsteps, kc, conv, t_points,
                   k_iters, _p(rp), _p(rv), _p(dr), _pl(cnt))
        return rp, rv, dr, cnt


_cache: dict[str, Checker] = {}


def checker(kind: str) -> Checker:
    if kind not in _cache:
        _cache[kind] = Checker(kind)
    return _cache[kind]


def have(kind: str) -> bool:
    return (REF_SO if kind == "ref" else PORT_SO).exists()
