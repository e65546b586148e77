"""B200-native MSM force / velocity-Verlet / parareal path of arXiv 1309.1889.

A Python mirror of the reference library's (`paramd`, /root/reference/proj)
interface for this path -- same names, argument meaning and error behaviour --
over the C ABI in include/msmb.h (lib/libmsmb.so: hand-written sm_100a
kernels).  Every compute call runs on the GPU; without a usable B200 the
constructors raise :class:`CudaUnavailableError` (no CPU fallback).

Reference interface -> here:
  paramd::MsmConfig            include/paramd/msm_grid.hpp:10-18  -> MsmConfig
  paramd::UnitsConfig          include/paramd/units.hpp:16-27     -> UnitsConfig
  paramd::ParticleSystem       include/paramd/system.hpp:10-18    -> ParticleSystem
  paramd::PotentialResult      include/paramd/potential.hpp:18-24 -> PotentialResult
  paramd::ForceField/MsmField  include/paramd/force_field.hpp:14-73 -> ForceField/MsmField
  paramd::CutoffParams         include/paramd/potential.hpp:26-31 -> CutoffParams
  paramd::SimpleCutoffField/WolfField
                               include/paramd/force_field.hpp:34-60 -> SimpleCutoffField/WolfField
  paramd::simple_cutoff/wolf_summation/direct_coulomb
                               include/paramd/electrostatics.hpp:9-22 -> same names
  paramd::DirectCoulombField/PairRepulsionOverlay
                               include/paramd/force_field.hpp:23-32,75-97 -> same names
  paramd::msm_potential        include/paramd/msm.hpp:24-25       -> msm_potential
  paramd::PropagatorSpec/propagate/verlet_step/energy_report
                               include/paramd/integrate.hpp:13-38 -> same names
  paramd::PararealConfig/parareal_init+iterate/parareal_run
                               include/paramd/parareal.hpp:40-144 -> parareal_window/parareal_run
  exceptions                   include/paramd/errors.hpp:7-49     -> same names
"""
from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native

__all__ = [
    "MsmConfig", "UnitsConfig", "ParticleSystem", "PotentialResult", "ForceField", "MsmField",
    "GpuField", "CutoffParams", "SimpleCutoffField", "WolfField", "simple_cutoff", "wolf_summation",
    "DirectCoulombField", "PairRepulsionOverlay", "direct_coulomb",
    "msm_potential", "PropagatorSpec", "propagate", "verlet_step", "energy_report", "EnergyReport",
    "PararealConfig", "PararealResult", "parareal_window", "parareal_run", "SequentialExecutor", "GpuExecutor",
    "AsyncExecutor", "DeviceSystem", "Error", "ConfigError", "DomainError", "CoverageError",
    "CoincidentParticlesError", "HierarchyError", "RuntimeFault", "NonConvergenceError",
    "CudaUnavailableError", "device_count", "grid_geometry",
]


# ---------------------------------------------------------------- exceptions
class Error(RuntimeError):
    """paramd::Error (errors.hpp:7-9)."""

    def __init__(self, msg: str = "", i: int = -1, j: int = -1, step: int = -1):
        super().__init__(msg)
        self.i, self.j, self.step = i, j, step


class ConfigError(Error): pass            # errors.hpp:12-14
class DomainError(Error): pass            # errors.hpp:17-19
class CoverageError(Error): pass          # errors.hpp:37-39
class CoincidentParticlesError(Error): pass  # errors.hpp:32-34
class HierarchyError(Error): pass         # errors.hpp:42-44
class RuntimeFault(Error): pass           # errors.hpp:47-49
class NonConvergenceError(Error): pass    # parareal.hpp:124-128
class CudaUnavailableError(Error): pass   # no reference equivalent: no usable B200
class InternalError(Error): pass


_ERR = {1: ConfigError, 2: DomainError, 3: CoverageError, 4: CoincidentParticlesError,
        5: HierarchyError, 6: RuntimeFault, 7: NonConvergenceError, 8: CudaUnavailableError,
        9: InternalError}


def _raise(handle, rc: int):
    kind = C.c_int()
    i, j = C.c_int64(), C.c_int64()
    step = C.c_int()
    buf = C.create_string_buffer(1024)
    _native.lib().msmb_last_error(handle, C.byref(kind), C.byref(i), C.byref(j), C.byref(step), buf, 1024)
    msg = buf.value.decode()
    raise _ERR.get(rc, Error)(msg, i.value, j.value, step.value)


def _check(handle, rc: int):
    if rc != 0:
        _raise(handle, rc)


_D = C.POINTER(C.c_double)


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


# ---------------------------------------------------------------- data types
@dataclass
class MsmConfig:
    """paramd::MsmConfig (msm_grid.hpp:10-18), same defaults."""
    cutoff_a: float = 8.0
    spacing_h: float = 2.0
    levels_l: int = 2
    interp_order_p: int = 3
    smoothing_m: int = 2

    def _c(self):
        return _native.MsmConfigC(self.cutoff_a, self.spacing_h, self.levels_l, self.interp_order_p,
                                  self.smoothing_m)


@dataclass
class UnitsConfig:
    """paramd::UnitsConfig (units.hpp:16-27)."""
    coulomb_constant: float = 332.0636
    energy_to_native: float = 4.184e-4

    @staticmethod
    def physical():
        return UnitsConfig(332.0636, 4.184e-4)

    @staticmethod
    def reduced():
        return UnitsConfig(1.0, 1.0)

    def validate(self):
        if not (self.coulomb_constant > 0.0):
            raise ConfigError("coulomb_constant must be > 0")
        if not (self.energy_to_native > 0.0):
            raise ConfigError("energy_to_native must be > 0")

    def _c(self):
        return _native.UnitsC(self.coulomb_constant, self.energy_to_native)


@dataclass
class ParticleSystem:
    """paramd::ParticleSystem (system.hpp:10-18): positions/velocities (n,3), charges, masses, box."""
    positions: np.ndarray
    velocities: np.ndarray
    charges: np.ndarray
    masses: np.ndarray
    box: np.ndarray

    def __post_init__(self):
        self.positions = _f64(self.positions, (-1, 3))
        n = len(self.positions)
        self.velocities = _f64(self.velocities if self.velocities is not None else np.zeros((n, 3)), (-1, 3))
        self.charges = _f64(self.charges)
        self.masses = _f64(self.masses if self.masses is not None else np.ones(n))
        self.box = _f64(self.box)

    def size(self):
        return len(self.positions)

    def copy(self):
        return ParticleSystem(self.positions.copy(), self.velocities.copy(), self.charges.copy(),
                              self.masses.copy(), self.box.copy())


@dataclass
class PotentialResult:
    """paramd::PotentialResult (potential.hpp:18-24)."""
    per_particle_potential: np.ndarray
    per_particle_force: np.ndarray
    total_energy: float
    short_part: Optional[np.ndarray] = None
    long_part: Optional[np.ndarray] = None


def device_count() -> int:
    return _native.lib().msmb_device_count()


def grid_geometry(config: MsmConfig, box):
    """build_grid_hierarchy geometry (src/msm_grid.cpp:24-54): dims (l,3), spacing (l,), origin (l,3)."""
    L = _native.lib()
    l = config.levels_l
    dims = (C.c_int32 * (3 * max(l, 1)))()
    sp = np.zeros(max(l, 1))
    org = np.zeros(3 * max(l, 1))
    cfg = config._c()
    rc = L.msmb_grid_geometry(C.byref(cfg), _p(_f64(box)), dims, _p(sp), _p(org))
    _check(None, rc)
    return np.array(list(dims)).reshape(-1, 3)[:l], sp[:l], org.reshape(-1, 3)[:l]


# ---------------------------------------------------------------- force fields
class ForceField:
    """paramd::ForceField plugin interface (force_field.hpp:14-21)."""

    def evaluate(self, s: ParticleSystem) -> PotentialResult:  # pragma: no cover - abstract
        raise NotImplementedError

    def cost_flops_per_step(self, n: int) -> float:  # pragma: no cover - abstract
        raise NotImplementedError

    def name(self) -> str:  # pragma: no cover - abstract
        raise NotImplementedError


class GpuField(ForceField):
    """A force field bound to one B200 (a msmb_field handle): the common part of
    MsmField, SimpleCutoffField, WolfField, DirectCoulombField and PairRepulsionOverlay.  ``evaluate`` is const and safe to
    call from several threads (calls on one field are serialised on its GPU stream)."""

    _h = None

    @property
    def handle(self):
        return self._h

    def units(self) -> UnitsConfig:
        return self._units

    def cost_flops_per_step(self, n: int) -> float:
        return _native.lib().msmb_cost_flops_per_step(self._h, n)

    def evaluate(self, s: ParticleSystem) -> PotentialResult:
        self._last_box = s.box
        n = s.size()
        phi, ps, pl = np.zeros(n), np.zeros(n), np.zeros(n)
        f = np.zeros((n, 3))
        e = np.zeros(1)
        rc = _native.lib().msmb_evaluate(self._h, n, _p(s.positions), _p(s.charges), _p(s.box), _p(phi),
                                         _p(ps), _p(pl), _p(f), _p(e))
        _check(self._h, rc)
        if _native.lib().msmb_field_kind(self._h) != 0:  # only MSM fills short_part/long_part
            ps = pl = None
        return PotentialResult(phi, f, float(e[0]), ps, pl)

    # -- measurement / diagnostics
    def set_pair_skin(self, skin: float):
        """Pair-list skin in A (default 0.2; 0 = rebuild the list at every evaluation,
        making forces a pure function of the positions).  See msmb_set_pair_skin."""
        _check(self._h, _native.lib().msmb_set_pair_skin(self._h, float(skin)))

    def set_list_reuse(self, reuse: bool):
        """Keep a still-valid pair list across evaluate / propagate calls (default off:
        every call starts from a fresh list and is a pure function of its input)."""
        _check(self._h, _native.lib().msmb_set_list_reuse(self._h, int(bool(reuse))))

    def set_stage_timing(self, on: bool):
        _native.lib().msmb_set_stage_timing(self._h, int(on))

    def stage_times(self):
        cap = 32
        ms = np.zeros(cap)
        nl = np.zeros(cap, dtype=np.int64)
        names = (C.c_char_p * cap)()
        n = _native.lib().msmb_stage_times(self._h, _p(ms), nl.ctypes.data_as(C.POINTER(C.c_int64)), names, cap)
        return {names[i].decode(): (float(ms[i]), int(nl[i])) for i in range(n)}

    def reset_stage_times(self):
        _native.lib().msmb_reset_stage_times(self._h)

    def work_counters(self):
        out = np.zeros(8, dtype=np.int64)
        _native.lib().msmb_work_counters(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)), 8)
        keys = ["pairs", "candidates", "clusters", "lattice_taps", "top_taps", "launches_per_eval",
                "list_rebuilds", "pair_split"]
        return dict(zip(keys, map(int, out)))

    def kernel_launches(self) -> int:
        return int(_native.lib().msmb_kernel_launches(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if sys is None or sys.is_finalizing():  # process teardown releases the device anyway
            return
        if h is not None and h.value:
            try:
                _native.lib().msmb_destroy(h)
            except Exception:
                pass
            self._h = C.c_void_p()


class MsmField(GpuField):
    """paramd::MsmField (force_field.hpp:62-73) evaluated on a B200."""

    def __init__(self, config: MsmConfig, units: UnitsConfig = None, device: int = 0):
        units = units or UnitsConfig.physical()
        self._config, self._units = config, units
        self._device = device
        self._h = C.c_void_p()
        cfg, u = config._c(), units._c()
        rc = _native.lib().msmb_create(C.byref(cfg), C.byref(u), device, C.byref(self._h))
        if rc:
            _raise(None, rc)

    def config(self) -> MsmConfig:
        return self._config

    def name(self) -> str:
        return "msm"

    def set_lattice_method(self, direct: bool):
        """Lattice cutoff by zero-padded FFT convolution (default) or by the direct
        stencil sum of the reference (src/msm_phases.cpp:93-134)."""
        _check(self._h, _native.lib().msmb_set_lattice_method(self._h, int(bool(direct))))

    def debug_levels(self):
        dims, _, _ = grid_geometry(self._config, self._last_box)
        tot = int(sum(int(np.prod(d)) for d in dims))
        qc, qp = np.zeros(tot), np.zeros(tot)
        _check(self._h, _native.lib().msmb_debug_levels(self._h, _p(qc), _p(qp)))
        return qc, qp

    def debug_cells(self, positions, box):
        pos = _f64(positions, (-1, 3))
        n = len(pos)
        cells = np.zeros((n, 3), dtype=np.int32)
        cov = np.zeros(n, dtype=np.int32)
        rc = _native.lib().msmb_debug_cells(self._h, n, _p(pos), _p(_f64(box)),
                                            cells.ctypes.data_as(C.POINTER(C.c_int32)),
                                            cov.ctypes.data_as(C.POINTER(C.c_int32)))
        _check(self._h, rc)
        return cells, cov.astype(bool)

    def debug_bin_keys(self, positions, box):
        """Level-0 cell triples from the production binning kernel's sort keys."""
        pos = _f64(positions, (-1, 3))
        n = len(pos)
        cells = np.zeros((n, 3), dtype=np.int32)
        cov = np.zeros(n, dtype=np.int32)
        rc = _native.lib().msmb_debug_bin_keys(self._h, n, _p(pos), _p(_f64(box)),
                                               cells.ctypes.data_as(C.POINTER(C.c_int32)),
                                               cov.ctypes.data_as(C.POINTER(C.c_int32)))
        _check(self._h, rc)
        return cells, cov.astype(bool)

    def debug_stage(self, stage: int, k: int, box, inp, out=None, positions=None):
        """Single stage on caller lattices: bit-exact variants 0 restrict, 1 lattice cutoff,
        2 top, 3 prolong, 4 interp; production kernels 5 restriction chain (level-0 charges
        -> all levels), 6 top, 7 prolongation chain (all levels' potentials in / out)."""
        dims, _, _ = grid_geometry(self._config, box)
        total = int(sum(int(np.prod(d)) for d in dims))
        if stage == 0:
            out = np.zeros(int(np.prod(dims[k + 1])))
        elif stage in (5, 7):
            out = np.zeros(total)
        elif stage in (1, 2, 6):
            out = np.zeros(len(inp))
        elif stage == 3:
            out = np.array(out, dtype=np.float64, copy=True)
        pos = None
        n = 0
        if stage == 4:
            pos = _f64(positions, (-1, 3))
            n = len(pos)
            out = np.zeros(n)
        rc = _native.lib().msmb_debug_stage(self._h, stage, k, _p(_f64(box)), _p(_f64(inp)), _p(out), n, _p(pos))
        _check(self._h, rc)
        return out


@dataclass
class CutoffParams:
    """paramd::CutoffParams (potential.hpp:26-31)."""
    cutoff: float = 12.0
    wolf_alpha: Optional[float] = None

    def validate(self, need_alpha: bool):  # src/electrostatics.cpp:38-42
        if not (self.cutoff > 0.0):
            raise ConfigError("cutoff must be > 0")
        if need_alpha and self.wolf_alpha is None:
            raise ConfigError("wolf_alpha is required")
        if self.wolf_alpha is not None and not (self.wolf_alpha >= 0.0):
            raise ConfigError("wolf_alpha must be >= 0")


class _PairField(GpuField):
    """Pair-only GPU fields (msmb_create_cutoff): the MSM engine's binning, cluster
    pair list and pair kernel with the field's pair function and no grid.  The box
    of an evaluated system only sets the binning extent (atoms outside it are
    still handled); ``short_part`` is the potential and ``long_part`` zeros."""
    _kind = 0
    _default_fpp = 0.0

    def __init__(self, params: CutoffParams = None, units: UnitsConfig = None,
                 flops_per_particle: float = None, device: int = 0):
        self._params = params or CutoffParams()
        self._units = units or UnitsConfig.physical()
        self._fpp = self._default_fpp if flops_per_particle is None else float(flops_per_particle)
        self._device = device
        self._h = C.c_void_p()
        p = self._params
        pc = _native.CutoffParamsC(p.cutoff, int(p.wolf_alpha is not None), float(p.wolf_alpha or 0.0), self._fpp)
        u = self._units._c()
        rc = _native.lib().msmb_create_cutoff(self._kind, C.byref(pc), C.byref(u), device, C.byref(self._h))
        if rc:
            _raise(None, rc)

    def params(self) -> CutoffParams:
        return self._params


class SimpleCutoffField(_PairField):
    """paramd::SimpleCutoffField (force_field.hpp:34-46): Coulomb truncated at r >= cutoff
    (simple_cutoff, src/electrostatics.cpp:66-89), on a B200."""
    _kind = 1
    _default_fpp = 301.0

    def name(self) -> str:
        return "cutoff"


class WolfField(_PairField):
    """paramd::WolfField (force_field.hpp:48-60): damped-shifted-force electrostatics
    (wolf_summation, src/electrostatics.cpp:91-129), on a B200."""
    _kind = 2
    _default_fpp = 350.0

    def name(self) -> str:
        return "wolf"


class DirectCoulombField(GpuField):
    """paramd::DirectCoulombField (force_field.hpp:23-32): the exact O(N^2) Coulomb sum
    (direct_coulomb, src/electrostatics.cpp:43-64), all pairs on a B200.  No box needed."""

    def __init__(self, units: UnitsConfig = None, device: int = 0):
        self._units = units or UnitsConfig.physical()
        self._device = device
        self._h = C.c_void_p()
        u = self._units._c()
        rc = _native.lib().msmb_create_direct(C.byref(u), device, C.byref(self._h))
        if rc:
            _raise(None, rc)

    def name(self) -> str:
        return "direct"


class PairRepulsionOverlay(GpuField):
    """paramd::PairRepulsionOverlay (force_field.hpp:75-97; force_field.cpp:45-68):
    the base GPU field plus U = sum_{i<j} eps (sigma/r)^12 over all pairs (forces and
    total energy include it; the per-particle potential stays electrostatic).  The
    overlay is its own GPU handle (msmb_create_overlay); ``base`` is unchanged."""

    def __init__(self, base: GpuField, epsilon: float = 0.1, sigma: float = 1.0):
        if not isinstance(base, GpuField):
            raise ConfigError("PairRepulsionOverlay needs a GPU base field")
        self._base = base
        self._units = base.units()
        self._device = base._device
        self._eps, self._sigma = float(epsilon), float(sigma)
        self._h = C.c_void_p()
        rc = _native.lib().msmb_create_overlay(base.handle, self._eps, self._sigma, C.byref(self._h))
        if rc:
            _raise(None, rc)

    def name(self) -> str:
        return self._base.name() + "+rep"



def direct_coulomb(s: ParticleSystem, units: UnitsConfig = None) -> PotentialResult:
    """paramd::direct_coulomb (electrostatics.hpp:9) on the GPU."""
    return DirectCoulombField(units or UnitsConfig.physical()).evaluate(s)


def simple_cutoff(s: ParticleSystem, params: CutoffParams, units: UnitsConfig = None) -> PotentialResult:
    """paramd::simple_cutoff (electrostatics.hpp:12-13) on the GPU."""
    return SimpleCutoffField(params, units or UnitsConfig.physical()).evaluate(s)


def wolf_summation(s: ParticleSystem, params: CutoffParams, units: UnitsConfig = None) -> PotentialResult:
    """paramd::wolf_summation (electrostatics.hpp:21-22) on the GPU."""
    return WolfField(params, units or UnitsConfig.physical()).evaluate(s)


def msm_potential(s: ParticleSystem, config: MsmConfig, units: UnitsConfig = None) -> PotentialResult:
    """paramd::msm_potential (msm.hpp:24-25; src/msm.cpp:52-90) on the GPU."""
    f = MsmField(config, units or UnitsConfig.physical())
    f._last_box = s.box
    return f.evaluate(s)


class DeviceSystem:
    """A ParticleSystem resident in HBM (msmb_system), for device-resident propagation."""

    def __init__(self, field: GpuField, s: ParticleSystem):
        self.field = field
        self.n = s.size()
        self.box = s.box.copy()
        field._last_box = self.box  # debug_levels reads the lattices of this box
        self._h = C.c_void_p()
        rc = _native.lib().msmb_system_create(field.handle, self.n, _p(s.positions), _p(s.velocities),
                                              _p(s.charges), _p(s.masses), _p(s.box), C.byref(self._h))
        _check(field.handle, rc)

    def propagate(self, dt: float, steps: int):
        _check(self.field.handle, _native.lib().msmb_system_propagate(self.field.handle, self._h, dt, steps))

    def upload(self, positions=None, velocities=None):
        rc = _native.lib().msmb_system_upload(self._h, _p(None if positions is None else _f64(positions, (-1, 3))),
                                              _p(None if velocities is None else _f64(velocities, (-1, 3))))
        _check(self.field.handle, rc)

    def download(self):
        pos, vel = np.zeros((self.n, 3)), np.zeros((self.n, 3))
        _check(self.field.handle, _native.lib().msmb_system_download(self._h, _p(pos), _p(vel)))
        return pos, vel

    def evaluate(self, outputs=True):
        n = self.n
        phi, ps, pl, f, e = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros((n, 3)), np.zeros(1)
        rc = _native.lib().msmb_system_evaluate(self.field.handle, self._h, _p(phi), _p(ps), _p(pl), _p(f), _p(e))
        _check(self.field.handle, rc)
        return PotentialResult(phi, f, float(e[0]), ps, pl)

    def __del__(self):
        h = getattr(self, "_h", None)
        if sys is None or sys.is_finalizing():
            return
        if h is not None and h.value:
            try:
                _native.lib().msmb_system_destroy(h)
            except Exception:
                pass
            self._h = C.c_void_p()


# ---------------------------------------------------------------- integrator
@dataclass
class PropagatorSpec:
    """paramd::PropagatorSpec (integrate.hpp:13-20)."""
    force_field: Optional[ForceField] = None
    dt: float = 1.0
    steps_per_slice: int = 1

    def slice_span(self) -> float:
        return self.dt * self.steps_per_slice

    def validate(self):  # src/integrate.cpp:7-11
        if self.force_field is None:
            raise ConfigError("propagator has no force field")
        if not (self.dt > 0.0):
            raise ConfigError("dt must be > 0")
        if self.steps_per_slice < 1:
            raise ConfigError("steps_per_slice must be >= 1")


def propagate(spec: PropagatorSpec, s: ParticleSystem, units: UnitsConfig = None) -> ParticleSystem:
    """paramd::propagate (src/integrate.cpp:13-36), device-resident on the B200."""
    spec.validate()
    units = units or UnitsConfig.physical()
    if not isinstance(spec.force_field, GpuField):
        raise ConfigError("this build propagates GPU force fields (MsmField, SimpleCutoffField, WolfField) only")
    out = s.copy()
    u = units._c()
    ff = spec.force_field
    rc = _native.lib().msmb_propagate_ex(ff.handle, out.size(), _p(out.positions), _p(out.velocities),
                                         _p(out.charges), _p(out.masses), _p(out.box), spec.dt,
                                         spec.steps_per_slice, C.byref(u))
    _check(ff.handle, rc)
    return out


def verlet_step(s: ParticleSystem, ff: ForceField, dt: float, units: UnitsConfig = None) -> ParticleSystem:
    """paramd::verlet_step (src/integrate.cpp:38-45)."""
    return propagate(PropagatorSpec(ff, dt, 1), s, units)


@dataclass
class EnergyReport:
    kinetic: float = 0.0
    potential: float = 0.0
    total: float = 0.0


def energy_report(s: ParticleSystem, ff: ForceField, units: UnitsConfig = None) -> EnergyReport:
    """paramd::energy_report (src/integrate.cpp:47-55)."""
    units = units or UnitsConfig.physical()
    units.validate()
    if not isinstance(ff, GpuField):
        raise ConfigError("energy_report: force field is not a B200 field")
    out = np.zeros(3)
    u = units._c()
    rc = _native.lib().msmb_energy_report(ff.handle, s.size(), _p(s.positions), _p(s.velocities), _p(s.charges),
                                          _p(s.masses), _p(s.box), C.byref(u), _p(out))
    _check(ff.handle, rc)
    rep = EnergyReport()
    rep.kinetic, rep.potential, rep.total = float(out[0]), float(out[1]), float(out[2])
    return rep


# ---------------------------------------------------------------- parareal
class SequentialExecutor:
    """paramd::SequentialExecutor (parareal.hpp:22-26).  On the GPU the fine
    slices of one iteration run back to back on the fine field's stream; the
    executor choice never changes results (pure propagators)."""


class AsyncExecutor(SequentialExecutor):
    def __init__(self, threads: int = 1):
        self.threads = threads


class GpuExecutor(SequentialExecutor):
    """The Executor plug-in (parareal.hpp:15-31, used at parareal.cpp:151) over GPUs:
    replicas of the fine field, typically one per device.  parareal_run deals the
    fine slices of every iteration to the fine field and the replicas
    (msmb_parareal_run_ex), like AsyncExecutor::parallel_for (parareal.cpp:16-36).
    Results are bitwise those of a single fine field."""

    def __init__(self, fine_replicas):
        self.fine_replicas = list(fine_replicas)


@dataclass
class PararealConfig:
    """paramd::PararealConfig (parareal.hpp:40-51)."""
    window_points: int = 8
    max_iter: int = 5
    tol: float = 1e-6
    fine: PropagatorSpec = field(default_factory=PropagatorSpec)
    coarse: PropagatorSpec = field(default_factory=PropagatorSpec)
    units: UnitsConfig = field(default_factory=UnitsConfig)
    skip_threshold: Optional[float] = None
    short_circuit: bool = True

    def _c(self):
        def prop(sp):
            h = sp.force_field.handle if isinstance(sp.force_field, GpuField) else None
            return _native.PropagatorC(h, sp.dt, sp.steps_per_slice)
        return _native.PararealC(self.window_points, self.max_iter, self.tol, prop(self.fine),
                                 prop(self.coarse), self.units._c(), int(self.skip_threshold is not None),
                                 float(self.skip_threshold or 0.0), int(self.short_circuit))


@dataclass
class PararealResult:
    trajectory: list
    counts: dict
    windows: int
    converged: bool
    # ConvergenceReport::rows (window, point, iteration, delta_rms, converged) and
    # ::point_iterations (parareal.hpp:108-122)
    report_rows: list = field(default_factory=list)
    point_iterations: list = field(default_factory=list)


class _RowC(C.Structure):
    _fields_ = [("window", C.c_int), ("point", C.c_int), ("iteration", C.c_int), ("delta_rms", C.c_double),
                ("converged", C.c_int)]


def _cfg_handle(cfg):
    return cfg.fine.force_field.handle if isinstance(cfg.fine.force_field, GpuField) else None


def parareal_window(v: ParticleSystem, cfg: PararealConfig, t_points: int, k_iters: int,
                    exec=None):
    """parareal_init + k_iters x parareal_iterate (src/parareal.cpp:94-180).
    Returns (final lambda row as a list of ParticleSystems n=0..t, delta_rms, counts)."""
    n = v.size()
    rp = np.zeros((t_points + 1, n, 3))
    rv = np.zeros((t_points + 1, n, 3))
    dr = np.zeros(t_points + 1)
    cnt = np.zeros(3, dtype=np.int64)
    c = cfg._c()
    rc = _native.lib().msmb_parareal_window(C.byref(c), n, _p(v.positions), _p(v.velocities),
                                            _p(v.charges), _p(v.masses), _p(v.box), t_points, k_iters,
                                            _p(rp), _p(rv), _p(dr),
                                            cnt.ctypes.data_as(C.POINTER(C.c_int64)))
    _check(_cfg_handle(cfg), rc)
    row = [ParticleSystem(rp[i], rv[i], v.charges, v.masses, v.box) for i in range(t_points + 1)]
    return row, dr, dict(g_evals=int(cnt[0]), f_evals=int(cnt[1]), f_skipped=int(cnt[2]))


def parareal_run(v: ParticleSystem, total_points: int, cfg: PararealConfig, exec=None) -> PararealResult:
    """paramd::parareal_run (src/parareal.cpp:182-239).  exec = GpuExecutor([...])
    spreads the fine sweep over fine-field replicas (GPUs)."""
    n = v.size()
    tp = np.zeros((max(total_points, 1), n, 3))
    tv = np.zeros((max(total_points, 1), n, 3))
    rep = np.zeros(6, dtype=np.int64)
    c = cfg._c()
    reps = [r.handle for r in getattr(exec, "fine_replicas", [])]
    rarr = (C.c_void_p * max(len(reps), 1))(*reps)
    cap = max(1, cfg.max_iter * cfg.window_points * max(total_points, 1))
    rows = (_RowC * cap)()
    nrows = C.c_int64(0)
    piters = np.zeros(max(total_points, 1), dtype=np.int32)
    rc = _native.lib().msmb_parareal_run_ex(C.byref(c), rarr, len(reps), n, _p(v.positions), _p(v.velocities),
                                            _p(v.charges), _p(v.masses), _p(v.box), total_points, _p(tp), _p(tv),
                                            rep.ctypes.data_as(C.POINTER(C.c_int64)), C.cast(rows, C.c_void_p),
                                            cap, C.byref(nrows), piters.ctypes.data_as(C.POINTER(C.c_int32)))
    report_rows = [(r.window, r.point, r.iteration, r.delta_rms, bool(r.converged))
                   for r in rows[:min(nrows.value, cap)]]
    counts = dict(g_evals=int(rep[0]), f_evals=int(rep[1]), f_skipped=int(rep[2]))
    try:
        _check(_cfg_handle(cfg), rc)
    except NonConvergenceError as e:
        e.report = PararealResult([], counts, int(rep[3]), False, report_rows, [int(x) for x in piters[:rep[5]]])
        raise
    traj = [ParticleSystem(tp[i], tv[i], v.charges, v.masses, v.box) for i in range(total_points)]
    return PararealResult(traj, counts, int(rep[3]), bool(rep[4]), report_rows, [int(x) for x in piters[:rep[5]]])
