"""ctypes binding of lib/libmsmb.so (the C ABI declared in include/msmb.h).

Loading fails loudly when the library is missing; there is no Python or CPU
fallback for any compute entry point.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# MSMB_LIB overrides the library path (used only by tools/ to compare kernel variants)
LIB_PATH = Path(os.environ.get("MSMB_LIB", Path(__file__).resolve().parent / "lib" / "libmsmb.so"))

_D = C.POINTER(C.c_double)
_L = C.POINTER(C.c_int64)
_I = C.POINTER(C.c_int32)
_VP = C.c_void_p


class MsmConfigC(C.Structure):
    _fields_ = [("cutoff_a", C.c_double), ("spacing_h", C.c_double), ("levels_l", C.c_int),
                ("interp_order_p", C.c_int), ("smoothing_m", C.c_int)]


class UnitsC(C.Structure):
    _fields_ = [("coulomb_constant", C.c_double), ("energy_to_native", C.c_double)]


class CutoffParamsC(C.Structure):
    _fields_ = [("cutoff", C.c_double), ("has_wolf_alpha", C.c_int), ("wolf_alpha", C.c_double),
                ("flops_per_particle", C.c_double)]


class PropagatorC(C.Structure):
    _fields_ = [("field", _VP), ("dt", C.c_double), ("steps_per_slice", C.c_int)]


class PararealC(C.Structure):
    _fields_ = [("window_points", C.c_int), ("max_iter", C.c_int), ("tol", C.c_double),
                ("fine", PropagatorC), ("coarse", PropagatorC), ("units", UnitsC),
                ("has_skip_threshold", C.c_int), ("skip_threshold", C.c_double),
                ("short_circuit", C.c_int)]


# name -> (restype, argtypes); mirrors include/msmb.h one to one
SIGNATURES = {
    "msmb_abi_version": (C.c_int, []),
    "msmb_device_count": (C.c_int, []),
    "msmb_create": (C.c_int, [C.POINTER(MsmConfigC), C.POINTER(UnitsC), C.c_int, C.POINTER(_VP)]),
    "msmb_destroy": (None, [_VP]),
    "msmb_create_cutoff": (C.c_int, [C.c_int, C.POINTER(CutoffParamsC), C.POINTER(UnitsC), C.c_int,
                                     C.POINTER(_VP)]),
    "msmb_field_kind": (C.c_int, [_VP]),
    "msmb_create_direct": (C.c_int, [C.POINTER(UnitsC), C.c_int, C.POINTER(_VP)]),
    "msmb_create_overlay": (C.c_int, [_VP, C.c_double, C.c_double, C.POINTER(_VP)]),
    "msmb_evaluate": (C.c_int, [_VP, C.c_int64, _D, _D, _D, _D, _D, _D, _D, _D]),
    "msmb_propagate": (C.c_int, [_VP, C.c_int64, _D, _D, _D, _D, _D, C.c_double, C.c_int]),
    "msmb_propagate_ex": (C.c_int, [_VP, C.c_int64, _D, _D, _D, _D, _D, C.c_double, C.c_int,
                                    C.POINTER(UnitsC)]),
    "msmb_energy_report": (C.c_int, [_VP, C.c_int64, _D, _D, _D, _D, _D, C.POINTER(UnitsC), _D]),
    "msmb_host_alloc": (_VP, [C.c_int64]),
    "msmb_host_free": (None, [_VP]),
    "msmb_cost_flops_per_step": (C.c_double, [_VP, C.c_int64]),
    "msmb_last_error": (C.c_int, [_VP, C.POINTER(C.c_int), _L, _L, C.POINTER(C.c_int), C.c_char_p, C.c_int]),
    "msmb_system_create": (C.c_int, [_VP, C.c_int64, _D, _D, _D, _D, _D, C.POINTER(_VP)]),
    "msmb_system_destroy": (None, [_VP]),
    "msmb_system_upload": (C.c_int, [_VP, _D, _D]),
    "msmb_system_download": (C.c_int, [_VP, _D, _D]),
    "msmb_system_copy": (C.c_int, [_VP, _VP]),
    "msmb_system_propagate_ex": (C.c_int, [_VP, _VP, C.c_double, C.c_int, C.POINTER(UnitsC)]),
    "msmb_set_lattice_method": (C.c_int, [_VP, C.c_int]),
    "msmb_set_pair_skin": (C.c_int, [_VP, C.c_double]),
    "msmb_set_list_reuse": (C.c_int, [_VP, C.c_int]),
    "msmb_dd_plan": (C.c_int, [C.POINTER(MsmConfigC), C.POINTER(UnitsC), _D, C.c_int64, C.c_int, C.c_int, _I,
                              C.c_int]),
    "msmb_nccl_unique_id": (C.c_int, [_VP]),
    "msmb_slab_create": (C.c_int, [C.POINTER(_VP), C.c_int, C.c_int, C.c_int, _VP, _VP, C.POINTER(_VP)]),
    "msmb_slab_destroy": (None, [_VP]),
    "msmb_slab_propagate": (C.c_int, [_VP, C.c_int64, _D, _D, _D, _D, _D, C.c_double, C.c_int, C.POINTER(UnitsC),
                                      _D, _D]),
    "msmb_slab_stats": (C.c_int, [_VP, _L, C.c_int]),
    "msmb_slab_last_error": (C.c_int, [_VP, C.POINTER(C.c_int), _L, _L, C.POINTER(C.c_int), C.c_char_p, C.c_int]),
    "msmb_state_sub_device": (C.c_int, [_VP, C.c_int64, _VP, _VP, _VP, _D]),
    "msmb_state_add_device": (C.c_int, [_VP, C.c_int64, _VP, _VP, _VP]),
    "msmb_state_rms_change_device": (C.c_int, [_VP, C.c_int64, _VP, _VP, _D]),
    "msmb_system_set_state_device": (C.c_int, [_VP, _VP]),
    "msmb_system_get_state_device": (C.c_int, [_VP, _VP]),
    "msmb_system_propagate": (C.c_int, [_VP, _VP, C.c_double, C.c_int]),
    "msmb_system_evaluate": (C.c_int, [_VP, _VP, _D, _D, _D, _D, _D]),
    "msmb_parareal_window": (C.c_int, [C.POINTER(PararealC), C.c_int64, _D, _D, _D, _D, _D, C.c_int,
                                       C.c_int, _D, _D, _D, _L]),
    "msmb_parareal_run": (C.c_int, [C.POINTER(PararealC), C.c_int64, _D, _D, _D, _D, _D, C.c_int,
                                    _D, _D, _L]),
    "msmb_parareal_run_ex": (C.c_int, [C.POINTER(PararealC), C.POINTER(_VP), C.c_int, C.c_int64, _D, _D, _D, _D,
                                       _D, C.c_int, _D, _D, _L, _VP, C.c_int64, _L, _I]),
    "msmb_set_stage_timing": (C.c_int, [_VP, C.c_int]),
    "msmb_stage_times": (C.c_int, [_VP, _D, _L, C.POINTER(C.c_char_p), C.c_int]),
    "msmb_reset_stage_times": (None, [_VP]),
    "msmb_work_counters": (C.c_int, [_VP, _L, C.c_int]),
    "msmb_kernel_launches": (C.c_int64, [_VP]),
    "msmb_bench_propagate": (C.c_int, [_VP, _VP, C.c_double, C.c_int, C.c_int, _D, _D,
                                       C.POINTER(C.c_char_p), _L]),
    "msmb_measure_fp64_peak": (C.c_int, [C.c_int, C.c_double, _D]),
    "msmb_grid_geometry": (C.c_int, [C.POINTER(MsmConfigC), _D, _I, _D, _D]),
    "msmb_debug_levels": (C.c_int, [_VP, _D, _D]),
    "msmb_debug_cells": (C.c_int, [_VP, C.c_int64, _D, _D, _I, _I]),
    "msmb_debug_stage": (C.c_int, [_VP, C.c_int, C.c_int, _D, _D, _D, C.c_int64, _D]),
    "msmb_debug_bin_keys": (C.c_int, [_VP, C.c_int64, _D, _D, _I, _I]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(SIGNATURES)
