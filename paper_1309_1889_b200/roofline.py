"""Per-stage roofline model of one MSM force + Verlet step.

Compute stages are counted in FP64 issue slots (one DFMA/DMUL/DADD/DSETP = 1
slot); the slot rate is the FP64 FMA rate = P64/2 (P64 in flop/s, FMA = 2).
Memory stages are counted in algorithmic HBM bytes.  T_roof(step) =
sum_s max(B_s / BW, W_s / (P64/2)); a stage's fraction = roof_s / measured_s.

Stage -> engine stages:
  S1 bin/sort   (B = 72 N)                 -> bin + sort
  S2 pairs      (W = 30 P_u)               -> clusters + pairs (search overhead included)
  S3 anterp     (W = 144 N, B = 32N + 8M0) -> anterp
  S4 restrict   (B = sum 8 (M_k + M_k+1))  -> restrict
  S5 lattice    (W = clipped nonzero taps) -> lattice
  S6 top        (W = M_top^2)              -> top
  S7 prolong    (B = sum 8 (M_k+1 + 2 M_k))-> prolong
  S8 interp     (W = 330 N, B = 64 N)      -> interp + finalize
  S10 verlet    (B = 128 N)                -> verlet (kick/drift kernels)
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
PAIR_SLOTS = 30            # FP64 issue slots per unordered in-cutoff pair (Newton-3 accounting)
PAIR_FLOPS = 40            # algorithmic flops per unordered pair (FMA = 2, rsqrt = 1)


def hbm_peak_gbs():
    """(GB/s, source) -- MEASURED_PEAKS.json when present, else the profiling guide's fallback."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (of measured)"
        except Exception:
            pass
    return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s (of fallback)"


def stage_model(n, level_sizes, pairs_u, lattice_taps, top_taps):
    """Algorithmic work per stage for one evaluation: dict stage -> (slots, bytes)."""
    M = [int(m) for m in level_sizes]
    l = len(M)
    restrict_b = sum(8 * (M[k] + M[k + 1]) for k in range(l - 1))
    prolong_b = sum(8 * (M[k + 1] + 2 * M[k]) for k in range(l - 1))
    return {
        "S1_bin": (0.0, 72.0 * n),
        "S2_pairs": (PAIR_SLOTS * float(pairs_u), 0.0),
        "S3_anterp": (144.0 * n, 32.0 * n + 8.0 * M[0]),
        "S4_restrict": (0.0, float(restrict_b)),
        "S5_lattice": (float(lattice_taps), 0.0),
        "S6_top": (float(top_taps), 0.0),
        "S7_prolong": (0.0, float(prolong_b)),
        "S8_interp": (330.0 * n, 64.0 * n),
        "S10_verlet": (0.0, 128.0 * n),
    }


ENGINE_STAGES = {
    "S1_bin": ["bin", "sort"],
    "S2_pairs": ["clusters", "pairs"],
    "S3_anterp": ["anterp"],
    "S4_restrict": ["restrict"],
    "S5_lattice": ["lattice"],
    "S6_top": ["top"],
    "S7_prolong": ["prolong"],
    "S8_interp": ["interp", "finalize"],
    "S10_verlet": ["verlet"],
}


def evaluate(n, level_sizes, pairs_u, lattice_taps, top_taps, stage_ms_per_step, fp64_tflops, hbm_gbs):
    """Returns (per-stage dict, T_roof ms, T_measured ms)."""
    model = stage_model(n, level_sizes, pairs_u, lattice_taps, top_taps)
    slot_rate = fp64_tflops * 1e12 / 2.0
    bw = hbm_gbs * 1e9
    out = {}
    t_roof = t_meas = 0.0
    for s, (slots, byts) in model.items():
        roof = max(slots / slot_rate, byts / bw) * 1e3
        meas = sum(stage_ms_per_step.get(e, 0.0) for e in ENGINE_STAGES[s])
        out[s] = {"ms": round(meas, 5), "roof_ms": round(roof, 5),
                  "frac": round(roof / meas, 4) if meas > 0 else None,
                  "bound": "fp64" if slots / slot_rate >= byts / bw else "hbm"}
        t_roof += roof
        t_meas += meas
    return out, t_roof, t_meas
