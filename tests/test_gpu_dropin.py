"""Drop-in at the reference's own plugin boundary: the unmodified reference
library (oracle/_ref, compiled from /root/reference/proj/src) drives
paramd::GpuMsmField (include/paramd_b200/gpu_msm_field.hpp) through
paramd::ForceField -- its propagate() and parareal_run() run unchanged with
the B200 field plugged in (oracle/dropin_driver.cpp)."""
import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
DRIVER = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "dropin_driver"


def test_reference_drives_gpu_field():
    if not DRIVER.exists():
        pytest.skip("oracle/_ref/dropin_driver not built (needs /root/reference at build time)")
    out = subprocess.run([str(DRIVER)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["de"] <= 1e-10 and r["df"] <= 1e-8
    assert r["dx_plugin_propagate"] <= 1e-8 and r["dx_device_propagate"] <= 1e-8
    assert r["parareal_ok"] == 1
    assert r["dx_parareal_plugin"] <= 1e-8 and r["dx_parareal_device"] <= 1e-8
    c = r["counts"]
    assert c[0] == c[2] == c[4] and c[1] == c[3] == c[5]
    assert r["coincident_ref"] and r["coincident_ref"] == r["coincident_gpu"]
    assert r["coverage_ref"] and r["coverage_ref"] == r["coverage_gpu"]
    assert r["name"] == "msm" and r["cost"] == r["cost_ref"]
    # pair-only fields through the same plugin boundary
    assert r["pf_de"] <= 1e-10 and r["pf_df"] <= 1e-8
    assert r["pf_dx_plugin_propagate"] <= 1e-8 and r["pf_dx_device_propagate"] <= 1e-8
    assert 0 <= r["pf_dx_parareal_device"] <= 1e-8
    # all-pairs fields (F3 direct Coulomb, F2 repulsion overlay)
    assert r["ap_de"] <= 1e-10 and r["ap_df"] <= 1e-8
    # paramd_b200::GpuExecutor (fine replicas) == one fine field, bit for bit, with the
    # reference's ConvergenceReport rows / point_iterations; a host field on the device
    # path raises ConfigError instead of running on the CPU
    assert r["dx_executor"] == 0.0 and r["rows_ok"] == 1 and r["fallback_rejected"] == 1
