"""Summarises Nsight Compute output into the committed profiles/ directory.

    python tools/ncu_summary.py launches <launches.csv> <out.md>
        per-kernel share of one timed step from an `ncu --metrics gpu__time_duration.sum`
        launch list (cold-cache, serialised launches: compare SHARES, not absolutes)
    python tools/ncu_summary.py full <report.ncu-rep> <out.md> [--traffic-key NAME]
        key metrics of one `ncu --set full` capture; with --traffic-key, also records
        dram read+write bytes per launch in profiles/ncu_traffic.json (read by bench.py)
"""
from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("msmb::", "").strip()


def launches(csv_path: str, out: str) -> None:
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10 and r[0] != "ID"]
    seq = [(_short(r[4]), float(r[-1]), r[8]) for r in rows if r[-3] == "gpu__time_duration.sum"]
    # one step = the launches between two consecutive k_kick_drift launches in the timed region
    kd = [i for i, (n, _, _) in enumerate(seq) if n.startswith("k_kick_drift")]
    if len(kd) >= 2:
        # the shortest interval between two drifts that holds a pair-kernel launch (the bench also
        # launches the FP64 peak microbenchmark and per-stage timing passes between some of them)
        spans = [(sum(t for _, t, _ in seq[x:y]), x, y) for x, y in zip(kd[:-1], kd[1:])
                 if any(n.startswith("k_pairs_mw") for n, _, _ in seq[x:y])]
        _, a, b = min(spans) if spans else (0, kd[-2], kd[-1])
    else:
        a, b = 0, len(seq)
    step = seq[a:b]
    tot = sum(t for _, t, _ in step)
    agg: "OrderedDict[str, list]" = OrderedDict()
    for n, t, grid in step:
        e = agg.setdefault(n, [0, 0.0, grid])
        e[0] += 1
        e[1] += t
    lines = [f"# Launch list summary ({Path(csv_path).name})", "",
             "Source: `ncu --metrics gpu__time_duration.sum --clock-control none` over "
             "`python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e` (C2-S, 300,000 atoms).",
             "ncu serialises launches and runs them cold-cache, and the side-stream overlap of the",
             "long-range chain is lost, so absolute times exceed the bench's; the per-kernel SHARE",
             "of one step is what this list is for.", "",
             f"One Verlet step (launches {a}..{b - 1} of the list): {len(step)} launches, "
             f"sum of kernel durations {tot / 1e3:.1f} us.", "",
             "| kernel | launches | sum (us) | share of step |", "|---|---:|---:|---:|"]
    for n, (c, t, _) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {n} | {c} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
    Path(out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue slots busy"),
    ("sm__inst_executed.sum.per_cycle_active", "IPC (per SM... summed)"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe (inst executed)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles active"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared-memory bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared-memory pipe busy"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput"),
    ("smsp__pcsamp_warps_issue_stalled_no_instructions", None),
]


def _to_bytes(val: str, unit: str) -> float:
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(val.replace(",", "")) * mult.get(unit, 1)


def full(rep: str, out: str, traffic_key: str | None) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(head)}
    kname = vals[col["Kernel Name"]] if "Kernel Name" in col else "?"
    lines = [f"# ncu --set full: {_short(kname)} ({Path(rep).name})", "",
             "Captured with `ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 2 -c 1`",
             "over `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e` (C2-S, 300,000 atoms).", "",
             "| metric | value | unit |", "|---|---:|---|"]
    got = {}
    for m, label in WANT:
        if m in col and label:
            got[m] = (vals[col[m]], units[col[m]])
            lines.append(f"| {label} (`{m}`) | {vals[col[m]]} | {units[col[m]]} |")
    # warp-stall breakdown (top reasons)
    stalls = []
    for h, i in col.items():
        mm = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", h)
        if mm:
            try:
                stalls.append((float(vals[i]), mm.group(1)))
            except ValueError:
                pass
    if stalls:
        lines += ["", "Top warp-stall reasons (warps stalled per issued instruction):", ""]
        for v, n in sorted(stalls, reverse=True)[:8]:
            lines.append(f"- {n}: {v:.3f}")
    Path(out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_key and "dram__bytes_read.sum" in got and "dram__bytes_write.sum" in got:
        tb = _to_bytes(*got["dram__bytes_read.sum"]) + _to_bytes(*got["dram__bytes_write.sum"])
        tf = ROOT / "profiles" / "ncu_traffic.json"
        d = json.loads(tf.read_text()) if tf.exists() else {}
        ent = d.setdefault(traffic_key, {})
        ent[f"{_short(kname)}_dram_bytes"] = tb
        if _short(kname).startswith("k_pairs_mw"):
            ent["k_pairs_mw_dram_bytes"] = tb
        ent["source"] = f"profiles/{Path(out).name}"
        tf.write_text(json.dumps(d, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
        full(sys.argv[2], sys.argv[3], key)
