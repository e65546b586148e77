#!/bin/bash
# A/B step times of bench.py under environment variants: tools/ab_bench.sh "VAR=a VAR2=b" "VAR=c" ...
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  env $cfg python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-scaling-base > /tmp/ab.json 2>/tmp/ab.err || { echo "$cfg FAILED"; tail -3 /tmp/ab.err; continue; }
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("/tmp/ab.json").read().strip().splitlines()[-1])
s = d["stage_ms_per_eval"]; w = d["work"]
print(sys.argv[1], "ms/step %.4f" % d["ms_per_step"], " ".join("%s %.4f" % (k, s[k]) for k in ("pairs", "anterp", "sort", "clusters", "interp")),
      "cand %.4g pairs %.4g clk/warp-step %.1f" % (w["candidates"], w["pairs"], s["pairs"] * 1.965e6 * 148 / (w["candidates"] / 32.0)),
      "rebuild-every-step %.4f" % d["rebuild_every_step"]["ms_per_step"])
PY
done
