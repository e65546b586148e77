#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  env $cfg python bench.py --config c5s --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-scaling-base > /tmp/ab.json 2>/tmp/ab.err || { echo "$cfg FAILED"; tail -3 /tmp/ab.err; continue; }
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("/tmp/ab.json").read().strip().splitlines()[-1])
s = d["stage_ms_per_eval"]
print(sys.argv[1], "ms/step %.4f" % d["ms_per_step"], "pairs %.4f" % s["pairs"], d["config"].get("n_atoms"))
PY
done
