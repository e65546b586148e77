bash tools/ab_bench.sh "X=0" "X=1"
MSMB_TIMELINE=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-scaling-base 2>&1 >/dev/null | grep -E "timeline|chain:" | head -2
timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/t37_t.txt 2>&1; tail -n 3 gpurun_out/t37_t.txt
