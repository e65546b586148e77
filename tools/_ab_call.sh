bash tools/ab_bench.sh "X=0" "X=1"
timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/t33_t.txt 2>&1; tail -n 3 gpurun_out/t33_t.txt
