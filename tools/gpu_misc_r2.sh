#!/usr/bin/env bash
# Sustained config-5 run (500 steps) and the N-rank harness at N = 4 and 8 on one GPU (gloo).
set -u
OUT=gpurun_out/${1:-misc}
mkdir -p "$OUT"
timeout 600 python bench.py --steps 500 --warmup 5 --no-e2e --no-cpu-baseline > "$OUT/bench_cfg5_500steps.jsonl" 2> "$OUT/bench_cfg5_500steps.err"
for n in 4 8; do
  PYRIT_B200_DIST_BACKEND=gloo timeout 1200 python bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    > "$OUT/bench_gloo$n.jsonl" 2> "$OUT/bench_gloo$n.err"
done
echo done > "$OUT/DONE"
