#!/usr/bin/env bash
# Full pass after the paired-shift cases of the runtime-matrix kernel: gpu_round.sh, then
# bench_rt (BASELINE configs, random patterns, erasure counts, the paper code) and a soak.
set -u
TAG=${1:-r2l}
bash tools/gpu_round.sh $TAG
OUT=$PWD/gpurun_out/$TAG
for r in 1 2; do
  timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 8 --paper >> "$OUT/bench_rt.jsonl" 2>> "$OUT/bench_rt.err"
done
PYRIT_B200_RT_PAIRS=0 timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 8 --paper >> "$OUT/bench_rt_singles_only.jsonl" 2>> "$OUT/bench_rt.err"
timeout 1200 python tools/soak.py --rt --cases 1000 --seed 61 > "$OUT/soak_rt_seed61.json" 2> "$OUT/soak_rt_seed61.err"
timeout 300 python tools/host_cost.py > "$OUT/host_cost.json" 2> "$OUT/host_cost.err"
echo done > "$OUT/DONE2"
