#!/usr/bin/env bash
# Final paired-shift build (incremental case selection): ring_rt tests, bench_rt, host cost
# of first calls, and ncu --set full of the kernel at configs 4 and 5.
set -u
OUT=$PWD/gpurun_out/${1:-rt_pairs6}
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_ring_rt.py tests/test_negative_control.py tests/test_gpu_generic.py tests/test_gpu_fullsize_reference.py -m gpu -x -q > "$OUT/pytest_rt.log" 2>&1
echo "exit $?" >> "$OUT/pytest_rt.log"
timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 8 >> "$OUT/bench_rt.jsonl" 2>> "$OUT/bench_rt.err"
timeout 300 python tools/host_cost.py > "$OUT/host_cost.json" 2> "$OUT/host_cost.err"
timeout 300 python tools/probe_rt_small.py > "$OUT/rt_small.json" 2>> "$OUT/host_cost.err"
bash tools/gpu_rt_final.sh $(basename $OUT)/ncu
timeout 1200 python tools/soak.py --rt --cases 600 --seed 71 > "$OUT/soak_rt_seed71.json" 2> "$OUT/soak_rt_seed71.err"
echo done > "$OUT/DONE"
