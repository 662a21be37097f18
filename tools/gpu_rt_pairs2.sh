#!/usr/bin/env bash
# Paired-shift build (D = 3, footprint-limited): ring_rt GPU tests, negative control,
# bench_rt for the BASELINE configs and random patterns, the code-budget sweep, a soak.
set -u
OUT=$PWD/gpurun_out/${1:-rt_pairs2}
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_ring_rt.py tests/test_negative_control.py tests/test_gpu_generic.py -m gpu -x -q > "$OUT/pytest_rt.log" 2>&1
echo "exit $?" >> "$OUT/pytest_rt.log"
for r in 1 2; do
  timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 6 >> "$OUT/bench_rt.jsonl" 2>> "$OUT/bench_rt.err"
done
for kb in 0 24 30 34 38 44 64; do
  PYRIT_B200_RT_CODE_KB=$kb timeout 600 python tools/bench_rt.py --configs 2,3,4,5 >> "$OUT/code_kb_$kb.jsonl" 2>> "$OUT/code_kb.err"
done
timeout 600 python tools/bench_rt.py --configs 5 --paper >> "$OUT/bench_rt_paper.jsonl" 2>> "$OUT/bench_rt.err"
timeout 1200 python tools/soak.py --rt --cases 600 --seed 51 > "$OUT/soak_rt_seed51.json" 2> "$OUT/soak_rt_seed51.err"
echo "exit $?" >> "$OUT/soak_rt_seed51.err"
echo done > "$OUT/DONE"
