#!/usr/bin/env bash
# All-distance pair cases chosen per matrix within an instruction-cache budget
# (runtime.cpp rt_select_pairs): budget sweep, then tests, random patterns and a soak
# at the default.
set -u
OUT=$PWD/gpurun_out/${1:-rt_pairs3}
mkdir -p "$OUT"
for r in 1 2; do
for kb in 0 16 20 24 28 32 36 40; do
  PYRIT_B200_RT_CODE_KB=$kb timeout 600 python tools/bench_rt.py --configs 2,3,4,5 >> "$OUT/code_kb_$kb.jsonl" 2>> "$OUT/code_kb.err"
done
done
timeout 900 python -m pytest tests/test_gpu_ring_rt.py tests/test_negative_control.py tests/test_gpu_generic.py -m gpu -x -q > "$OUT/pytest_rt.log" 2>&1
echo "exit $?" >> "$OUT/pytest_rt.log"
timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 6 --paper >> "$OUT/bench_rt.jsonl" 2>> "$OUT/bench_rt.err"
timeout 1200 python tools/soak.py --rt --cases 600 --seed 52 > "$OUT/soak_rt_seed52.json" 2> "$OUT/soak_rt_seed52.err"
echo "exit $?" >> "$OUT/soak_rt_seed52.err"
timeout 300 python tools/host_cost.py > "$OUT/host_cost.json" 2> "$OUT/host_cost.err"
echo done > "$OUT/DONE"
