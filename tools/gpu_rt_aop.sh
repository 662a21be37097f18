#!/usr/bin/env bash
# A/B: every pair distance in the all-one-polynomial fields (this tree) vs distances <= 3
# everywhere (build/ab_old = the previous commit), budgets 18/22/26 KB; config-5 decode patterns.
set -u
OUT=$PWD/gpurun_out/${1:-rt_aop}
mkdir -p "$OUT"
cp tools/bench_rt.py build/ab_old/tools/
for r in 1 2; do
  (cd build/ab_old && timeout 900 python tools/bench_rt.py --configs 1,3,5 --patterns 6 --pattern-config 5) >> "$OUT/old.jsonl" 2>> "$OUT/err.log"
  for kb in 18 22 26; do
    PYRIT_B200_RT_CODE_KB=$kb timeout 900 python tools/bench_rt.py --configs 1,3,5 --patterns 6 --pattern-config 5 >> "$OUT/new_kb$kb.jsonl" 2>> "$OUT/err.log"
  done
done
timeout 600 python tools/bench_rt.py --configs 2,4 --patterns 4 >> "$OUT/new_c24.jsonl" 2>> "$OUT/err.log"
timeout 900 python -m pytest tests/test_gpu_ring_rt.py tests/test_negative_control.py -m gpu -x -q > "$OUT/pytest_rt.log" 2>&1
timeout 1200 python tools/soak.py --rt --cases 600 --seed 81 > "$OUT/soak_rt_seed81.json" 2> "$OUT/soak.err"
echo done > "$OUT/DONE"
