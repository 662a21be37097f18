#!/usr/bin/env bash
# Build with pair distances <= 3: min-use x budget of the planner's case selection.
set -u
OUT=$PWD/gpurun_out/${1:-rt_pairs5}
mkdir -p "$OUT"
for r in 1 2 3; do
for mu in 1 2 3; do
for kb in 20 26 34; do
  PYRIT_B200_RT_PAIR_MINUSE=$mu PYRIT_B200_RT_CODE_KB=$kb timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 4 >> "$OUT/mu${mu}_kb${kb}.jsonl" 2>> "$OUT/err.log"
done
done
done
echo done > "$OUT/DONE"
