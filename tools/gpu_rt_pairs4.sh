#!/usr/bin/env bash
# Pair-distance cap x case-code budget sweep of the runtime-matrix planner.
set -u
OUT=$PWD/gpurun_out/${1:-rt_pairs4}
mkdir -p "$OUT"
for r in 1 2; do
for dm in 1 2 3 4 6 8; do
for kb in 16 20 24 34; do
  PYRIT_B200_RT_PAIR_DMAX=$dm PYRIT_B200_RT_CODE_KB=$kb timeout 600 python tools/bench_rt.py --configs 2,4,5 --patterns 3 >> "$OUT/d${dm}_kb${kb}.jsonl" 2>> "$OUT/err.log"
done
done
done
echo done > "$OUT/DONE"
