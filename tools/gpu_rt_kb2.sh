#!/usr/bin/env bash
# Case-code budget of the runtime-matrix planner re-swept with the producer warp group.
set -u
OUT=$PWD/gpurun_out/${1:-rt_kb2}
mkdir -p "$OUT"
for r in 1 2; do
for kb in 18 22 26 30 34; do
  PYRIT_B200_RT_CODE_KB=$kb timeout 300 python tools/bench_rt.py --configs 2,3,4,5 --patterns 4 --pattern-config 5 >> "$OUT/kb$kb.jsonl" 2>> "$OUT/err.log"
done
done
echo done > "$OUT/DONE"
