#!/usr/bin/env bash
# Case-code budget for the GF(2^8)/R17 code (config 2/4 and random config-4 patterns), fine sweep.
set -u
OUT=$PWD/gpurun_out/${1:-rt_kb3}
mkdir -p "$OUT"
for r in 1 2; do
for kb in 10 12 14 16 18 20 22 26; do
  PYRIT_B200_RT_CODE_KB=$kb timeout 300 python tools/bench_rt.py --configs 2,4 --patterns 8 >> "$OUT/kb$kb.jsonl" 2>> "$OUT/err.log"
done
done
echo done > "$OUT/DONE"
