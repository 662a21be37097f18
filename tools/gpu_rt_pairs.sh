#!/usr/bin/env bash
# A/B in one lease: runtime-matrix kernel variants built by tools/prep_rt_pairs.sh
# (HEAD, and paired-shift cases with D = 0..3), alternating, two rounds.
set -u
OUT=$PWD/gpurun_out/${1:-rt_pairs}
mkdir -p "$OUT"
for r in 1 2; do
  for v in head d0 d1 d2 d3; do
    (cd build/ab_$v && timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 6) >> "$OUT/$v.jsonl" 2>> "$OUT/$v.err"
  done
done
echo done > "$OUT/DONE"
