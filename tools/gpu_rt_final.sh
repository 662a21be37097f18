#!/usr/bin/env bash
# ncu --set full of the kept runtime-matrix kernel at configs 4 and 5 (csv exports only).
set -u
OUT=gpurun_out/${1:-rt_final}
mkdir -p "$OUT"
for c in 4 5; do
  R=/tmp/rtf_cfg$c
  timeout 300 python tools/bench_rt.py --configs $c --reps 2 > "$OUT/plain_c$c.log" 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_rt_kernel -c 1 \
    -f -o $R python tools/bench_rt.py --configs $c --reps 2 > "$OUT/ncu_c$c.log" 2>&1
  ncu -i $R.ncu-rep --page raw --csv > "$OUT/raw_c$c.csv" 2>/dev/null
done
echo done > "$OUT/DONE"
