#!/usr/bin/env bash
# ncu --set full of the runtime-matrix kernel with the producer group at configs 4 and 5:
# raw metrics and the per-instruction source page (csv exports only).
set -u
OUT=$PWD/gpurun_out/${1:-rt_ncu2}
mkdir -p "$OUT"
for c in 4 5; do
  R=/tmp/rtn_cfg$c
  timeout 300 python tools/bench_rt.py --configs $c --reps 2 > "$OUT/plain_c$c.log" 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_rt_kernel -c 1 \
    -f -o $R python tools/bench_rt.py --configs $c --reps 2 > "$OUT/ncu_c$c.log" 2>&1
  ncu -i $R.ncu-rep --page raw --csv > "$OUT/raw_c$c.csv" 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass > "$OUT/src_c$c.csv" 2>/dev/null
done
echo done > "$OUT/DONE"
