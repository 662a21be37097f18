#!/usr/bin/env bash
# ncu --set full with source-level (SASS) stall samples of the runtime-matrix kernel
# at one config: raw csv + source csv land in gpurun_out/$TAG/.
#   usage: tools/gpu_rt_src.sh TAG [CONFIGS="4 5"]
set -u
OUT=gpurun_out/${1:-rt_src}
CFGS=${2:-"4 5"}
mkdir -p "$OUT"
for c in $CFGS; do
  R=/tmp/rts_cfg$c
  timeout 300 python tools/bench_rt.py --configs $c --reps 5 > "$OUT/plain_c$c.log" 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:ring_rt_kernel -c 1 \
    -f -o $R python tools/bench_rt.py --configs $c --reps 2 > "$OUT/ncu_c$c.log" 2>&1
  ncu -i $R.ncu-rep --page raw --csv > "$OUT/raw_c$c.csv" 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass > "$OUT/src_c$c.csv" 2>/dev/null
done
echo done > "$OUT/DONE"
