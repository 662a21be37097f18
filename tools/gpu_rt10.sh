#!/usr/bin/env bash
# Runtime-matrix kernel: ring_rt GPU tests, bench_rt (two runs), ncu of configs 4 and 5.
set -u
OUT=gpurun_out/${1:-rt10}
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_ring_rt.py tests/test_gpu_fullsize_reference.py tests/test_negative_control.py -q -m gpu -x > "$OUT/tests.log" 2>&1
echo "tests exit $?" >> "$OUT/tests.log"
for r in a b; do
  timeout 600 python tools/bench_rt.py --configs 1,2,3,4,5 --patterns 6 > "$OUT/bench_rt_$r.jsonl" 2> "$OUT/bench_rt_$r.err"
done
for c in 4 5; do
  R=/tmp/rt10_cfg$c
  timeout 300 python tools/bench_rt.py --configs $c --reps 2 > "$OUT/plain_c$c.log" 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_rt_kernel -c 1 \
    -f -o $R python tools/bench_rt.py --configs $c --reps 2 > "$OUT/ncu_c$c.log" 2>&1
  ncu -i $R.ncu-rep --page raw --csv > "$OUT/raw_c$c.csv" 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass > "$OUT/src_c$c.csv" 2>/dev/null
done
echo done > "$OUT/DONE"
