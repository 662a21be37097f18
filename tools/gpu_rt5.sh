#!/usr/bin/env bash
# Runtime-matrix kernel V=2 vs V=4: ring_rt GPU tests (default V), bench_rt on
# both, ncu --set full of the ring_rt kernel at config 4 and 5 for both
# (exported to csv on the box; only the V=4 config-4 report is kept).
set -u
OUT=gpurun_out/${1:-rt5}
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_ring_rt.py tests/test_gpu_fullsize_reference.py tests/test_negative_control.py -q -m gpu -x > "$OUT/tests.log" 2>&1
echo "tests exit $?" >> "$OUT/tests.log"
for v in 2 4; do
  PYRIT_B200_RT_V=$v timeout 600 python tools/bench_rt.py --configs 1,2,3,4,5 --patterns 6 > "$OUT/bench_rt_v$v.jsonl" 2> "$OUT/bench_rt_v$v.err"
done
for v in 2 4; do for c in 4 5; do
  R=/tmp/rt_v${v}_cfg$c
  PYRIT_B200_RT_V=$v timeout 300 python tools/bench_rt.py --configs $c --reps 2 > "$OUT/plain_v${v}_c$c.log" 2>&1 && \
  PYRIT_B200_RT_V=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_rt_kernel -c 1 \
    -f -o $R python tools/bench_rt.py --configs $c --reps 2 > "$OUT/ncu_v${v}_c$c.log" 2>&1
  ncu -i $R.ncu-rep --page raw --csv > "$OUT/raw_v${v}_c$c.csv" 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass > "$OUT/src_v${v}_c$c.csv" 2>/dev/null
  ls -la $R.ncu-rep >> "$OUT/sizes.txt" 2>&1
done; done
cp /tmp/rt_v4_cfg4.ncu-rep "$OUT/" 2>/dev/null
du -sh gpurun_out > "$OUT/du.txt"
echo done > "$OUT/DONE"
