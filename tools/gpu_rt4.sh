#!/usr/bin/env bash
# Runtime-matrix kernel V=2 (two 256-thread parts) vs V=4 (16 bytes per thread,
# up to four 128-thread parts): GPU tests on the default (V=4), bench_rt on both,
# one ncu --set full capture of the V=4 config-4 decode kernel.
set -u
OUT=gpurun_out/${1:-rt4}
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_ring_rt.py tests/test_gpu_fullsize_reference.py tests/test_negative_control.py -q -m gpu -x > "$OUT/tests.log" 2>&1
echo "tests exit $?" >> "$OUT/tests.log"
for v in 2 4; do
  PYRIT_B200_RT_V=$v timeout 600 python tools/bench_rt.py --configs 1,2,3,4,5 --patterns 6 > "$OUT/bench_rt_v$v.jsonl" 2> "$OUT/bench_rt_v$v.err"
done
PYRIT_B200_RT_V=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_rt_kernel -c 1 \
  -o "$OUT/rt_v4_cfg4" python tools/bench_rt.py --configs 4 --reps 2 > "$OUT/ncu.log" 2>&1
echo done > "$OUT/DONE"
