#!/usr/bin/env bash
# Runtime-matrix kernel: four parts per CTA vs two parts per CTA (two CTAs per SM, output groups).
set -u
OUT=gpurun_out/${1:-rt13}
mkdir -p "$OUT"
for p in 4 2 4 2; do
  PYRIT_B200_RT_PARTS=$p timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 6 >> "$OUT/bench_rt_p$p.jsonl" 2>> "$OUT/bench_rt_p$p.err"
done
PYRIT_B200_RT_PARTS=2 timeout 600 python -m pytest tests/test_gpu_ring_rt.py -q -m gpu -x > "$OUT/tests_p2.log" 2>&1
echo done > "$OUT/DONE"
