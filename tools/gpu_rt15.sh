#!/usr/bin/env bash
# Runtime-matrix kernel: outputs as solo groups (one 256-thread part per unit, 2 CTAs/SM) vs parts.
set -u
OUT=gpurun_out/${1:-rt15}
mkdir -p "$OUT"
for s in 0 1 0 1; do
  PYRIT_B200_RT_SOLO=$s timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 2 >> "$OUT/bench_solo$s.jsonl" 2>> "$OUT/bench_solo$s.err"
done
PYRIT_B200_RT_SOLO=1 timeout 600 python -m pytest tests/test_gpu_ring_rt.py -q -m gpu -x > "$OUT/tests_solo.log" 2>&1
echo done > "$OUT/DONE"
