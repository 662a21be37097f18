#!/usr/bin/env bash
# Runtime-matrix kernel with output groups: ring_rt GPU tests, bench_rt incl. the paper's (60,40) code.
set -u
OUT=gpurun_out/${1:-rt12}
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_ring_rt.py tests/test_negative_control.py -q -m gpu -x > "$OUT/tests.log" 2>&1
echo "tests exit $?" >> "$OUT/tests.log"
timeout 900 python tools/bench_rt.py --configs 2,3,4,5 --patterns 6 --paper > "$OUT/bench_rt.jsonl" 2> "$OUT/bench_rt.err"
timeout 900 python tools/soak.py --rt --cases 300 --seed 43 > "$OUT/soak_rt.json" 2> "$OUT/soak_rt.err"
echo done > "$OUT/DONE"
