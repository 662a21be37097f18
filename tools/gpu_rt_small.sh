#!/usr/bin/env bash
# A/B of tiny runtime-matrix launches: build/ab_old (commit before the paired-shift cases) vs now.
set -u
OUT=$PWD/gpurun_out/${1:-rt_small}
mkdir -p "$OUT"
cp tools/probe_rt_small.py build/ab_old/tools/
for r in 1 2; do
  (cd build/ab_old && timeout 300 python tools/probe_rt_small.py) >> "$OUT/old.jsonl" 2>> "$OUT/err.log"
  timeout 300 python tools/probe_rt_small.py >> "$OUT/new.jsonl" 2>> "$OUT/err.log"
  (cd build/ab_old && timeout 300 python tools/host_cost.py) >> "$OUT/old_host_cost.jsonl" 2>> "$OUT/err.log"
  timeout 300 python tools/host_cost.py >> "$OUT/new_host_cost.jsonl" 2>> "$OUT/err.log"
done
timeout 600 python -m pytest tests/test_gpu_ring_rt.py -m gpu -x -q -k rebind > "$OUT/pytest_rebind.log" 2>&1
echo done > "$OUT/DONE"
