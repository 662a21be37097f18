#!/usr/bin/env bash
# Compile latency per plan, steady state (after a warm-up compile), in process and tiered, twice.
set -u
OUT=gpurun_out/${1:-jit2}
mkdir -p "$OUT"
for r in 1 2; do
  timeout 1500 python tools/jit_latency.py --tiered >> "$OUT/jit_tiered.jsonl" 2>> "$OUT/jit_tiered.err"
  timeout 1500 python tools/jit_latency.py >> "$OUT/jit_inprocess.jsonl" 2>> "$OUT/jit_inprocess.err"
done
echo done > "$OUT/DONE"
