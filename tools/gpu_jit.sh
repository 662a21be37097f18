#!/usr/bin/env bash
# Kernel compile latency per plan (tools/jit_latency.py), in process and tiered.
set -u
OUT=gpurun_out/${1:-jit}
mkdir -p "$OUT"
nproc > "$OUT/host.txt"; lscpu | grep -E "Model name|^CPU\(s\)" >> "$OUT/host.txt"
timeout 1500 python tools/jit_latency.py > "$OUT/jit_inprocess.jsonl" 2> "$OUT/jit_inprocess.err"
timeout 1500 python tools/jit_latency.py --tiered > "$OUT/jit_tiered.jsonl" 2> "$OUT/jit_tiered.err"
echo done > "$OUT/DONE"
