#!/usr/bin/env bash
set -u
OUT=gpurun_out/${1:-e2e_small}
mkdir -p "$OUT"
timeout 300 python tools/probe_e2e_small.py > "$OUT/e2e_small.jsonl" 2> "$OUT/e2e_small.err"
echo done > "$OUT/DONE"
