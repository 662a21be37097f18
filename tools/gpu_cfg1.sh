#!/usr/bin/env bash
# Config-1 floor: the encode kernel vs torch kernels moving the same bytes in the same graph setup.
set -u
OUT=gpurun_out/${1:-cfg1}
mkdir -p "$OUT"
for r in 1 2 3; do
  timeout 300 python tools/cfg1_launch.py --steps 200 >> "$OUT/cfg1_launch.jsonl" 2>> "$OUT/cfg1_launch.err"
done
echo done > "$OUT/DONE"
