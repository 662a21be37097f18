#!/usr/bin/env bash
set -u
OUT=gpurun_out/${1:-copyfloor}
mkdir -p "$OUT"
for r in 1 2; do
  timeout 900 python tools/copy_floor.py >> "$OUT/copy_floor.jsonl" 2>> "$OUT/copy_floor.err"
done
echo done > "$OUT/DONE"
