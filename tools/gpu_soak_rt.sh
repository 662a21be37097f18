#!/usr/bin/env bash
# Randomised soak of the runtime-matrix ring kernel (tools/soak.py --rt), two seeds.
set -u
OUT=gpurun_out/${1:-soak_rt}
mkdir -p "$OUT"
for s in 41 42; do
  timeout 1200 python tools/soak.py --rt --cases 600 --seed $s > "$OUT/soak_rt_seed$s.json" 2> "$OUT/soak_rt_seed$s.err"
  echo "exit $?" >> "$OUT/soak_rt_seed$s.err"
done
echo done > "$OUT/DONE"
