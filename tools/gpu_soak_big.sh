#!/usr/bin/env bash
# A long soak on the final build: generated kernels with random knobs, and the runtime-matrix kernel.
set -u
OUT=gpurun_out/${1:-soak_big}
mkdir -p "$OUT"
timeout 2400 python tools/soak.py --knobs --cases 1200 --seed 61 > "$OUT/soak_knobs_seed61.json" 2> "$OUT/soak_knobs_seed61.err"
timeout 2400 python tools/soak.py --rt --cases 2000 --seed 62 > "$OUT/soak_rt_seed62.json" 2> "$OUT/soak_rt_seed62.err"
timeout 2400 python tools/soak.py --cases 800 --seed 63 > "$OUT/soak_seed63.json" 2> "$OUT/soak_seed63.err"
echo done > "$OUT/DONE"
