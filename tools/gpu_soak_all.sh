#!/usr/bin/env bash
# Randomised soak of the generated kernels (default and --knobs) and of the runtime-matrix kernel.
set -u
OUT=gpurun_out/${1:-soak_all}
mkdir -p "$OUT"
timeout 1500 python tools/soak.py --cases 300 --seed 51 > "$OUT/soak_seed51.json" 2> "$OUT/soak_seed51.err"
timeout 1500 python tools/soak.py --knobs --cases 300 --seed 52 > "$OUT/soak_knobs_seed52.json" 2> "$OUT/soak_knobs_seed52.err"
timeout 1500 python tools/soak.py --rt --cases 400 --seed 53 > "$OUT/soak_rt_seed53.json" 2> "$OUT/soak_rt_seed53.err"
echo done > "$OUT/DONE"
