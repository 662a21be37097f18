#!/usr/bin/env bash
# Config 5: the tuned kernel (512 threads, no pair sharing) vs 256 threads with pair sharing
# within one output's rows (1905 instead of 2745 XORs per column word), short and sustained.
set -u
OUT=gpurun_out/${1:-cse5}
mkdir -p "$OUT"
for r in 1 2; do
  for v in base cse; do
    if [ $v = cse ]; then export PYRIT_B200_THREADS=256 PYRIT_B200_PART_CSE=1 PYRIT_B200_CSE_WINDOW=13; else unset PYRIT_B200_THREADS PYRIT_B200_PART_CSE PYRIT_B200_CSE_WINDOW; fi
    timeout 600 python bench.py --steps 20 --no-e2e --no-cpu-baseline >> "$OUT/bench20_$v.jsonl" 2>> "$OUT/err_$v.log"
    timeout 600 python bench.py --steps 500 --no-e2e --no-cpu-baseline >> "$OUT/bench500_$v.jsonl" 2>> "$OUT/err_$v.log"
  done
done
echo done > "$OUT/DONE"
