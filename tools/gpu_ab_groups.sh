#!/usr/bin/env bash
# A/B in one lease: the runtime-matrix kernel before output groups (build/ab_old, a
# worktree of the previous commit) vs now; alternating runs.
set -u
OUT=gpurun_out/${1:-ab_groups}
mkdir -p "$OUT"
for r in 1 2; do
  (cd build/ab_old && timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 6) >> "$OUT/old.jsonl" 2>> "$OUT/old.err"
  timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 6 >> "$OUT/new.jsonl" 2>> "$OUT/new.err"
done
echo done > "$OUT/DONE"
