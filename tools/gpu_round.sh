#!/usr/bin/env bash
# One measurement pass on a gpurun box (run from the repo root):
#   GPU parity tests, smoke, bench (config 5 + the other configs), the reference
#   CPU arm, the ncu launch list of the default bench command and one
#   `ncu --set full` capture of the config-5 kernel.
#   usage: tools/gpu_round.sh TAG [quick]
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > "$OUT/smi.txt" 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke exit $?" >> "$OUT/smoke.log"
timeout 600 python bench.py > "$OUT/bench_cfg5.jsonl" 2> "$OUT/bench_cfg5.err"
if [ "${2:-}" != "quick" ]; then
  for c in 1 2 3 4; do
    timeout 300 python bench.py --config $c --no-cpu-baseline >> "$OUT/bench_cfgs.jsonl" 2>> "$OUT/bench_cfgs.err"
  done
  timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.jsonl" 2> "$OUT/bench_reference.err"
  CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
  $CMD > "$OUT/plain.log" 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches_cfg5.csv" $CMD > "$OUT/ncu_launches.log" 2>&1
  $CMD > "$OUT/plain2.log" 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pyrit_ring -s 3 -c 1 \
    -o "$OUT/prof_cfg5" $CMD > "$OUT/ncu_full.log" 2>&1
fi
echo done > "$OUT/DONE"
