#!/usr/bin/env bash
# Early PDL trigger in the direct kernels (PYRIT_B200_PDL_EARLY) A/B: config-1
# launch floor tool and bench lines for configs 1 and 2, GPU parity tests.
set -u
OUT=gpurun_out/${1:-pdl}
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > "$OUT/tests.log" 2>&1
echo "tests exit $?" >> "$OUT/tests.log"
for e in 1 0 1 0; do
  PYRIT_B200_PDL_EARLY=$e timeout 300 python tools/cfg1_launch.py --steps 200 >> "$OUT/cfg1_launch_e$e.json" 2>> "$OUT/cfg1_launch_e$e.err"
  for c in 1 2; do
    PYRIT_B200_PDL_EARLY=$e timeout 300 python bench.py --config $c --no-cpu-baseline >> "$OUT/bench_e$e.jsonl" 2>> "$OUT/bench_e$e.err"
  done
done
echo done > "$OUT/DONE"
