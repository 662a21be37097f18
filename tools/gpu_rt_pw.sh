#!/usr/bin/env bash
# Runtime-matrix kernel, four-part shape: TMA copies from a producer warp group
# (PYRIT_B200_RT_PW=1, setmaxnreg 112/24) vs from the lightest part's first thread.
# A short canary first: a wrong register budget would make setmaxnreg.inc wait for ever.
set -u
OUT=$PWD/gpurun_out/${1:-rt_pw}
mkdir -p "$OUT"
PYRIT_B200_RT_PW=1 timeout 120 python tools/probe_rt_small.py > "$OUT/canary.json" 2> "$OUT/canary.err"
rc=$?
echo "canary exit $rc" >> "$OUT/canary.err"
if [ $rc -ne 0 ]; then nvidia-smi > "$OUT/smi_after_canary.txt" 2>&1; echo canary-failed > "$OUT/DONE"; exit 0; fi
PYRIT_B200_RT_PW=1 timeout 600 python -m pytest tests/test_gpu_ring_rt.py tests/test_negative_control.py -m gpu -x -q > "$OUT/pytest_rt_pw1.log" 2>&1
rc=$?
echo "exit $rc" >> "$OUT/pytest_rt_pw1.log"
if [ $rc -ne 0 ]; then echo tests-failed > "$OUT/DONE"; exit 0; fi
for r in 1 2 3; do
  for pw in 0 1; do
    PYRIT_B200_RT_PW=$pw timeout 300 python tools/bench_rt.py --configs 2,3,4,5 --patterns 4 >> "$OUT/pw$pw.jsonl" 2>> "$OUT/err.log"
  done
done
PYRIT_B200_RT_PW=1 timeout 300 python tools/bench_rt.py --configs 5 --patterns 4 --pattern-config 5 >> "$OUT/pw1_c5dec.jsonl" 2>> "$OUT/err.log"
PYRIT_B200_RT_PW=0 timeout 300 python tools/bench_rt.py --configs 5 --patterns 4 --pattern-config 5 >> "$OUT/pw0_c5dec.jsonl" 2>> "$OUT/err.log"
PYRIT_B200_RT_PW=1 timeout 600 python tools/soak.py --rt --cases 400 --seed 91 > "$OUT/soak_rt_pw1.json" 2> "$OUT/soak.err"
echo done > "$OUT/DONE"
