set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_ring_rt.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/rt1_tests.log
timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 6 --out gpurun_out/rt1_bench.jsonl > gpurun_out/rt1_bench.log 2>&1
for v in 1 2; do PYRIT_B200_RT_V=$v timeout 300 python tools/bench_rt.py --configs 4,5 > gpurun_out/rt1_bench_v$v.log 2>&1; done
