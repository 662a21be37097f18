mkdir -p gpurun_out
timeout 300 python tools/bench_rt.py --configs 2,3,4,5 --patterns 4 > gpurun_out/rt2_alg0.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ring_rt.py -x -q -m gpu 2>&1 | tail -5 > gpurun_out/rt2_tests_alg1.log
