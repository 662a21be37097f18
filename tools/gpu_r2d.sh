mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize_reference.py tests/test_gpu_ring_rt.py -q -m gpu > gpurun_out/r2d_tests.log 2>&1
timeout 300 python tools/bench_rt.py --configs 2,3,4,5 > gpurun_out/r2d_bench_rt.log 2>&1
timeout 2400 bash tools/ncu_traffic.sh r2d_traffic
