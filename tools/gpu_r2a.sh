mkdir -p gpurun_out
timeout 300 python tools/host_cost.py > gpurun_out/r2a_host_cost.json 2>&1
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/r2a_gpu_tests.log 2>&1
tail -3 gpurun_out/r2a_gpu_tests.log
