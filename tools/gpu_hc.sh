timeout 300 python tools/host_cost.py > gpurun_out/r2a_host_cost.json 2>&1
