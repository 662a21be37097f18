mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_negative_control.py tests/test_gpu_ring_rt.py tests/test_gpu_generic.py -q -m gpu > gpurun_out/r2c_tests.log 2>&1
timeout 300 python tools/pipe_trace.py --config 5 --out gpurun_out/r2c_pipe_trace_cfg5.json > gpurun_out/r2c_pipe.log 2>&1
timeout 300 python tools/pipe_trace.py --config 4 --out gpurun_out/r2c_pipe_trace_cfg4.json >> gpurun_out/r2c_pipe.log 2>&1
timeout 300 python tools/cfg1_launch.py --out gpurun_out/r2c_cfg1_launch.json > gpurun_out/r2c_cfg1.log 2>&1
timeout 600 python bench.py --config 4 --erased 0,1,2,3 > gpurun_out/r2c_bench_cfg4_data.json 2> gpurun_out/r2c_bench_cfg4_data.err
timeout 2400 bash tools/exit_race.sh 100 > gpurun_out/r2c_exit_race.log 2>&1
