mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2b_bench_cfg5.json 2> gpurun_out/r2b_bench_cfg5.err
timeout 600 python bench.py --config 4 > gpurun_out/r2b_bench_cfg4.json 2> gpurun_out/r2b_bench_cfg4.err
PYRIT_B200_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 > gpurun_out/r2b_bench_gloo2.json 2> gpurun_out/r2b_bench_gloo2.err
free -g > gpurun_out/r2b_free.txt; nproc >> gpurun_out/r2b_free.txt
