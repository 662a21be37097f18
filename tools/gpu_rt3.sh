mkdir -p gpurun_out
export PYRIT_B200_RT_ALG=${ALG:-0}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ring_rt_kernel -c 1 -o gpurun_out/rt3_cfg4_alg$PYRIT_B200_RT_ALG python tools/bench_rt.py --configs 4 --reps 2 > gpurun_out/rt3_ncu.log 2>&1
tail -5 gpurun_out/rt3_ncu.log
