#!/usr/bin/env bash
# Build A/B variants of the library under build/ab_*: HEAD as committed (ab_head) and the
# working tree with PYRIT_RT_PAIR_D = 0..3 (ab_d0..ab_d3).  Run here (CPU); the copies
# travel to the GPU box with gpurun, tools/gpu_rt_pairs.sh runs them.
set -eu
cd "$(dirname "$0")/.."
rm -rf build/ab_head build/ab_d0 build/ab_d1 build/ab_d2 build/ab_d3
mkdir -p build/ab_head
git archive HEAD | tar -x -C build/ab_head
cp MEASURED_PEAKS.json build/ab_head/ 2>/dev/null || true
mkdir -p build/ab_head/paper_1709_00178_b200/kernels
cp paper_1709_00178_b200/kernels/*.cubin build/ab_head/paper_1709_00178_b200/kernels/
(cd build/ab_head && python -c "from paper_1709_00178_b200 import build as B; B.build_library()" > build.log 2>&1)
for d in 0 1 2 3; do
  v=build/ab_d$d
  mkdir -p $v
  cp -r paper_1709_00178_b200 tools include MEASURED_PEAKS.json $v/ 2>/dev/null || true
  rm -f $v/paper_1709_00178_b200/libpyrit_b200.so
  (cd $v && PYRIT_B200_BUILD_RT_PAIR_D=$d python -c "from paper_1709_00178_b200 import build as B; B.build_library()" > build.log 2>&1)
  ls -la $v/paper_1709_00178_b200/libpyrit_b200.so
done
