#!/usr/bin/env bash
# ncu --set full captures of the bench kernel of every config (N = 1) and of
# rank 0's config-5 shard at N = 2, 4, 8 (tools/shard_scaling.py), each after
# the same command has exited 0 without ncu.  Output: gpurun_out/$TAG/.
#   usage: tools/ncu_traffic.sh TAG
set -u
TAG=${1:-traffic}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for c in 1 2 3 4 5; do
  CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
  $CMD > "$OUT/plain_cfg$c.log" 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pyrit_ring \
    -s 3 -c 1 -o "$OUT/prof_cfg$c" $CMD > "$OUT/ncu_cfg$c.log" 2>&1
done
for n in 2 4 8; do
  CMD="python tools/shard_scaling.py --config 5 --only $n --steps 2 --warmup 2"
  $CMD > "$OUT/plain_shard$n.log" 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pyrit_ring \
    -s 1 -c 1 -o "$OUT/prof_cfg5_shard$n" $CMD > "$OUT/ncu_shard$n.log" 2>&1
done
echo done > "$OUT/DONE"
