#!/usr/bin/env bash
# ncu --set full captures of the bench kernel of every config (N = 1), the
# config-4 all-data pattern, the runtime-matrix kernel on configs 4 and 5, and
# rank 0's config-5 shard at N = 2, 4, 8 (tools/shard_scaling.py) -- each after
# the same command has exited 0 without ncu.  tools/traffic_json.py then writes
# profiles/traffic.json keyed by kernel name and shard strip bytes.
#   usage: tools/ncu_traffic.sh TAG
set -u
TAG=${1:-traffic}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
run() { # name, command...
  local name=$1; shift
  "$@" > "$OUT/plain_$name.log" 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"pyrit_ring|ring_rt" \
    -s 3 -c 1 -o "$OUT/prof_$name" "$@" > "$OUT/ncu_$name.log" 2>&1
}
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
for c in 1 2 3 4 5; do run cfg$c $B --config $c; done
run cfg4_e0123 $B --config 4 --erased 0,1,2,3
PYRIT_B200_RT=2 run cfg4_rt $B --config 4
PYRIT_B200_RT=2 run cfg5_rt $B --config 5
for n in 2 4 8; do
  CMD="python tools/shard_scaling.py --config 5 --only $n --steps 2 --warmup 2"
  $CMD > "$OUT/plain_shard$n.log" 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"pyrit_ring|ring_rt" \
    -s 1 -c 1 -o "$OUT/prof_cfg5_shard$n" $CMD > "$OUT/ncu_shard$n.log" 2>&1
done
echo done > "$OUT/DONE"
