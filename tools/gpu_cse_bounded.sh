#!/usr/bin/env bash
# The paper's (60,40) GF(2^6) embedding code: pair sharing bounded by a cap on the
# temporaries per fragment group (PYRIT_B200_PART_TEMPS), over group sizes and parts.
set -u
OUT=$PWD/gpurun_out/${1:-cse_bounded}
mkdir -p "$OUT"
V=""
for g in 25 8 4 2; do
  V="$V;PART_GROUP=$g,PART_CSE=0"
  for t in 4 8 16 32 64; do
    V="$V;PART_GROUP=$g,PART_CSE=1,PART_TEMPS=$t"
  done
done
V=${V#;}
timeout 1500 python tools/tune.py --code 40,20,gf64 --frag 9600000 --rounds 2 --variants ";$V" > "$OUT/k40r20_parts2.jsonl" 2> "$OUT/err1.log"
V=""
for g in 8 4; do
  for t in 0 8 16 32; do
    c=1; [ $t = 0 ] && c=0
    V="$V;PARTS=4,THREADS=512,PART_GROUP=$g,PART_CSE=$c,PART_TEMPS=$t"
  done
done
V=${V#;}
timeout 1500 python tools/tune.py --code 40,20,gf64 --frag 9600000 --rounds 2 --variants ";$V" > "$OUT/k40r20_parts4.jsonl" 2> "$OUT/err2.log"
echo done > "$OUT/DONE"
