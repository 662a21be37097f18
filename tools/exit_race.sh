#!/usr/bin/env bash
# a process that exits while a background (tiered) compile is
# still running must exit cleanly -- repeated N times in one lease, each with a
# fresh JIT cache so the compile really is in flight at exit.
#   usage: tools/exit_race.sh [N] > log
N=${1:-100}
ok=0; bad=0
for i in $(seq 1 "$N"); do
  d=$(mktemp -d)
  out=$(PYRIT_B200_TIERED=1 PYRIT_B200_JIT_CACHE="$d" timeout 120 python -c '
import numpy as np
import paper_1709_00178_b200 as P
code = P.CodeSpec(11, 5, P.FieldSpec.aop(12))
data = np.random.default_rng(3).integers(0, 256, (11, 12 * 4096), dtype=np.uint8)
par = P.encode_host(data, code)
print(P.Plan.last_launch()["kernel"], int(par.sum()))
' 2>&1)
  rc=$?
  if [ $rc -eq 0 ]; then ok=$((ok+1)); else bad=$((bad+1)); fi
  echo "run $i rc=$rc $out" | tail -1
  rm -rf "$d"
done
echo "SUMMARY runs=$N clean=$ok failed=$bad"
