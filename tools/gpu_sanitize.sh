#!/usr/bin/env bash
# compute-sanitizer over the allocation-exact kernel driver (tests/sanitize_check.cpp):
# a plain run first, then memcheck, racecheck, synccheck and initcheck, each bounded.
set -u
OUT=gpurun_out/${1:-san}
mkdir -p "$OUT"
timeout 300 build/sanitize_check > "$OUT/plain.log" 2>&1
echo "plain exit $?" >> "$OUT/plain.log"
if grep -q "SANITIZE CHECK PASSED" "$OUT/plain.log"; then
  for t in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $t --error-exitcode 3 build/sanitize_check > "$OUT/$t.log" 2>&1
    echo "$t exit $?" >> "$OUT/$t.log"
  done
fi
echo done > "$OUT/DONE"
