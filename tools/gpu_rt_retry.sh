#!/usr/bin/env bash
# Re-measure the shapes dropped earlier in the round now that the fragment loop is rolled:
# two parts per CTA, solo groups, 8 bytes per thread; plus the NUMA bind and e2e of config 5.
set -u
OUT=$PWD/gpurun_out/${1:-rt_retry}
mkdir -p "$OUT"
for r in 1 2; do
  timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 4 >> "$OUT/default.jsonl" 2>> "$OUT/err.log"
  PYRIT_B200_RT_PARTS=2 timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 4 >> "$OUT/parts2.jsonl" 2>> "$OUT/err.log"
  PYRIT_B200_RT_SOLO=1 timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 4 >> "$OUT/solo.jsonl" 2>> "$OUT/err.log"
  PYRIT_B200_RT_V=2 timeout 600 python tools/bench_rt.py --configs 2,3,4,5 --patterns 4 >> "$OUT/v2.jsonl" 2>> "$OUT/err.log"
done
python -c "
import torch, os
from paper_1709_00178_b200 import _lib as L
lib = L.load(); torch.cuda.init()
print('cpus before', len(os.sched_getaffinity(0)))
print('numa node', lib.pyrit_numa_bind_thread(0), 'cpus after', len(os.sched_getaffinity(0)))
print(open('/sys/bus/pci/devices/' + torch.cuda.get_device_properties(0).pci_bus_id.lower() + '/numa_node').read() if hasattr(torch.cuda.get_device_properties(0), 'pci_bus_id') else '')
" > "$OUT/numa.log" 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > "$OUT/bench_cfg5.jsonl" 2>> "$OUT/err.log"
echo done > "$OUT/DONE"
