#!/usr/bin/env python
"""One-launch ncu summary (CSV lines) from a .ncu-rep: DRAM bytes, time, occupancy, pipes.

    python tools/ncu_summary.py gpurun_out/x/prof.ncu-rep "comment line" ... > profiles/...csv
"""
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]

rep = sys.argv[1]
for c in sys.argv[2:]:
    print("# " + c)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    for i, h in enumerate(hdr):
        if h in KEYS:
            print(f"{h},{r[i]},{units[i]}")
