#!/usr/bin/env python
"""profiles/traffic.json from the ncu reports of tools/ncu_traffic.sh, keyed by KERNEL NAME and
shard strip bytes, so bench.py's roofline.traffic is only ever the traffic of the kernel it ran.

    python tools/traffic_json.py gpurun_out/TAG [profiles/traffic.json]

Per entry: dram__bytes_read.sum + dram__bytes_write.sum of one launch (ncu --set full, cold
cache, serialised), its duration, and the report it came from.  The strip bytes come from the
plain (non-ncu) run's JSON line (bench.py config.shard_strip_bytes) or shard_scaling's output.
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for i, h in enumerate(hdr):
        d[h] = (vals[i], units[i])
    return d


def num(d, k):
    v, u = d[k]
    return float(v.replace(",", "")) * UNIT.get(u, 1)


def strip_of(plain_log):
    for ln in open(plain_log):
        if ln.startswith("{"):
            j = json.loads(ln)
            if "config" in j:
                return j["config"].get("shard_strip_bytes")
            if "shard_strip_bytes" in j:
                return j["shard_strip_bytes"]
    return None


def main():
    src = sys.argv[1]
    dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json"
    out = {"_source": f"tools/ncu_traffic.sh -> {src} -> tools/traffic_json.py: dram__bytes_read.sum + "
                      "dram__bytes_write.sum of one launch (ncu --set full, --clock-control none), keyed "
                      "'<kernel>|<shard strip bytes>'", "kernels": {}}
    for f in sorted(os.listdir(src)):
        if not (f.startswith("prof_") and f.endswith(".ncu-rep")):
            continue
        name = f[len("prof_"):-len(".ncu-rep")]
        d = raw(os.path.join(src, f))
        kern = d["Kernel Name"][0]
        plain = os.path.join(src, "plain_" + name.replace("cfg5_shard", "shard") + ".log")
        strip = strip_of(plain) if os.path.exists(plain) else None
        b = num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")
        tv, tu = d["gpu__time_duration.sum"]
        us = float(tv.replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
                                           "msecond": 1e3}.get(tu, 1)
        out["kernels"][f"{kern}|{strip}"] = {"traffic_bytes": int(b), "ncu_us": us, "capture": name,
                                             "report": os.path.join(src, f)}
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
