#!/usr/bin/env python
"""One summary line per bench.py JSON line: python tools/summarize_bench.py profiles/r01_s3/bench_*.jsonl"""
import json,sys
for fn in sys.argv[1:]:
    for line in open(fn):
        if not line.startswith('{'): continue
        d=json.loads(line)
        if 'roofline' not in d: print(fn, line[:200]); continue
        print(fn.split('/')[-1], d['config']['workload'][:28], d['config'].get('kernel','')[-40:], 'src %.0f'%d['value'], 'ms %.3f'%d['ms_per_step'], 'moved %.0f frac %.3f'%(d['roofline']['achieved'], d['roofline']['frac']), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), 'ver', d.get('verified'), 'e2e', d['e2e'] and round(d['e2e']['value'],1))
