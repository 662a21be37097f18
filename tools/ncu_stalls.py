"""Print duration, issue activity and the top warp-stall reasons of an ncu --page raw --csv dump."""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
hdr, units = r[0], r[1]
want = ['gpu__time_duration.sum', 'smsp__cycles_active.avg', 'smsp__inst_executed.sum', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__warps_eligible.avg.per_cycle_active', 'launch__registers_per_thread', 'launch__grid_size',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
for vals in r[2:]:
    print('--', vals[hdr.index('Kernel Name')][:90] if 'Kernel Name' in hdr else '')
    for i, h in enumerate(hdr):
        if h in want:
            print(' ', h, units[i], vals[i])
    st = []
    for i, h in enumerate(hdr):
        if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio'):
            try:
                st.append((float(vals[i].replace(',', '')), h))
            except ValueError:
                pass
    for v, h in sorted(st, reverse=True)[:10]:
        print('  %.3f %s' % (v, h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
