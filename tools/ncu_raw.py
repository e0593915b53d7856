#!/usr/bin/env python
"""Selected metrics per kernel from `ncu -i rep --page raw --csv` output.

  ncu -i x.ncu-rep --page raw --csv > raw.csv ; python tools/ncu_raw.py raw.csv"""
import csv
import sys

WANT = ['Kernel Name', 'launch__grid_size', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'smsp__inst_executed.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = [hdr.index(w) if w in hdr else -1 for w in WANT]
    seen = set()
    for d in data:
        k = (d[idx[0]][:60], d[idx[1]])
        if k in seen:
            continue
        seen.add(k)
        print('---')
        for w, i in zip(WANT, idx):
            if i >= 0:
                print(f'  {w}: {d[i]} {units[i]}')


if __name__ == '__main__':
    main()
