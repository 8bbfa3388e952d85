#!/usr/bin/env python
"""Summarise an ncu report: key raw metrics + top stall lines (source page)."""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'launch__registers_per_thread', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'sm__warps_active.avg.per_cycle_active', 'launch__grid_size',
        'dram__bytes_read.sum.per_second', 'smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg.per_second']


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=25):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print("kernel:", v[h.index("Kernel Name")][:110])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:66s} {v[i]:>18s} {u[i]}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv"]))))
    hh, data = src[1], src[2:]
    si, sc = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
    tot = sum(int(r[si]) for r in data if r[si].isdigit()) or 1
    print(f"  stall samples: {tot}")
    for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:top]:
        print(f"  {int(r[si]) / tot * 100:5.1f}%  {r[sc].strip()[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
