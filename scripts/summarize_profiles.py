#!/usr/bin/env python
"""Turn gpurun_out/<tag>_* ncu outputs into committed summaries under profiles/:

  profiles/<tag>_ncu_<cfg>.txt   key metrics + stall breakdown of each SpMV kernel
  profiles/<tag>_launches_<cfg>.csv   the launch list (kernel name, duration)
  profiles/ncu_traffic.json      dram read+write bytes per SpMV (all SpMV kernels of
                                 one step) keyed like bench.py's roofline lookup
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "sm__warps_active.avg.per_cycle_active", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
        "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
        "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio",
        "lts__t_sectors_evict_last_lookup_hit.sum", "lts__t_sectors_evict_last_lookup_miss.sum",
        "lts__t_sectors_srcunit_ltcfabric.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def to_bytes(val, unit):
    v = float(val)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def summarize(rep: Path):
    rows = list(csv.reader(io.StringIO(ncu([str(rep), "--page", "raw", "--csv"]))))
    h, u = rows[0], rows[1]
    lines, traffic = [], 0.0
    seen = set()
    for v in rows[2:]:
        name = v[h.index("Kernel Name")]
        kern = name.split("(")[0].split("::")[-1]
        if kern in seen:  # -c 2 captures one launch of each kernel of a step (heavy + light)
            continue
        seen.add(kern)
        lines.append(f"kernel: {name[:140]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"  {k:66s} {v[i]:>18s} {u[i]}")
        try:  # x gathers are the only L2 evict_last loads: their L2 hit rate
            xh = float(v[h.index("lts__t_sectors_evict_last_lookup_hit.sum")].replace(",", ""))
            xm = float(v[h.index("lts__t_sectors_evict_last_lookup_miss.sum")].replace(",", ""))
            if xh + xm > 0:
                lines.append(f"  {'x gathers: L2 hit rate (evict_last sectors)':66s} {100 * xh / (xh + xm):>18.2f} %")
        except (ValueError, IndexError):
            pass
        rb = to_bytes(v[h.index("dram__bytes_read.sum")], u[h.index("dram__bytes_read.sum")])
        wb = to_bytes(v[h.index("dram__bytes_write.sum")], u[h.index("dram__bytes_write.sum")])
        traffic += rb + wb
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v[i]), k.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        lines.append("  stalls (warps per issue): " + ", ".join(f"{n}={x:.2f}" for x, n in sorted(stalls)[::-1][:6]))
    return lines, traffic


def main(tag):
    PROF.mkdir(exist_ok=True)
    tfile = PROF / "ncu_traffic.json"
    traffic = json.loads(tfile.read_text()) if tfile.exists() else {}
    for rep in sorted(OUT.glob(f"{tag}_full_*.ncu-rep")):
        cfg = rep.stem[len(f"{tag}_full_"):]
        lines, t = summarize(rep)
        (PROF / f"{tag}_ncu_{cfg}.txt").write_text("\n".join(lines) + "\n")
        c, d = cfg.split("_dcs")
        d, _, layout = d.partition("_")
        traffic[f"{c}_tpg128_dcs{d}_{layout or 'reference'}"] = int(t)
        print(cfg, f"traffic/step = {t / 1e9:.3f} GB")
    for f in sorted(OUT.glob(f"{tag}_launches_*.csv")):
        rows = [r for r in csv.reader(open(f)) if r and r[0].isdigit()]
        keep = [["kernel", "duration_ns"]] + [[r[4][:120], r[-1]] for r in rows]
        with open(PROF / f.name, "w", newline="") as fh:
            csv.writer(fh).writerows(keep)
    tfile.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
