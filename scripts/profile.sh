#!/bin/bash
# ncu evidence for the bench configurations (run under gpurun, one GPU):
#   launch lists (gpu__time_duration per kernel, cold-cache, serialised) and one
#   `--set full` capture of each SpMV kernel per config.  Summarise here with
#   scripts/summarize_profiles.py.
export PYTHONWARNINGS=ignore
TAG=${TAG:-r01}
for cfg in ${CONFIGS:-C2:1 C2:32 C3:1 C4:1 C1:1}; do
  c=${cfg%%:*}; d=${cfg##*:}
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_${c}_dcs${d}.csv \
      python bench.py --config $c --dcs $d --steps 5 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:spmv_ -s 6 -c 2 \
      -o gpurun_out/${TAG}_full_${c}_dcs${d} python bench.py --config $c --dcs $d --steps 5 --warmup 3 \
      --no-variants --no-cpu-baseline > /dev/null 2>&1
  echo "$c dcs=$d done"
done
