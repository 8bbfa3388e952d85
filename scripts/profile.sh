#!/bin/bash
# ncu evidence for the bench configurations (run under gpurun, one GPU):
#   launch lists (gpu__time_duration per kernel, cold-cache, serialised) and one
#   `--set full` capture of each SpMV kernel per config.  Summarise here with
#   scripts/summarize_profiles.py <TAG>.
#   CONFIGS entries: <config>:<dcs>:<layout>
export PYTHONWARNINGS=ignore
TAG=${TAG:-r01}
for cfg in ${CONFIGS:-C2:1:compact C2:32:compact C3:1:compact C4:1:compact C1:1:compact}; do
  IFS=: read c d l <<< "$cfg"
  name=${c}_dcs${d}_${l}
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_${name}.csv \
      python bench.py --config $c --dcs $d --layout $l --steps 5 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:spmv_ -s 6 -c 2 \
      -o gpurun_out/${TAG}_full_${name} python bench.py --config $c --dcs $d --layout $l --steps 5 --warmup 3 \
      --no-variants --no-cpu-baseline > /dev/null 2>&1
  echo "$name done"
done
