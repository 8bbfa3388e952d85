#!/bin/bash
# ncu evidence of the final kernels (one GPU): the launch list of the default
# bench command, one `--set full` capture of the SpMV kernels of C2/C3/C4/C4f32,
# summarised ON the box (scripts/summarize_profiles.py) so that only the small
# summaries travel back (gpurun_out is capped at 64 MiB).
export PYTHONWARNINGS=ignore
TAG=${TAG:-r02b}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_C2_dcs1_compact.csv \
    python bench.py --steps 5 --warmup 3 --no-variants --no-cpu-baseline --no-configs > gpurun_out/${TAG}_launch_bench.log 2>&1
echo "launch list rc=$?"
for c in C2 C3 C4 C4f32; do
  ncu --set full --clock-control none --import-source on -k regex:spmv_ -s 6 -c 2 \
      -o gpurun_out/${TAG}_full_${c}_dcs1_compact python bench.py --config $c --steps 5 --warmup 3 \
      --no-variants --no-cpu-baseline --no-configs > gpurun_out/${TAG}_full_${c}.log 2>&1
  echo "$c rc=$?"
done
python scripts/summarize_profiles.py $TAG
for c in C2 C3; do python scripts/ncu_summary.py gpurun_out/${TAG}_full_${c}_dcs1_compact.ncu-rep 30 > gpurun_out/${TAG}_source_${c}.txt 2>&1; done
mkdir -p gpurun_out/prof_out && cp profiles/${TAG}_* profiles/ncu_traffic.json gpurun_out/prof_out/
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
