export ARGCSR_SPMV_VARIANT=LPD4P1B4
ncu --set full --clock-control none --import-source on -k regex:spmv_ -s 4 -c 2 -o gpurun_out/lp_C2 python bench.py --config C2 --steps 5 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
export ARGCSR_SPMV_VARIANT=U4P1B4
ncu --set full --clock-control none --import-source on -k regex:spmv_ -s 4 -c 2 -o gpurun_out/lp_C3 python bench.py --config C3 --steps 5 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_C3.csv python bench.py --config C3 --steps 5 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_C4.csv python bench.py --config C4 --steps 5 --warmup 3 --no-variants --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
