# r01e: ncu --set full of the final kernels with x-gather L2 hit rate, sector efficiency, fabric traffic
export PYTHONWARNINGS=ignore
mkdir -p gpurun_out/prof
TAG=r01e CONFIGS="C2:1:compact C3:1:compact C4:1:compact C1:1:compact C2:32:compact C4f32:1:compact" timeout 2400 bash scripts/profile.sh
python scripts/summarize_profiles.py r01e
cp profiles/r01e_* profiles/ncu_traffic.json gpurun_out/prof/
rm -f gpurun_out/r01e_full_*
