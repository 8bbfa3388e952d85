# r01g: ncu of the C3 kernels with dynamic light chunks
export PYTHONWARNINGS=ignore
mkdir -p gpurun_out/prof
TAG=r01g CONFIGS="C3:1:compact" timeout 1200 bash scripts/profile.sh
python scripts/summarize_profiles.py r01g
cp profiles/r01g_* profiles/ncu_traffic.json gpurun_out/prof/
rm -f gpurun_out/r01g_full_*
