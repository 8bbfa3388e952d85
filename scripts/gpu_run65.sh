# C3 with dynamic chunks: bigger tiles (more chunks to balance per CTA)
export PYTHONWARNINGS=ignore
V="U4P0B5 ARGCSR_TILE_THREADS=768 ARGCSR_TILE_THREADS=1024 ARGCSR_TILE_THREADS=2048"
CONFIGS="C3:1" VARIANTS="$V" STEPS=50 timeout 1500 bash scripts/sweep.sh > /dev/null 2>&1
cat gpurun_out/sweep.txt
