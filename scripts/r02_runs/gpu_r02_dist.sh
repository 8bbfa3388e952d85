#!/bin/bash
# Distributed code path on one GPU (the scaling run's path): BENCH_DIST at N=1 (all-gather / halo / p2p exchange), torchrun launch, power iteration
mkdir -p gpurun_out; out=gpurun_out/r02_dist.jsonl; : > $out
for ex in auto halo p2p; do
  ARGCSR_BENCH_DIST=1 timeout 600 python bench.py --steps 20 --warmup 3 --no-variants --no-configs --no-cpu-baseline --exchange $ex >> $out 2> gpurun_out/r02_dist_$ex.err; echo "dist $ex rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 --no-variants --no-configs --no-cpu-baseline >> $out 2> gpurun_out/r02_dist_torchrun.err; echo "torchrun rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 20 --warmup 3 --power-iteration --no-cpu-baseline >> $out 2> gpurun_out/r02_dist_pi.err; echo "torchrun pi rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/r02_dist.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), d.get("config", {}).get("exchange") or d.get("config"))
PY
