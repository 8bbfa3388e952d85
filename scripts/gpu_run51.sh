export PYTHONWARNINGS=ignore
timeout 1200 python -m pytest tests/test_peer.py tests/test_multigpu_device.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --config C5 --power-iteration --exchange p2p --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5 p2p N=1', d['ms_per_step'], d['value'], d['roofline']['frac'])"
