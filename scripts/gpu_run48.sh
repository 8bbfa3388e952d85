export PYTHONWARNINGS=ignore
timeout 900 python -m pytest tests/test_peer.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --config C2 --power-iteration --exchange p2p --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 PI p2p N=1', d['ms_per_step'], d['value'], d['roofline']['frac'])"
