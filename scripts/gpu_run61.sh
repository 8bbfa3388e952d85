export PYTHONWARNINGS=ignore
timeout 1200 python -m pytest tests/test_peer.py tests/test_gpu_parity.py -m gpu -x -q -k "peer or host_async or balance" 2>&1 | tail -3
