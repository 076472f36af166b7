timeout 300 python -m pytest tests/test_sht_gpu.py -x -q -m gpu -k "rader" 2>&1 | tail -2
timeout 300 python scripts/phi_only.py 2048 16 5
