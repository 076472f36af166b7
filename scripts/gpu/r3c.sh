timeout 900 python -m pytest tests/test_sht_gpu.py tests/test_engine_gpu.py -x -q -m gpu -k "graph or wave or planset or glrow or native_shard or full_size" 2>&1 | tail -2
timeout 300 python scripts/graph_timing.py 1024 16 4096 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("c3", d["graph_4096"]["legendre_ms"], d["graph_4096"]["pairs_per_s"], d["graph_4096"]["round_trip"])'
for r in "0 120" "1000 1120" "3000 3120"; do timeout 300 python scripts/range_timing.py 2048 $r 16 2>/dev/null | tail -1 | cut -c1-160; done
