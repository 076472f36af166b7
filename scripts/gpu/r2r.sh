for B in 17 4; do echo "== B $B"; timeout 120 python scripts/graph_debug_members.py 200 $B 2>&1 | tail -3; done
timeout 900 python -m pytest tests/test_sht_gpu.py tests/test_engine_gpu.py -x -q -m gpu -k "graph or wave or planset or glrow or native_shard or full_size" > gpurun_out/r2r_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2r_tests.log
timeout 300 python scripts/graph_timing.py 1024 16 4096 > gpurun_out/r2r_t.json 2>gpurun_out/r2r_t.err
tail -1 gpurun_out/r2r_t.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["graph_4096"]["legendre_ms"], d["graph_4096"]["pairs_per_s"], d["graph_4096"]["round_trip"])'
