set -x
for B in 2 4 16; do timeout 120 python scripts/graph_bisect.py 96 $B 2>&1 | grep -E "ok|Error" | head -3; done
timeout 900 python -m pytest tests/test_sht_gpu.py tests/test_engine_gpu.py -x -q -m gpu -k "graph or wave or planset or glrow or native_shard" > gpurun_out/r2q_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2q_tests.log
for d in 0 1; do
BFLY_GRAPH_DEBUG=$d timeout 300 python scripts/graph_timing.py 1024 16 4096 > gpurun_out/r2q_t$d.json 2>gpurun_out/r2q_t$d.err
echo "debug=$d $(tail -1 gpurun_out/r2q_t$d.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["graph_4096"]["legendre_ms"], d["graph_4096"]["pairs_per_s"])')"
done
