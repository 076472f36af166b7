set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sht_gpu.py tests/test_engine_gpu.py -x -q -m gpu -k "graph or wave or planset or glrow" > gpurun_out/r2n_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2n_tests.log
for d in 0 1; do
BFLY_GRAPH_DEBUG=$d timeout 300 python scripts/graph_timing.py 1024 16 4096 > gpurun_out/r2n_t$d.json 2>gpurun_out/r2n_t$d.err
echo "debug=$d $(tail -1 gpurun_out/r2n_t$d.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["graph_4096"]["legendre_ms"], d["graph_4096"]["pairs_per_s"])')"
done
