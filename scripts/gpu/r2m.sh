set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sht_gpu.py tests/test_engine_gpu.py -x -q -m gpu -k "graph or wave or planset or glrow" > gpurun_out/r2m_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2m_tests.log
BFLY_GRAPH_PROFILE=1 timeout 300 python scripts/graph_once.py 1024 16 > gpurun_out/r2m_prof.log 2>&1; echo rc=$?
grep "graph profile" gpurun_out/r2m_prof.log | tail -2
timeout 300 python scripts/graph_timing.py 1024 16 4096 > gpurun_out/r2m_t.json 2>gpurun_out/r2m_t.err
tail -1 gpurun_out/r2m_t.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["graph_4096"]["legendre_ms"], d["graph_4096"]["pairs_per_s"])'
