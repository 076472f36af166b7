set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sht_gpu.py tests/test_engine_gpu.py -x -q -m gpu -k "graph or wave or planset or glrow" > gpurun_out/r2e_tests.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2e_tests.log
timeout 900 python scripts/graph_timing.py 1024 16 4096 1000000 > gpurun_out/r2e_graph_c3.json 2> gpurun_out/r2e_graph_c3.err; echo "timing rc=$?"
tail -1 gpurun_out/r2e_graph_c3.json; tail -5 gpurun_out/r2e_graph_c3.err
