set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --deselect tests/test_parity_large.py --durations=15 > gpurun_out/r2d_tests.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2d_tests.log
timeout 900 python scripts/graph_timing.py 1024 16 4096 1024 65536 1000000 > gpurun_out/r2d_graph_c3.json 2> gpurun_out/r2d_graph_c3.err; echo "timing rc=$?"
tail -1 gpurun_out/r2d_graph_c3.json; tail -5 gpurun_out/r2d_graph_c3.err
