set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sht_gpu.py -x -q -k "graph_program or wave_programs" > gpurun_out/r2c_tests_graph.log 2>&1; echo "pytest graph rc=$?"
tail -30 gpurun_out/r2c_tests_graph.log
timeout 900 python scripts/graph_timing.py 1024 16 4096 1024 16384 > gpurun_out/r2c_graph_c3.json 2> gpurun_out/r2c_graph_c3.err; echo "timing rc=$?"
tail -3 gpurun_out/r2c_graph_c3.json; tail -5 gpurun_out/r2c_graph_c3.err
