set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sht_gpu.py tests/test_engine_gpu.py -x -q -m gpu -k "graph or wave or planset or glrow" > gpurun_out/r2i_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2i_tests.log
timeout 900 python scripts/graph_timing.py 1024 16 4096 > gpurun_out/r2i_graph_c3.json 2> gpurun_out/r2i_graph_c3.err; echo "timing rc=$?"
tail -1 gpurun_out/r2i_graph_c3.json; tail -3 gpurun_out/r2i_graph_c3.err
python scripts/graph_once.py 1024 16 > gpurun_out/r2i_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wgraph -s 2 -c 2 -o gpurun_out/r2i_graph_c3 python scripts/graph_once.py 1024 16 > gpurun_out/r2i_ncu.log 2>&1
echo "ncu rc=$?"
