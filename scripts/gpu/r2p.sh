export BFLY_GRAPH_DEBUG=7
timeout 300 /usr/local/cuda/bin/cuda-gdb -batch -ex "set cuda api_failures ignore" -ex run -ex "info cuda kernels" -ex "bt 3" -ex "x/6i \$pc-32" -ex "info line *\$pc" --args python scripts/graph_bisect.py 96 4 > gpurun_out/r2p_gdb.log 2>&1
echo rc=$?
tail -40 gpurun_out/r2p_gdb.log
