set -x
mkdir -p gpurun_out
python scripts/graph_once.py 1024 16 > gpurun_out/r2f_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wgraph -s 2 -c 2 -o gpurun_out/r2f_graph_c3 python scripts/graph_once.py 1024 16 > gpurun_out/r2f_ncu.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/r2f_plain.log; tail -5 gpurun_out/r2f_ncu.log
