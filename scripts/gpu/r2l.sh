set -x
mkdir -p gpurun_out
BFLY_GRAPH_PROFILE=1 timeout 300 python scripts/graph_once.py 1024 16 > gpurun_out/r2l_prof.log 2>&1; echo rc=$?
grep "graph profile" gpurun_out/r2l_prof.log | tail -4
BFLY_GRAPH_DEBUG=1 BFLY_GRAPH_PROFILE=1 timeout 300 python scripts/graph_once.py 1024 16 > gpurun_out/r2l_prof1.log 2>&1; echo rc=$?
grep "graph profile" gpurun_out/r2l_prof1.log | tail -4
