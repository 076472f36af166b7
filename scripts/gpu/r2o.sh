for d in 0 1 2 4 5 7; do echo "== debug $d"; BFLY_GRAPH_DEBUG=$d CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/graph_bisect.py 96 3 2>&1 | grep -E "ok|Error|error" | head -3; done
for B in 1 2 4 8 16; do echo "== B $B"; CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/graph_bisect.py 96 $B 2>&1 | grep -E "ok|Error|error" | head -3; done
