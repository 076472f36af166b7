set -x
mkdir -p gpurun_out
for d in 0 1 2 4 8 3 6 14 15; do
  BFLY_GRAPH_DEBUG=$d timeout 300 python scripts/graph_timing.py 1024 16 4096 > gpurun_out/r2j_dbg$d.json 2>/dev/null
  echo "debug=$d $(tail -1 gpurun_out/r2j_dbg$d.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["graph_4096"]["legendre_ms"])')"
done
