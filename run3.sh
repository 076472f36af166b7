#!/bin/bash
mkdir -p gpurun_out
R=gpurun_out/s4_exp3.log; : > $R
for g in 4096 65536 1000000; do
  echo "== c3 group $g" >> $R
  ( BFLY_GRAPH_GROUP=$g timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline ) 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['legendre_ms_per_direction'], d['roofline']['frac'], d['plan']['build_s'])" >> $R 2>&1
done
for g in 4096 65536; do
  echo "== l2048 [2000,2160) group $g" >> $R
  ( BFLY_GRAPH_GROUP=$g timeout 600 python scripts/range_timing.py 2048 2000 2160 16 ) >> $R 2>&1
done
cat $R
