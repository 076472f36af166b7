#!/bin/bash
mkdir -p gpurun_out
R=gpurun_out/s4_exp8.log; : > $R
( timeout 1200 python -m pytest tests/test_sht_gpu.py tests/test_engine_gpu.py -x -q -m gpu -k "wave or graph or plan or range or shard or streamed" ) >> $R 2>&1
echo "== c3 default" >> $R
( timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline ) 2>>$R | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['legendre_ms_per_direction'], d['roofline']['frac'], d['plan']['build_s'], d['round_trip_rel_l2'])" >> $R 2>&1
for rng in "0 160" "2000 2160"; do
  echo "== default l2048 [$rng)" >> $R
  ( timeout 600 python scripts/range_timing.py 2048 $rng 16 ) 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms'], d['tflops'])" >> $R 2>&1
done
for g in 8192 16384 32768 65536; do
  echo "== group $g l2048 [0 1024)" >> $R
  ( BFLY_GRAPH_GROUP=$g timeout 900 python scripts/range_timing.py 2048 0 1024 16 ) 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms'], d['tflops'])" >> $R 2>&1
done
grep -v "device_step_ms" $R | tail -20
