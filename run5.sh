#!/bin/bash
mkdir -p gpurun_out
R=gpurun_out/s4_exp5.log; : > $R
for v in default b8r64 b8r64s3 b8r128c3; do
  lib=""; [ $v != default ] && lib=$PWD/paper_0910_5435_b200/var_$v/libbfly_b200.so
  for rng in "0 160" "2000 2160" "3500 4096"; do
    echo "== $v l2048 [$rng)" >> $R
    ( BFLY_LIB=$lib timeout 600 python scripts/range_timing.py 2048 $rng 16 ) 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms'], d['tflops'])" >> $R 2>&1
  done
done
cat $R
