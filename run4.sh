#!/bin/bash
mkdir -p gpurun_out
( time timeout 3300 python scripts/c5_streamed.py --oracle --out gpurun_out/r02_c5_streamed.json ) > gpurun_out/s4_c5.log 2>&1
tail -c 2500 gpurun_out/s4_c5.log
