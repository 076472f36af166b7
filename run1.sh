#!/bin/bash
mkdir -p gpurun_out
export LD_PRELOAD=$PWD/scripts/segv_trace.so
( DEBUG_SAMPLE=48 timeout 900 python scripts/gpubuild_debug.py 1024 1e-12 ) > gpurun_out/s4_dbg1024.log 2>&1
grep -v "root rows" gpurun_out/s4_dbg1024.log | tail -8
( time timeout 900 python scripts/gpubuild_timing.py 2048 1e-12 ) > gpurun_out/s4_gpubuild_2048.log 2>&1
tail -8 gpurun_out/s4_gpubuild_2048.log
( time timeout 1800 python -m pytest tests -m gpu -x -q ) > gpurun_out/s4_pytest.log 2>&1
tail -8 gpurun_out/s4_pytest.log
