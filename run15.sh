#!/bin/bash
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/s4_pytest5.log 2>&1
tail -4 gpurun_out/s4_pytest5.log
( timeout 300 python __graft_entry__.py smoke ) > gpurun_out/s4_smoke2.log 2>&1; tail -1 gpurun_out/s4_smoke2.log
( time timeout 1800 python bench.py --impl reference ) > gpurun_out/s4_bench_ref2.log 2>&1
tail -1 gpurun_out/s4_bench_ref2.log | cut -c1-300; grep "^real" gpurun_out/s4_bench_ref2.log
( time timeout 1800 python bench.py ) > gpurun_out/s4_bench_c4d.log 2>&1
tail -c 1200 gpurun_out/s4_bench_c4d.log
