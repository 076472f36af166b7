#!/bin/bash
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/s4_pytest3.log 2>&1
tail -4 gpurun_out/s4_pytest3.log
( timeout 300 python __graft_entry__.py smoke ) > gpurun_out/s4_smoke.log 2>&1; tail -2 gpurun_out/s4_smoke.log
( time timeout 1800 python bench.py --impl reference --steps 3 --warmup 3 ) > gpurun_out/s4_bench_ref.log 2>&1
tail -c 700 gpurun_out/s4_bench_ref.log
( time timeout 1800 python bench.py ) > gpurun_out/s4_bench_c4c.log 2>&1
tail -c 1500 gpurun_out/s4_bench_c4c.log
