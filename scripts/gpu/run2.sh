set -x
timeout 600 python scripts/debug_c4_range.py 2048 0 8 > gpurun_out/r2_dbg_c4.log 2>&1; echo "dbg rc=$?"
cat gpurun_out/r2_dbg_c4.log | grep -v "^plan " | tail -30
timeout 600 python -m pytest tests/test_sht_gpu.py -x -q -k "rader or out_argument" > gpurun_out/r2_tests2.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2_tests2.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/r2_bench_c4.json; tail -20 gpurun_out/r2_bench_c4.err
