set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_large.py -q -m gpu --durations=30 > gpurun_out/r2b_tests_large.log 2>&1; echo "pytest large rc=$?"
grep -E "AssertionError: \{|passed|failed" gpurun_out/r2b_tests_large.log | tail -20
timeout 1800 python bench.py --steps 5 --warmup 3 > gpurun_out/r2b_bench_c4.json 2> gpurun_out/r2b_bench_c4.err; echo "bench rc=$?"
tail -c 5000 gpurun_out/r2b_bench_c4.json; tail -20 gpurun_out/r2b_bench_c4.err
