set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu --durations=20 --deselect tests/test_parity_large.py > gpurun_out/r4a_tests.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r4a_tests.log
timeout 1800 python bench.py --steps 5 --warmup 3 > gpurun_out/r4a_bench_c4.json 2> gpurun_out/r4a_bench_c4.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r4a_bench_c4.json; tail -5 gpurun_out/r4a_bench_c4.err
timeout 1800 python -m pytest tests/test_parity_large.py -q -m gpu --durations=30 > gpurun_out/r4a_tests_large.log 2>&1; echo "pytest large rc=$?"
tail -20 gpurun_out/r4a_tests_large.log
