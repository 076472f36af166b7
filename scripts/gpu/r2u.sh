set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --deselect tests/test_parity_large.py > gpurun_out/r2u_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2u_tests.log
timeout 300 python scripts/fft_probe.py 32768 > gpurun_out/r2u_fft.json 2>&1; cat gpurun_out/r2u_fft.json
timeout 600 python bench.py --mode sharded --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_shard_c3.json 2> gpurun_out/r2u_shard_c3.err; echo "shard bench rc=$?"
tail -c 2500 gpurun_out/r2u_shard_c3.json; tail -3 gpurun_out/r2u_shard_c3.err
