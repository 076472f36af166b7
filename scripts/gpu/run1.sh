set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json; cat gpurun_out/fp64_peak.json
timeout 1500 python -m pytest tests -x -q -m gpu --durations=30 > gpurun_out/r2_tests1.log 2>&1; echo "pytest rc=$?"
tail -45 gpurun_out/r2_tests1.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench_c4.json; tail -20 gpurun_out/r2_bench_c4.err
