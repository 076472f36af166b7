set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json; cat gpurun_out/fp64_peak.json
timeout 900 python -m pytest tests -x -q -m gpu --durations=30 --deselect tests/test_parity_large.py > gpurun_out/r2_tests_base.log 2>&1; echo "pytest base rc=$?"
tail -45 gpurun_out/r2_tests_base.log
timeout 2400 python -m pytest tests/test_parity_large.py -q -m gpu --durations=30 > gpurun_out/r2_tests_large.log 2>&1; echo "pytest large rc=$?"
tail -60 gpurun_out/r2_tests_large.log
