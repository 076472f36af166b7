set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpubuild.py -x -q -m gpu --durations=10 > gpurun_out/r4b_gpubuild.log 2>&1; echo "pytest gpubuild rc=$?"
tail -30 gpurun_out/r4b_gpubuild.log
for l in 256 1024 2048; do timeout 900 python scripts/gpubuild_timing.py $l 1e-12 2>&1 | tail -2; done
