set -x
mkdir -p gpurun_out
timeout 1800 python bench.py --steps 5 --warmup 3 > gpurun_out/r3a_bench_c4.json 2> gpurun_out/r3a_bench_c4.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r3a_bench_c4.json; tail -5 gpurun_out/r3a_bench_c4.err
