#!/bin/bash
mkdir -p gpurun_out
( time timeout 1800 python bench.py --steps 5 --warmup 3 ) > gpurun_out/s4_bench_c4.log 2>&1
tail -c 3000 gpurun_out/s4_bench_c4.log
( timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"wgraph|wave|phi|rader|combine|split" -c 400 --csv --log-file gpurun_out/r02_c4_launches.csv \
   python scripts/c4_run.py --steps 1 ) > gpurun_out/s4_ncu_launches.log 2>&1
tail -3 gpurun_out/s4_ncu_launches.log
( timeout 1500 ncu --set full --import-source on --clock-control none -k regex:wgraph -s 11 -c 2 \
   -o gpurun_out/r02_c4_wgraph_full -f python scripts/c4_run.py --steps 1 ) > gpurun_out/s4_ncu_full.log 2>&1
tail -3 gpurun_out/s4_ncu_full.log
ncu -i gpurun_out/r02_c4_wgraph_full.ncu-rep --page details --csv > gpurun_out/r02_c4_wgraph_details.csv 2>/dev/null
ncu -i gpurun_out/r02_c4_wgraph_full.ncu-rep --page raw --csv > gpurun_out/r02_c4_wgraph_raw.csv 2>/dev/null
ls -la gpurun_out | tail -12
