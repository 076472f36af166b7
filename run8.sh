#!/bin/bash
mkdir -p gpurun_out
for c in c1 c2 c3; do
  ( timeout 900 python bench.py --config $c ) > gpurun_out/r02_bench_${c}_final.log 2>&1
  grep '^{"metric"' gpurun_out/r02_bench_${c}_final.log | tail -1 > gpurun_out/r02_bench_${c}_final.json
  python -c "import json; d=json.load(open('gpurun_out/r02_bench_${c}_final.json')); print('$c', d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'] if d['cpu_baseline'] else None)"
done
( timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"wgraph|wave|phi|rader|combine|split" -c 400 --csv --log-file gpurun_out/r02_c4_launches_final.csv \
   python scripts/c4_run.py --steps 1 ) > gpurun_out/s4_ncu_launches2.log 2>&1
tail -2 gpurun_out/s4_ncu_launches2.log
( timeout 1800 ncu --set full --import-source on --clock-control none -k regex:wgraph -s 11 -c 2 \
   -o gpurun_out/r02_c4_wgraph_final -f python scripts/c4_run.py --steps 1 ) > gpurun_out/s4_ncu_full2.log 2>&1
tail -2 gpurun_out/s4_ncu_full2.log
ncu -i gpurun_out/r02_c4_wgraph_final.ncu-rep --page details --csv > gpurun_out/r02_c4_wgraph_final_details.csv 2>/dev/null
ncu -i gpurun_out/r02_c4_wgraph_final.ncu-rep --page raw --csv > gpurun_out/r02_c4_wgraph_final_raw.csv 2>/dev/null
ls -la gpurun_out | grep final
