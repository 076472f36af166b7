#!/bin/bash
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/s4_pytest4.log 2>&1
tail -4 gpurun_out/s4_pytest4.log
( BFLY_GRAPH_WAVEFRONT=1 BFLY_GRAPH_GROUP=64 timeout 1200 python -m pytest tests/test_sht_gpu.py tests/test_engine_gpu.py tests/test_parity_large.py -x -q -m gpu -k "wave or graph or plan or range or shard or streamed or c3_own" ) > gpurun_out/s4_pytest_wf.log 2>&1
tail -3 gpurun_out/s4_pytest_wf.log
( timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline ) 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', d['value'], d['roofline']['legendre_ms_per_direction'], d['roofline']['frac'])"
( BFLY_GRAPH_WAVEFRONT=1 BFLY_GRAPH_GROUP=2048 timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline ) 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 wavefront 2048', d['value'], d['roofline']['legendre_ms_per_direction'], d['roofline']['frac'])"
( timeout 900 python bench.py --impl reference --steps 5 --warmup 3 ) 2>/dev/null | tail -1 | cut -c1-200
