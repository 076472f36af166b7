#!/bin/bash
mkdir -p gpurun_out
R=gpurun_out/s4_exp10.log; : > $R
( timeout 900 python -m pytest tests/test_gpubuild.py -x -q -m gpu ) >> $R 2>&1
( DEBUG_SAMPLE=64 timeout 900 python scripts/gpubuild_debug.py 256 1e-12 --twice ) 2>&1 | grep -v "root rows" | tail -4 >> $R
( DEBUG_SAMPLE=48 timeout 900 python scripts/gpubuild_debug.py 1024 1e-12 ) 2>&1 | grep -v "root rows" | tail -3 >> $R
( BFLY_BUILD_VERBOSE=1 timeout 900 python scripts/gpubuild_timing.py 2048 1e-12 ) >> $R 2>&1
( BFLY_BUILD_VERBOSE=1 timeout 900 python -c "
import time, paper_0910_5435_b200 as bb
t=time.time(); s=bb.SHT(2048, eps=1e-12); print('sht create', time.time()-t)
" ) >> $R 2>&1
cat $R | tail -24
