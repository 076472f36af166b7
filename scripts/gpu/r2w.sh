python scripts/phi_only.py 2048 2 2 > gpurun_out/r2y_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rader -c 2 -o gpurun_out/r2y_rader python scripts/phi_only.py 2048 2 1 > gpurun_out/r2y_ncu.log 2>&1
echo rc=$?; tail -2 gpurun_out/r2y_ncu.log
