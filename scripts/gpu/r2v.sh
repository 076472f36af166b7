set -x
timeout 300 python -m pytest tests/test_sht_gpu.py -x -q -m gpu -k "rader or native_shard" 2>&1 | tail -2
for v in "" var_rold; do
  if [ -n "$v" ]; then export BFLY_LIB=$PWD/paper_0910_5435_b200/$v/libbfly_b200.so; else unset BFLY_LIB; fi
  echo "== ${v:-new}"; timeout 300 python scripts/phi_only.py 2048 16 5; timeout 300 python scripts/phi_only.py 1024 16 5; timeout 120 python scripts/phi_only.py 256 1 20
done
