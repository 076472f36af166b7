for v in "" var_w8; do
  if [ -n "$v" ]; then export BFLY_LIB=$PWD/paper_0910_5435_b200/$v/libbfly_b200.so; else unset BFLY_LIB; fi
  echo "== ${v:-w4}"
  for r in "0 120" "1000 1120" "2000 2120" "3000 3120" "3900 4020"; do timeout 300 python scripts/range_timing.py 2048 $r 16 2>/dev/null | tail -1 | cut -c1-200; done
done
