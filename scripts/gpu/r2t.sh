for v in "" var_c4 var_w8; do
  if [ -n "$v" ]; then export BFLY_LIB=$PWD/paper_0910_5435_b200/$v/libbfly_b200.so; else unset BFLY_LIB; fi
  echo "== variant ${v:-default}"
  timeout 300 python scripts/graph_timing.py 1024 16 4096 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("c3", d["graph_4096"]["legendre_ms"], d["graph_4096"]["pairs_per_s"], d["graph_4096"]["round_trip"])'
  timeout 300 python scripts/range_timing.py 2048 0 160 16 2>/dev/null | tail -1
  timeout 300 python scripts/range_timing.py 2048 2000 2160 16 2>/dev/null | tail -1
done
