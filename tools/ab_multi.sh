#!/bin/bash
# A/B/... of several builds in alternating processes: bash tools/ab_multi.sh N dir1 dir2 ...
N=$1; shift
for i in $(seq $N); do
  for d in "$@"; do
    (cd $d && timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --extra "" --sweep "" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['value'], 'dense', d['dense_ms'], 'x%.3f'%d['speedup_vs_dense'], 'clk', d['clocks']['sm_mhz'], 'attend', round(d['stages_ms']['attend'],3))")
  done
done
