#!/bin/bash
# A/B of one build under two environment settings in alternating processes:
#   bash tools/ab_env.sh "VAR=a" "VAR=b" [rounds] [extra bench args]
A=$1; B=$2; N=${3:-3}; shift 3; EXTRA="$@"
for i in $(seq $N); do
  for e in "$A" "$B"; do
    env $e timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --extra "" --sweep "" $EXTRA 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$e', d['value'], 'eager', d['eager_ms'], 'dense', d['dense_ms'], 'x%.3f'%d['speedup_vs_dense'], 'clk', d['clocks']['sm_mhz'], {k: round(v,3) for k,v in d['stages_ms'].items() if v > 0.01})"
  done
done
