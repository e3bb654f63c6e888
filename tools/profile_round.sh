#!/bin/bash
# One GPU session's measurement pass: bench line, ncu launch list, ncu full set.
# usage (under gpurun): bash tools/profile_round.sh <tag>
set -x
TAG=${1:-r1}
mkdir -p gpurun_out/$TAG
timeout 900 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/$TAG/launches.csv python bench.py --steps 1 --warmup 1 --sweep "" \
    --no-e2e --no-cpu-baseline --no-dense --extra "" > gpurun_out/$TAG/launches_bench.log 2>&1
python tools/launches.py gpurun_out/$TAG/launches.csv > gpurun_out/$TAG/launches.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -c 9 \
    -k regex:"attend|gather|select|budget|score|headsum|zero" \
    -o gpurun_out/$TAG/layer128k python tools/profile_layer.py > gpurun_out/$TAG/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/$TAG/layer128k.ncu-rep gpurun_out/$TAG/ncu_full.json \
    > gpurun_out/$TAG/ncu_full.txt 2>&1
ls -la gpurun_out/$TAG
ncu -i gpurun_out/$TAG/layer128k.ncu-rep --page details > gpurun_out/$TAG/ncu_details.txt 2>&1
du -sh gpurun_out/$TAG/layer128k.ncu-rep
[ -n "$KEEP_REP" ] || rm -f gpurun_out/$TAG/layer128k.ncu-rep
