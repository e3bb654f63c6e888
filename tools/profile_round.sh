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
ncu -i gpurun_out/$TAG/layer128k.ncu-rep --page raw --csv > gpurun_out/$TAG/ncu_raw.csv 2>&1
python tools/ncu_summary.py gpurun_out/$TAG/ncu_raw.csv > gpurun_out/$TAG/ncu_full.txt 2>&1
ls -la gpurun_out/$TAG
ncu -i gpurun_out/$TAG/layer128k.ncu-rep --page details > gpurun_out/$TAG/ncu_details.txt 2>&1
du -sh gpurun_out/$TAG/layer128k.ncu-rep
[ -n "$KEEP_REP" ] || rm -f gpurun_out/$TAG/layer128k.ncu-rep
# cfg5: one rank's share of the 8-GPU split (8 Q / 1 KV heads at 128K)
timeout 900 ncu --set full --clock-control none -c 9 \
    -k regex:"attend|gather|select|budget|score|headsum|zero" \
    -o gpurun_out/$TAG/cfg5shard python tools/profile_layer.py 131072 8 1 > gpurun_out/$TAG/cfg5.log 2>&1
ncu -i gpurun_out/$TAG/cfg5shard.ncu-rep --page raw --csv > gpurun_out/$TAG/ncu_cfg5_raw.csv 2>&1
python tools/ncu_summary.py gpurun_out/$TAG/ncu_cfg5_raw.csv > gpurun_out/$TAG/ncu_cfg5_shard.txt 2>&1
[ -n "$KEEP_REP" ] || rm -f gpurun_out/$TAG/cfg5shard.ncu-rep
