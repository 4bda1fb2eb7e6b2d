#!/bin/bash
# usage: tools/launch_list.sh CONFIG TAG  -> gpurun_out/launches_<TAG>.csv (+ .md summary printed)
set -e
c=$1; tag=$2
mkdir -p gpurun_out
python bench.py --config $c --profile --steps 1 > gpurun_out/prof_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --config $c --profile --steps 1 > gpurun_out/ncu_$tag.log 2>&1
python tools/ncu_summary.py --launches gpurun_out/launches_$tag.csv > gpurun_out/launches_$tag.md
