#!/bin/bash
# config 5 launch list with the final code (long: ~32k kernels under ncu)
tag=${1:-prof}; out=gpurun_out/$tag; mkdir -p $out
python bench.py --config 5 --profile --steps 1 --warmup 1 > $out/plain_c5.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c5.csv \
    python bench.py --config 5 --profile --steps 1 --warmup 1 > $out/ncu_launch_c5.log 2>&1
ls -la $out
