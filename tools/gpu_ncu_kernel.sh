#!/bin/bash
# ncu --set full of named kernels in one bench config (after a plain run)
#   bash tools/gpu_ncu_kernel.sh TAG CONFIG REGEX COUNT
tag=$1; c=$2; rx=$3; cnt=${4:-2}; out=gpurun_out/$tag; mkdir -p $out
python bench.py --config $c --profile --steps 1 --warmup 1 > $out/plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name regex:"$rx" -c $cnt -o $out/full \
   python bench.py --config $c --profile --steps 1 --warmup 1 > $out/ncu.log 2>&1
python tools/ncu_summary.py $out/full.ncu-rep > $out/full.md 2>&1
ls -la $out
