#!/bin/bash
# Round-2 evidence refresh after the row-CTA change: launch lists of configs 2
# and 4, ncu --set full of config 2's top kernels.
#   gpurun --timeout 2400 -- 'bash tools/gpu_prof_r02b.sh TAG'
tag=${1:-prof}; out=gpurun_out/$tag; mkdir -p $out
for c in 2 4; do
  python bench.py --config $c --profile --steps 1 --warmup 1 > $out/plain_c$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c$c.csv \
      python bench.py --config $c --profile --steps 1 --warmup 1 > $out/ncu_launch_c$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none \
    --kernel-name regex:"k_chirpz_fused|k_chirpz_rows|k_chirpz_cols|k_rec_inverse_ws|k_rec_forward_ws" -c 10 -o $out/full_c2 \
    python bench.py --config 2 --profile --steps 1 --warmup 1 > $out/full_c2.log 2>&1
ls -la $out
