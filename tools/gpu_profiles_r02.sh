#!/bin/bash
# Round-2 evidence for profiles/: launch lists (configs 3, 2, 4, 5) and
# ncu --set full captures of the top kernels of configs 3 and 2.
#   gpurun --timeout 3000 -- 'bash tools/gpu_profiles_r02.sh TAG'
tag=${1:-r02}
out=gpurun_out/prof_$tag
mkdir -p $out
for c in 3 2 4 5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c$c.csv \
      python bench.py --config $c --profile --steps 1 --warmup 1 > $out/ncu_launch_c$c.log 2>&1
  python tools/ncu_summary.py --launches $out/launches_c$c.csv > $out/launches_c$c.md 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -c 8 -o $out/full_c3 \
    python bench.py --config 3 --profile --steps 1 --warmup 1 > $out/full_c3.log 2>&1
python tools/ncu_summary.py $out/full_c3.ncu-rep > $out/full_c3.md 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    --kernel-name regex:"k_chirpz_fused|k_chirpz_rows|k_rec_gemm|k_chirpz_cols|k_rec_inverse_ws|k_rec_forward_ws" -c 12 -o $out/full_c2 \
    python bench.py --config 2 --profile --steps 1 --warmup 1 > $out/full_c2.log 2>&1
python tools/ncu_summary.py $out/full_c2.ncu-rep > $out/full_c2.md 2>&1
for f in $out/*.ncu-rep; do [ $(stat -c %s $f) -gt 30000000 ] && rm -f $f; done
ls -la $out
