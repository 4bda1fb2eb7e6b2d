#!/bin/bash
# Round-2 final evidence, part B (ncu; one GPU): launch lists (configs 3, 2,
# 4, 5), per-stage DRAM traffic (configs 3, 2), ncu --set full of config 3's
# three kernels and config 2's top kernels.
#   gpurun --timeout 3600 -- 'bash tools/gpu_prof_r02.sh TAG'
tag=${1:-prof}; out=gpurun_out/$tag; mkdir -p $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 3 2 4 5; do
  python bench.py --config $c --profile --steps 1 --warmup 1 > $out/plain_c$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c$c.csv \
      python bench.py --config $c --profile --steps 1 --warmup 1 > $out/ncu_launch_c$c.log 2>&1
done
for c in 3 2; do
  for st in fwd_rec fwd_blocks fwd_edge inv_rec inv_blocks inv_edge; do
    python bench.py --config $c --profile-stage $st --warmup 1 > $out/plain_tr_c${c}_$st.log 2>&1 && \
    timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $out/traffic_c${c}_$st.csv \
        python bench.py --config $c --profile-stage $st --warmup 1 > $out/traffic_c${c}_$st.log 2>&1
  done
done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:"k_half_fwd_warp|k_half_inv_umma" -c 2 -o $out/full_c3 \
    python bench.py --config 3 --profile --steps 1 --warmup 1 > $out/full_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    --kernel-name regex:"k_chirpz_fused|k_chirpz_rows|k_chirpz_cols|k_rec_inverse_ws|k_rec_forward_ws" -c 10 -o $out/full_c2 \
    python bench.py --config 2 --profile --steps 1 --warmup 1 > $out/full_c2.log 2>&1
for f in $out/*.ncu-rep; do [ $(stat -c %s $f) -gt 40000000 ] && rm -f $f; done
ls -la $out
