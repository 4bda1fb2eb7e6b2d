out=gpurun_out/r01s5; mkdir -p $out
timeout 1500 ncu --set full --clock-control none --import-source on \
    --kernel-name regex:"k_rec_inverse_ws|k_rec_forward_ws|k_chirpz_rows|k_chirpz_cols_fwd" -c 5 -o $out/full_c4 \
    python bench.py --config 4 --profile --steps 1 --warmup 1 > $out/ncu_full_c4.log 2>&1
ncu -i $out/full_c4.ncu-rep --page raw --csv > $out/full_c4_raw.csv 2>/dev/null
python tools/ncu_summary.py $out/full_c4.ncu-rep > $out/full_c4.md 2>&1
ls -la $out
