#!/bin/bash
# One GPU session: parity tests, smoke, bench lines for every config, the
# reference arm, the config-2 launch list and an ncu --set full capture of
# the top kernels (kept under gpurun's 64 MiB return limit).
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG [CONFIGS]'
tag=${1:-r01}
configs=${2:-"2 1 3 4 5"}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
for c in $configs; do
  timeout 900 python bench.py --config $c > $out/bench_c$c.json 2> $out/bench_c$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref_c2.json 2> $out/bench_ref_c2.err
# launch list (cold cache, serialised) then a full capture of the top kernels of one step
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c2.csv \
    python bench.py --config 2 --profile --steps 1 --warmup 1 > $out/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
    --kernel-name regex:"k_chirpz_fused|k_chirpz_rows|k_rec_gemm|k_chirpz_cols" -c 12 -o $out/full_c2 \
    python bench.py --config 2 --profile --steps 1 --warmup 1 > $out/ncu_full.log 2>&1
ncu -i $out/full_c2.ncu-rep --page raw --csv > $out/full_c2_raw.csv 2>/dev/null
python tools/ncu_summary.py $out/full_c2.ncu-rep > $out/full_c2.md 2>&1
python tools/ncu_summary.py --launches $out/launches_c2.csv > $out/launches_c2.md 2>&1
[ $(stat -c %s $out/full_c2.ncu-rep) -gt 40000000 ] && rm -f $out/full_c2.ncu-rep
ls -la $out
