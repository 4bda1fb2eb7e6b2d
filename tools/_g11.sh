out=gpurun_out/r01s12; mkdir -p $out
for v in 12 11; do for c in 4 5 2; do CJT_MP_L2MAX=$v timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $out/bench_c${c}_l2_$v.json 2>/dev/null; done; done
