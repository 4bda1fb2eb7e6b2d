out=gpurun_out/r01s15; mkdir -p $out
for s in 2 8 12; do CJT_RAGGED_STREAMS=$s timeout 900 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 5 > $out/bench_c5_s$s.json 2>/dev/null; done
