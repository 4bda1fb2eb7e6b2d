out=gpurun_out/r01s13; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; tail -1 $out/pytest.log
for c in 1 2 3 4 5; do timeout 900 python bench.py --config $c --no-cpu-baseline > $out/bench_c$c.json 2> $out/bench_c$c.err; done
