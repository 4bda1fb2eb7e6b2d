out=gpurun_out/r01s18; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1
for v in 1 0; do for c in 2 5 4; do CJT_MP8K=$v timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $out/bench_c${c}_mp$v.json 2>/dev/null; done; done
