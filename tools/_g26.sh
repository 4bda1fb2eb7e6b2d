out=gpurun_out/r01s27; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1
for v in 1 0; do for c in 2 4 5 3; do CJT_CONCURRENT=$v timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $out/c${c}_conc$v.json 2>/dev/null; done; done
