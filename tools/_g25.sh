out=gpurun_out/r01s26; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1
for c in 2 1 3 4; do timeout 900 python bench.py --config $c --no-cpu-baseline > $out/c${c}.json 2>/dev/null; done
