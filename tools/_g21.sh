out=gpurun_out/r01s22; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1
for c in 4 5 2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $out/c${c}_q.json 2>/dev/null
  bash tools/swap_lib.sh _exp/lib_head.so timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $out/c${c}_head.json 2>/dev/null
done
