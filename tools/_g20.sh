out=gpurun_out/r01s21; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1
for c in 4 5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $out/c${c}_ctw1.json 2>/dev/null
  bash tools/swap_lib.sh _exp/lib_ctw0.so timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $out/c${c}_ctw0.json 2>/dev/null
done
