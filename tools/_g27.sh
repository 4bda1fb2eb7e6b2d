out=gpurun_out/r01s28; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1
for v in 40 0 20 80; do for c in 2 5; do CJT_MP_L2_MB=$v timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $out/c${c}_l2_$v.json 2>/dev/null; done; done
