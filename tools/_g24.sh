out=gpurun_out/r01s25; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1
for d in 0 2; do echo "DBG=$d" >> $out/probe.txt; CJT_WS_DBG=$d python tools/rec_probe.py 32767 0.5 0.5 2>/dev/null | grep N= | head -3 >> $out/probe.txt; done
for c in 2 4 5; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > $out/c${c}.json 2>/dev/null; done
