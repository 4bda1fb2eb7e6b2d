out=gpurun_out/r01s9; mkdir -p $out
python tools/rec_probe.py 32767 0.5 0.5 2>/dev/null | grep N= > $out/rec_probe.txt
CJT_WS_DBG=2 python tools/rec_probe.py 32767 0.5 0.5 2>/dev/null | grep N= | head -2 >> $out/rec_probe.txt
python tools/rec_probe.py 16383 -0.25 0.4 2>/dev/null | grep N= >> $out/rec_probe.txt
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; tail -1 $out/pytest.log >> $out/rec_probe.txt
for c in 2 4 5; do timeout 900 python bench.py --config $c --no-cpu-baseline > $out/bench_c$c.json 2> $out/bench_c$c.err; done
