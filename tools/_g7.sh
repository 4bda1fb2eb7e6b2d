out=gpurun_out/r01s8; mkdir -p $out
python tools/rec_probe.py 32767 0.5 0.5 > $out/rec_probe.txt 2>&1
python tools/rec_probe.py 16383 -0.25 0.4 >> $out/rec_probe.txt 2>&1
for d in 1 2; do echo "CJT_WS_DBG=$d" >> $out/rec_probe.txt; CJT_WS_DBG=$d python tools/rec_probe.py 32767 0.5 0.5 2>/dev/null | head -4 >> $out/rec_probe.txt; done
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; tail -2 $out/pytest.log >> $out/rec_probe.txt
