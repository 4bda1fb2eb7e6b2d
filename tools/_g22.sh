out=gpurun_out/r01s23; mkdir -p $out
for d in 0 1 2; do echo "DBG=$d" >> $out/probe.txt; CJT_WS_DBG=$d python tools/rec_probe.py 32767 0.5 0.5 2>/dev/null | grep N= | head -3 >> $out/probe.txt; done
