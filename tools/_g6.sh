out=gpurun_out/r01s7; mkdir -p $out
for d in 0 1 2; do echo "CJT_WS_DBG=$d" >> $out/ws_dbg.txt; CJT_WS_DBG=$d python tools/rec_probe.py 32767 0.5 0.5 2>/dev/null | head -4 >> $out/ws_dbg.txt; done
