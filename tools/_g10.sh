out=gpurun_out/r01s11; mkdir -p $out
CJT_WS_DBG=2 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_rec_forward_ws -c 2 -o $out/ws_dbg2 python tools/ws_profile.py > $out/ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_rec_forward_ws -c 2 -o $out/ws_full python tools/ws_profile.py >> $out/ncu.log 2>&1
