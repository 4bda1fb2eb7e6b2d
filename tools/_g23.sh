out=gpurun_out/r01s24; mkdir -p $out
CJT_WS_DBG=2 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_rec_inverse_ws -c 2 -o $out/inv_dbg2 python tools/ws_profile.py inverse > $out/ncu.log 2>&1
