out=gpurun_out/r01s6; mkdir -p $out
python tools/rec_probe.py 32767 0.5 0.5 > $out/rec_probe.txt 2>&1
python tools/rec_probe.py 16383 -0.25 0.4 >> $out/rec_probe.txt 2>&1
