out=gpurun_out/r01s10; mkdir -p $out
./tools/fp64_latency > $out/lat.txt 2>&1
python tools/rec_probe.py 4095 0.5 0.5 2>/dev/null | grep N= > $out/rec_probe.txt
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; tail -1 $out/pytest.log >> $out/rec_probe.txt
for c in 3; do timeout 900 python bench.py --config $c --no-cpu-baseline > $out/bench_c$c.json 2> $out/bench_c$c.err; done
