out=gpurun_out/r01s16; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1
python tools/rec_probe.py 32767 0.5 0.5 2>/dev/null | grep N= | head -4 > $out/probe.txt
for c in 5; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e > $out/bench_c$c.json 2> $out/bench_c$c.err; done
