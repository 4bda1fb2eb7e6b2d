out=gpurun_out/r01s4; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "exit $?" >> $out/pytest_gpu.log
for c in 2 4 5 1; do timeout 900 python bench.py --config $c > $out/bench_c$c.json 2> $out/bench_c$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c4.csv \
    python bench.py --config 4 --profile --steps 1 --warmup 1 > $out/ncu_launch_c4.log 2>&1
python tools/ncu_summary.py --launches $out/launches_c4.csv > $out/launches_c4.md 2>&1
