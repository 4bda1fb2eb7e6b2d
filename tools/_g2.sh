out=gpurun_out/r01s3; mkdir -p $out
timeout 600 python -m pytest tests/test_recurrences.py -m gpu -x -q > $out/pytest_recur.log 2>&1
for c in 4 5; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c$c.csv \
    python bench.py --config $c --profile --steps 1 --warmup 1 > $out/ncu_launch_c$c.log 2>&1
python tools/ncu_summary.py --launches $out/launches_c$c.csv > $out/launches_c$c.md 2>&1
done
