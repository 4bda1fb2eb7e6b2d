#!/bin/bash
# config-3 iteration: half tests, bench line, launch list of the timed kernels
tag=${1:-c3}; out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_half.py -x -q -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e > $out/bench_c3.json 2> $out/bench_c3.err
python bench.py --config 3 --profile --steps 1 --warmup 1 > $out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   --kernel-name regex:"k_half|k_to_bf16|nvjet|gemm|umma" --csv --log-file $out/launches_c3.csv \
   python bench.py --config 3 --profile --steps 1 --warmup 1 > $out/ncu.log 2>&1
ls -la $out
