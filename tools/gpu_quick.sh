#!/bin/bash
# Quick GPU iteration: selected tests + bench lines without the CPU legs.
#   gpurun -- 'bash tools/gpu_quick.sh TAG "TESTS" "CONFIGS"'
tag=${1:-q}; tests=${2:-tests/test_gpu_half.py}; configs=${3:-3}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest $tests -x -q -s -p no:cacheprovider > $out/pytest.log 2>&1; echo "pytest exit $?" >> $out/pytest.log
for c in $configs; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $out/bench_c$c.json 2> $out/bench_c$c.err
done
ls -la $out
