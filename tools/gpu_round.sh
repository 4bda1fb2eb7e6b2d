#!/bin/bash
# One GPU session: parity tests, smoke, bench lines for the given configs and
# the reference arm of the headline config.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG [CONFIGS]'
tag=${1:-r02}
configs=${2:-"3 2 1 4 5"}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
for c in $configs; do
  timeout 900 python bench.py --config $c > $out/bench_c$c.json 2> $out/bench_c$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref_c3.json 2> $out/bench_ref_c3.err
ls -la $out
