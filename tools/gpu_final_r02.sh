#!/bin/bash
# Round-2 final evidence, part A (no profiler): GPU tests, smoke, the five
# bench lines, the reference arm on the headline config, and config 3 at the
# per-GPU shard sizes of 2 / 4 / 8 GPUs (one GPU per gpurun call).
#   gpurun --timeout 3600 -- 'bash tools/gpu_final_r02.sh TAG'
tag=${1:-final}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?" >> $out/smoke.log
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err
for c in 2 1 4 5; do
  timeout 900 python bench.py --config $c > $out/bench_c$c.json 2> $out/bench_c$c.err
done
for b in 4096 2048 1024; do
  timeout 600 python bench.py --config 3 --batch $b --no-cpu-baseline > $out/bench_c3_b$b.json 2> $out/bench_c3_b$b.err
done
timeout 900 python bench.py --impl reference > $out/bench_ref_c3.json 2> $out/bench_ref_c3.err
ls -la $out
