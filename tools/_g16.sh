out=gpurun_out/r01s17; mkdir -p $out
for v in base 64 32; do
  if [ $v = base ]; then cmd="python bench.py --config 2 --no-cpu-baseline --no-e2e"; else cmd="bash tools/swap_lib.sh _exp/lib_ncw$v.so python bench.py --config 2 --no-cpu-baseline --no-e2e"; fi
  $cmd > $out/c2_$v.json 2>/dev/null
  if [ $v = base ]; then c5="python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 5"; else c5="bash tools/swap_lib.sh _exp/lib_ncw$v.so python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 5"; fi
  $c5 > $out/c5_$v.json 2>/dev/null
done
