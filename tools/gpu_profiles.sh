#!/bin/bash
# Evidence for profiles/: launch lists (configs 2, 4), per-stage DRAM traffic
# (configs 2, 4), ncu --set full captures of config 2's stages.
#   gpurun --timeout 3000 -- 'bash tools/gpu_profiles.sh TAG'
tag=${1:-r01}
out=gpurun_out/prof_$tag
mkdir -p $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 2 4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c$c.csv \
      python bench.py --config $c --profile --steps 1 --warmup 1 > $out/ncu_launch_c$c.log 2>&1
  python tools/ncu_summary.py --launches $out/launches_c$c.csv > $out/launches_c$c.md 2>&1
  for st in fwd_rec fwd_blocks fwd_edge inv_rec inv_blocks inv_edge; do
    timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $out/traffic_c${c}_$st.csv \
        python bench.py --config $c --profile-stage $st --warmup 1 > $out/traffic_c${c}_$st.log 2>&1
  done
done
for st in inv_blocks fwd_blocks inv_rec fwd_rec; do
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -o $out/full_c2_$st \
      python bench.py --config 2 --profile-stage $st --warmup 1 > $out/full_c2_$st.log 2>&1
  python tools/ncu_summary.py $out/full_c2_$st.ncu-rep > $out/full_c2_$st.md 2>&1
  ncu -i $out/full_c2_$st.ncu-rep --page raw --csv > $out/full_c2_${st}_raw.csv 2>/dev/null
  [ $(stat -c %s $out/full_c2_$st.ncu-rep) -gt 15000000 ] && rm -f $out/full_c2_$st.ncu-rep
done
ls -la $out
