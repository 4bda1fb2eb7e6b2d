#!/bin/bash
# A/B of alternative builds of libcjt_b200.so on bench configs (no CPU legs):
#   gpurun -- 'bash tools/ab_lib.sh TAG "CONFIGS" _exp/libA/libcjt_b200.so ...'
# The in-tree library is measured first as "base".
tag=$1; configs=$2; shift 2
out=gpurun_out/$tag; mkdir -p $out
run() { # name
  for c in $configs; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $out/$1_c$c.json 2> $out/$1_c$c.err
    python - $out/$1_c$c.json $1 $c <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2],"config",sys.argv[3],"ms",round(d["ms_per_step"],4))
except Exception as e: print(sys.argv[2],sys.argv[3],"ERR",e)
PY
  done
}
run base | tee -a $out/summary.txt
cp paper_1602_02618_b200/_lib/libcjt_b200.so /tmp/libcjt_orig.so
for alt in "$@"; do
  cp $alt paper_1602_02618_b200/_lib/libcjt_b200.so
  run $(basename $(dirname $alt)) | tee -a $out/summary.txt
done
cp /tmp/libcjt_orig.so paper_1602_02618_b200/_lib/libcjt_b200.so
