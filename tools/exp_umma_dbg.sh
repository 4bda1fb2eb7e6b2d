#!/bin/bash
# timing experiments on the tcgen05 inverse (build with -DCJT_UMMA_DBG_BUILD in _exp/lib_dbg)
out=gpurun_out/$1; mkdir -p $out
cp paper_1602_02618_b200/_lib/libcjt_b200.so /tmp/libcjt_orig.so
cp _exp/lib_dbg/libcjt_b200.so paper_1602_02618_b200/_lib/libcjt_b200.so
for d in ${2:-0 1 2 4}; do
  CJT_UMMA_DBG=$d timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e > $out/dbg$d.json 2> $out/dbg$d.err
  python - $out/dbg$d.json $d <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print("dbg",sys.argv[2],"ms",round(d["ms_per_step"],4))
PY
done 2>&1 | tee $out/summary.txt
cp /tmp/libcjt_orig.so paper_1602_02618_b200/_lib/libcjt_b200.so
