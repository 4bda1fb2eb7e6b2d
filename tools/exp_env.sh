#!/bin/bash
# (committed copy of the session script tools/_genv.sh)
# bench configs under environment variants: _genv.sh TAG "CONFIGS" "ENV1" "ENV2" ...
tag=$1; configs=$2; shift 2
out=gpurun_out/$tag; mkdir -p $out
i=0
for ev in "" "$@"; do
  for c in $configs; do
    env $ev timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $out/v${i}_c$c.json 2> $out/v${i}_c$c.err
    python - $out/v${i}_c$c.json "$ev" $c <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print("env[",sys.argv[2],"] config",sys.argv[3],"ms",round(d["ms_per_step"],4), d.get("parity_check_vector0"))
except Exception as e: print(sys.argv[2],sys.argv[3],"ERR",e)
PY
  done
  i=$((i+1))
done 2>&1 | tee $out/summary.txt
