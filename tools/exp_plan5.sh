#!/bin/bash
out=gpurun_out/$1; mkdir -p $out
python - <<'PY' 2>&1 | tee $out/plan5.txt
import os, sys, time, json
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "oracle")]
import torch
import cjt_oracle as O
from paper_1602_02618_b200.ragged import RaggedPlan
torch.zeros(1, device="cuda")
draws = O.config5_draws(4096)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); rp = RaggedPlan(draws); torch.cuda.synchronize()
    print(json.dumps({"rep": rep, "ragged_threaded_s": round(time.perf_counter() - t0, 3)}))
    del rp
PY
