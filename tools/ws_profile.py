"""One recurrence stage (K1 or K2, VT=16) of (1/2, 1/2), N=32767, for ncu.
    python tools/ws_profile.py [forward|inverse]"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1602_02618_b200 as cj  # noqa: E402
from paper_1602_02618_b200 import _native as nat  # noqa: E402

n, B = 32767, 16
p = cj.JacobiParameters(0.5, 0.5)
direction = sys.argv[1] if len(sys.argv) > 1 else "forward"
fp = cj.plan(direction, p, n)
x = torch.randn(B, n + 1, dtype=torch.float64, device="cuda")
y = (cj.forward_batched if direction == "forward" else cj.inverse_batched)(fp, x)
dp = fp.device_plan(0)
st = torch.cuda.current_stream().cuda_stream
torch.cuda.synchronize()
nat.check(nat.lib().cjt_execute_stage(dp.handle, x.data_ptr(), y.data_ptr(), B, nat.STAGE_REC, st))
torch.cuda.synchronize()
