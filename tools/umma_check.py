"""tcgen05 inverse (alpha = beta = 1/2) vs the cuBLAS path and the oracle.
    CJT_HALF_CUBLAS=1 selects the cuBLAS GEMM + finish (fallback) in a subprocess."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np


def run(n, batch, out):
    import torch
    import cjt_oracle as O
    import paper_1602_02618_b200 as cj
    p = cj.JacobiParameters(0.5, 0.5)
    fp, ip = cj.plan("forward", p, n), cj.plan("inverse", p, n)
    c = np.stack([O.seeded_vector(3, v, n) for v in range(batch)])
    f = cj.forward_batched(fp, torch.from_numpy(c).cuda())
    i = cj.inverse_batched(ip, f)
    torch.cuda.synchronize()
    np.save(out, i.cpu().numpy())
    np.save(out + ".f.npy", f.cpu().numpy())


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "run":
        run(int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
        sys.exit(0)
    import cjt_oracle as O
    res = {}
    for n, batch in ((4095, 300), (1023, 17), (255, 5), (8191, 40)):
        a, b = f"/tmp/umma_{n}.npy", f"/tmp/cublas_{n}.npy"
        subprocess.check_call([sys.executable, __file__, "run", str(n), str(batch), a], timeout=300)
        subprocess.check_call([sys.executable, __file__, "run", str(n), str(batch), b], timeout=300,
                              env=dict(os.environ, CJT_HALF_CUBLAS="1"))
        ia, ib, f = np.load(a), np.load(b), np.load(a + ".f.npy")
        l1 = np.abs(f).sum(axis=1)
        d = float((np.max(np.abs(ia - ib), axis=1) / l1).max())
        worst = 0.0
        for v in (0, batch - 1):
            ref = O.oracle_inverse(0.5, 0.5, f[v])
            worst = max(worst, O.parity(ia[v], ref, f[v]))
        res[n] = {"umma_vs_cublas": d, "umma_vs_oracle": worst}
        print(json.dumps({n: res[n]}), flush=True)
