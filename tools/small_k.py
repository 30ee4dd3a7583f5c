"""Small-K evaluation latency (paper Table 1 shape): K = 1000 random solutions, f
only, at n = 2500 (density 0.1).  Prints the device time per call (CUDA graph of 50 calls)
for the pair / single-CTA kernels and forced K splits (UBQP_KSPLIT)."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import torch

    from inputs import generate_Q
    from paper_1706_00037_b200 import Ubqp
    n = int(os.environ.get("N", 2500))
    torch.cuda.set_stream(torch.cuda.Stream())
    Q = generate_Q(n, 0.1 if n == 2500 else 1.0, seed=2)
    u = Ubqp(0, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q(Q, 1000)
    u.random(2, 1000)
    f = torch.zeros(1000, dtype=torch.int64, device="cuda")
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    for _ in range(5):
        u.eval_batch(0, f, st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.current_stream()):
        for _ in range(50):
            u.eval_batch(0, f, st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{e0.elapsed_time(e1) / 50 * 1e3:.1f} us", int(f.sum().item()), flush=True)
else:
    for n in (2500, 7000):
        for pair in ("1", "0"):
            for ks in ("0", "1", "2", "4", "8", "16"):
                env = dict(os.environ, UBQP_EVAL_2SM=pair, UBQP_KSPLIT=ks, N=str(n))
                r = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True)
                print(f"n={n} pair={pair} ksplit={ks}: {r.stdout.strip()} {r.stderr.strip()[-200:]}", flush=True)
