"""Paper Table 1 shape: 1000 random solutions evaluated at n = 2500/5000/7000."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from inputs import generate_Q  # noqa: E402
from paper_1706_00037_b200 import Ubqp  # noqa: E402

torch.cuda.set_stream(torch.cuda.Stream())
for n, dens, sq in ((2500, 0.1, 2), (5000, 1.0, 3), (7000, 1.0, 4)):
    Q = generate_Q(n, dens, seed=sq)
    u = Ubqp(0, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q(Q, 1000)
    u.random(sq, 1000)
    f = torch.zeros(1000, dtype=torch.int64, device="cuda")
    for _ in range(5):
        u.eval_batch(0, f)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        u.eval_batch(0, f)
    e1.record()
    torch.cuda.synchronize()
    api_us = e0.elapsed_time(e1) / 50 * 1e3
    # the same 50 calls captured in a CUDA graph: device time without host launch overhead
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.current_stream()):
        for _ in range(50):
            u.eval_batch(0, f, st)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(n, f"{api_us:.1f} us per 1000 evals (API calls), {e0.elapsed_time(e1) / 50 * 1e3:.1f} us (graph replay)",
          int(f.sum().item()), st.tolist(), flush=True)
    u.close()
