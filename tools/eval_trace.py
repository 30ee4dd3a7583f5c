"""Milestones of one small-K evaluation launch (paper Table 1 shape: K = 1000 random solutions,
f only) from a trace build of the library (UBQP_NVCC_EXTRA=-DUBQP_EVAL_TRACE=1):
%globaltimer stamps per CTA, printed relative to the earliest kernel entry.
    UBQP_LIB=variants/trace.so python tools/eval_trace.py [n] [K]"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import generate_Q  # noqa: E402
from paper_1706_00037_b200 import Ubqp  # noqa: E402

NAMES = ["entry", "prologue done", "producer done", "first stage landed (MMA)", "MMA done",
         "epilogue: TMEM full", "epilogue done", "fold: last item in", "fold done", "exit sync",
         "fold: group counter back", "fold: group summed", "fold: global counter back", "fold: stats loaded",
         "fold: acquired (last arriver)", "fold: partials loaded"]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2500
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    torch.cuda.set_stream(torch.cuda.Stream())
    Q = generate_Q(n, 0.1 if n == 2500 else 1.0, seed=2)
    u = Ubqp(0, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q(Q, K)
    u.random(2, K)
    f = torch.zeros(K, dtype=torch.int64, device="cuda")
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    for _ in range(20):
        u.eval_batch(0, f, st)
    torch.cuda.synchronize()
    buf = np.zeros((512, 16), np.uint64)
    fn = u.lib.ubqp_debug_eval_trace
    fn.argtypes = [ctypes.c_void_p]
    assert fn(buf.ctypes.data) == 0
    ctas = int((buf[:, 0] > 0).sum())
    t = buf[:ctas].astype(np.float64)
    t0 = t[:, 0].min()
    print(f"n={n} K={K} CTAs={ctas}  (us after the first CTA entered; median / max over CTAs that stamped)")
    for i, name in enumerate(NAMES):
        v = t[:, i]
        v = v[v > 0]
        if len(v):
            print(f"  {i} {name:26s} {np.median(v - t0) / 1e3:7.2f} {np.max(v - t0) / 1e3:7.2f}  ({len(v)} CTAs)")


if __name__ == "__main__":
    main()
