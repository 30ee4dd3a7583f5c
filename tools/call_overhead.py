"""Host cost of one small evaluation call (paper Table 1 shape: K = 1000, f only) against its
device time: wall time of back-to-back calls without a sync (the host submission rate), the
same calls timed by events, and a CUDA graph of the calls (device only).
    python tools/call_overhead.py [n]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from inputs import generate_Q  # noqa: E402
from paper_1706_00037_b200 import Ubqp  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2500
    torch.cuda.set_stream(torch.cuda.Stream())
    Q = generate_Q(n, 0.1 if n == 2500 else 1.0, seed=2)
    u = Ubqp(0, stream=torch.cuda.current_stream().cuda_stream)
    u.load_Q(Q, 1000)
    u.random(2, 1000)
    f = torch.zeros(1000, dtype=torch.int64, device="cuda")
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    fp, sp = f.data_ptr(), st.data_ptr()
    for _ in range(20):
        u.eval_batch(0, f, st)
    torch.cuda.synchronize()
    reps = 200
    for label, args in (("torch tensors", (f, st)), ("raw pointers", (fp, sp))):
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            u.eval_batch(0, *args)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        print(f"n={n} {label}: host {(t1 - t0) / reps * 1e6:6.2f} us/call, events {e0.elapsed_time(e1) / reps * 1e3:6.2f} us/call")
    # the C call alone: ctypes with preconverted arguments
    import ctypes
    fn = u.lib.ubqp_eval_batch
    h = u.h
    t0 = time.perf_counter()
    for _ in range(reps):
        fn(h, 0, ctypes.c_void_p(fp), ctypes.c_void_p(sp))
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"n={n} bare ctypes: host {(t1 - t0) / reps * 1e6:6.2f} us/call")
    t0 = time.perf_counter()
    for _ in range(reps):
        fn(h, 0, None, None)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"n={n} bare ctypes, no outputs: host {(t1 - t0) / reps * 1e6:6.2f} us/call")
    q = u.lib.ubqp_query
    v = ctypes.c_int64()
    t0 = time.perf_counter()
    for _ in range(reps):
        q(h, 0, ctypes.byref(v))
    t1 = time.perf_counter()
    print(f"n={n} ubqp_query (guard only): host {(t1 - t0) / reps * 1e6:6.2f} us/call")
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
    print(f"n={n} graph: {e0.elapsed_time(e1) / 50 * 1e3:6.2f} us/call (device)")
    u.close()


if __name__ == "__main__":
    main()
