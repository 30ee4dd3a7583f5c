"""Quick correctness check of the CTA-pair evaluation against the oracle (small cases)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from inputs import generate_Q  # noqa: E402
from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp  # noqa: E402

for n, K in ((300, 500), (1100, 700), (2500, 300)):
    Q = generate_Q(n, 0.6, seed=n)
    u = Ubqp(0)
    u.load_Q(Q, K)
    u.random(3, K)
    X = oracle.random_solutions(n, 3, K)
    ref = oracle.eval_batch(Q, X, nthreads=8)
    for flags in (0, UBQP_EMIT_GAINS):
        f = np.zeros(K, np.int64)
        u.eval_batch(flags, f)
        ok = np.array_equal(f, ref)
        print(n, K, flags, "OK" if ok else "MISMATCH", int((f != ref).sum()), flush=True)
