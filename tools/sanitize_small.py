"""Small end-to-end exercise of every kernel for compute-sanitizer (one tool per run)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from inputs import generate_Q, generate_Q_real  # noqa: E402
from paper_1706_00037_b200 import UBQP_EMIT_GAINS, Ubqp, ubqp_stats, ubqp_stats_real  # noqa: E402

for pair in ("1", "0"):
    os.environ["UBQP_EVAL_2SM"] = pair
    for n, K in ((50, 300), (257, 129)):
        Q = generate_Q(n, 0.5, seed=n)
        u = Ubqp(0)
        u.load_Q(Q, K)
        b = np.zeros(u.W64, np.uint64)
        u.first_derivative(b)
        u.diversify(b, 0, K)
        f = np.zeros(K, np.int64)
        st = ubqp_stats()
        u.eval_batch(0, f, st)
        u.eval_batch(UBQP_EMIT_GAINS, f, st)
        surv = np.zeros(K, np.int32)
        m, T = u.screen(0.5, st.sum, st.count, (st.max_key >> 22) - (1 << 40), surv)
        fo = np.zeros(max(m, 1), np.int64)
        bo = np.zeros((max(m, 1), u.W64), np.uint64)
        u.ascend(surv[:m].copy(), m, 10 * n, fo, None, bo)
        u.random(3, K)
        u.eval_batch(0, f)
        G = np.zeros((K, n), np.int32)
        u.eval_batch(UBQP_EMIT_GAINS)
        u.get_gains(0, K, G)
        u.close()
        Qr = generate_Q_real(n, 0.5, seed=n)
        u = Ubqp(0)
        u.load_Q_real(Qr, K)
        u.random(3, K)
        fr = np.zeros(K)
        sr = ubqp_stats_real()
        u.eval_batch_real(fr, sr)
        m, T = u.screen_real(0.5, float(fr.mean()), float(fr.max()), surv)
        u.close()
        print("ok", pair, n, K, m, flush=True)
