"""World-size-2 (and 3) CPU tests of the multi-GPU exchange steps (gloo backend).

Each rank computes its shard (slot i <-> g = (rank + floor(i/2) world) 2 + i mod 2) with the
oracle, then the product's exchange code (paper_1706_00037_b200.multistart.combine_stats /
combine_best, the only collectives of the method) must reproduce the single-rank oracle
result exactly: global sum/count/max_key and the best ascended solution with its bits.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from inputs import generate_Q, pack_bits


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, K, lam, max_flips, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1706_00037_b200.multistart import combine_best, combine_stats, key_f
        Q = generate_Q(n, 0.5, seed=42)
        x0 = oracle.first_derivative_start(Q)
        f0 = oracle.xQx(Q, x0)
        B = 2                                        # the library's default sharding block (O10)
        kl = oracle.shard_count(rank, K, world, B)
        X = oracle.diversify(x0, 0, kl, rank, world, B)
        f = oracle.eval_batch(Q, X)
        st = torch.from_numpy(oracle.stats(f, rank, world, B))
        combine_stats(st)
        ssum, scount, skey, _ = st.tolist()
        T = oracle.threshold(lam, ssum, scount, max(f0, key_f(skey)))
        s = oracle.screen(f, T)
        key = -1
        row = np.zeros(len(pack_bits(x0)[0]), dtype=np.int64)
        if s.size:
            Xa, fa, _ = oracle.ascend(Q, X[s], f[s], max_flips)
            keys = [oracle.max_key(int(fa[i]), oracle.global_index(int(s[i]), rank, world, B)) for i in range(s.size)]
            b = int(np.argmax(keys))
            key = keys[b]
            row = pack_bits(Xa[b])[0].view(np.int64)
        gk, bits = combine_best(torch.tensor([key], dtype=torch.int64), torch.from_numpy(row.copy()))
        out[rank] = (ssum, scount, skey, gk, bits.numpy().tobytes(), int(s.size))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_matches_single_rank(world):
    n, K, lam, max_flips = 90, 400, 0.5, 900
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, K, lam, max_flips, out), nprocs=world, join=True)
    # single-rank oracle reference
    Q = generate_Q(n, 0.5, seed=42)
    x0 = oracle.first_derivative_start(Q)
    f0 = oracle.xQx(Q, x0)
    X = oracle.diversify(x0, 0, K)
    f = oracle.eval_batch(Q, X)
    st = oracle.stats(f)
    T = oracle.threshold(lam, int(st[0]), int(st[1]), max(f0, (int(st[2]) >> 22) - (1 << 40)))
    s = oracle.screen(f, T)
    Xa, fa, _ = oracle.ascend(Q, X[s], f[s], max_flips)
    keys = [oracle.max_key(int(fa[i]), int(s[i])) for i in range(s.size)]
    b = int(np.argmax(keys))
    ref_bits = pack_bits(Xa[b])[0].view(np.int64).tobytes()
    assert sum(out[r][5] for r in range(world)) == s.size     # survivors partition
    for r in range(world):
        ssum, scount, skey, gk, bits, _ = out[r]
        assert (ssum, scount, skey) == (int(st[0]), int(st[1]), int(st[2]))
        assert gk == keys[b]
        assert bits == ref_bits


def test_key_helpers_match_oracle():
    from paper_1706_00037_b200.multistart import key_f, key_g
    for f, g in ((0, 0), (-5, 17), (10**9, (1 << 22) - 1), (-(1 << 39), 3)):
        k = oracle.max_key(f, g)
        assert key_f(k) == f and key_g(k) == g


def test_blend_pool_update_matches_oracle_rules():
    """Host logic of the blend policy: multistart.pool_update on packed torch bits makes the
    same decisions as the oracle's pool_update on unpacked arrays (R11b)."""
    from paper_1706_00037_b200.multistart import pool_update
    rng = np.random.default_rng(31)
    n = 70
    sols = [rng.integers(0, 2, size=n).astype(np.uint8) for _ in range(5)]
    pool_o, pool_t = [], []
    for step in range(60):
        inc = sols[rng.integers(0, 5)]
        imp = sols[rng.integers(0, 5)] if rng.random() < 0.4 else None
        rb = sols[rng.integers(0, 5)] if rng.random() < 0.8 else None
        pool_o = oracle.pool_update(pool_o, 3, inc, imp, rb)
        tb = (lambda x: None if x is None else torch.from_numpy(pack_bits(x)[0].view(np.int64)))
        pool_t = pool_update(pool_t, 3, tb(inc), tb(imp), tb(rb))
        assert len(pool_o) == len(pool_t)
        for a, b in zip(pool_o, pool_t):
            assert np.array_equal(pack_bits(a)[0].view(np.int64), b.numpy())


def _worker_real(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1706_00037_b200.multistart import combine_real_stats

        class St:                                   # the ubqp_stats_real fields of one rank
            pass
        rng = np.random.default_rng(100 + rank)
        v = [int(x) << 40 for x in rng.integers(-(2**60), 2**60, size=5)] if rank != 1 else []   # int128 values
        total = sum(v)
        st = St()
        st.sum_hi, st.sum_lo = total >> 64, total & (2**64 - 1)     # uint64 low word, as in the C struct
        st.count = len(v)
        mx = max(v) if v else -(2**127)
        st.max_hi, st.max_lo = mx >> 64, mx & (2**64 - 1)
        st.exp = 7
        out[rank] = combine_real_stats(st)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_real_stats_exchange_is_exact(world):
    """MultiStartReal's exchange: int128 sums of f~ across ranks (one rank empty) are exact."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_real, args=(world, _free_port(), out), nprocs=world, join=True)
    vals = []
    for r in range(world):
        if r != 1:
            vals += [int(x) << 40 for x in np.random.default_rng(100 + r).integers(-(2**60), 2**60, size=5)]
    for r in range(world):
        assert out[r] == (sum(vals), len(vals), max(vals))
