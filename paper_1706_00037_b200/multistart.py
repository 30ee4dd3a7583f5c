"""One round of the diversified multi-start (Figure 2) over 1..N GPUs.

torch is plumbing here: device buffers, the CUDA stream shared with libubqp.so, and
torch.distributed (NCCL) for the only exchange steps of the method:
  * the screening statistics {sum f, count, max_key} of the sharded batch (T uses
    the Mean and Max over all solutions), and
  * the best-record key (MAX) plus a broadcast of the winner's bits from its owner rank
    (UpdateBestAndT).
Solutions are sharded in blocks of B = 2 dealt round robin (slot i on rank r <->
g = (r + floor(i/2) world) 2 + i mod 2, include/ubqp.h "Sharding") and Q is
replicated; every other step runs in the kernels behind include/ubqp.h.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

import torch
import torch.distributed as dist

from .ubqp import (OPT_SHARD_BLOCK, SHARD_BLOCK_DEFAULT, UBQP_EMIT_GAINS, Ubqp, global_index, shard_count,
                   shard_owner)

KEY_SHIFT = 22
F_OFFSET = 1 << 40
POLISH_MAX_PAIRS = 72            # E (E - 1) for an elite set of pool_cap + 1 = 9


def key_f(key: int) -> int:
    """objective value stored in a max_key (include/ubqp.h)"""
    return (int(key) >> KEY_SHIFT) - F_OFFSET


def key_g(key: int) -> int:
    """global solution index stored in a max_key"""
    return (1 << KEY_SHIFT) - 1 - (int(key) & ((1 << KEY_SHIFT) - 1))


def paper_lambda(mean: float, start_value: int) -> float:
    """P:55 "lambda is initially set to Max / Mean = Starting_solution / Mean", clamped to
    (0, 1]: the raw ratio exceeds 1 whenever the start beats the mean (R7)."""
    if mean <= 0 or start_value <= 0:
        return 0.5
    return min(1.0, max(1e-6, start_value / mean))


# UBQP_FORCE_COLLECTIVES=1 runs the exchange steps even at world size 1 (tests: the NCCL path
# on a single GPU, tests/test_gpu_nccl.py); results are identical either way
FORCE_COLLECTIVES = os.environ.get("UBQP_FORCE_COLLECTIVES", "0") == "1"


def dist_info(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def _collective(world: int) -> bool:
    return world > 1 or (FORCE_COLLECTIVES and dist.is_available() and dist.is_initialized())


# ---------------------------------------------------------------- exchange steps (tested on gloo)
def combine_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """stats int64[4] = {sum, count, max_key, 0} per rank -> global (SUM, SUM, MAX) in place."""
    _, world = dist_info(group)
    if _collective(world):
        sc = stats[:2].clone()
        mk = stats[2:3].clone()
        dist.all_reduce(sc, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(mk, op=dist.ReduceOp.MAX, group=group)
        stats[:2].copy_(sc)
        stats[2:3].copy_(mk)
    return stats


def combine_best(key: torch.Tensor, bits_row: torch.Tensor, group=None, block: int = SHARD_BLOCK_DEFAULT):
    """key int64[1] (rank-local best max_key, -1 = none), bits_row int64[W64] (that
    solution's bits on its rank).  Returns (global key, winner bits) on every rank: MAX of
    the keys, then a broadcast of the bits from the rank owning g = key_g (O10 sharding)."""
    rank, world = dist_info(group)
    if not _collective(world):
        return int(key.item()), bits_row
    gk = key.clone()
    dist.all_reduce(gk, op=dist.ReduceOp.MAX, group=group)
    k = int(gk.item())
    if k < 0:
        return k, bits_row
    owner = shard_owner(key_g(k), world, block)[0]
    out = bits_row.clone()
    src = dist.get_global_rank(group, owner) if group is not None else owner
    dist.broadcast(out, src=src, group=group)
    return k, out


def pool_update(pool: list, pool_cap: int, inc_bits: torch.Tensor, improved_from, round_best) -> list:
    """Parent pool of the blend policy (R11b): distinct local optima other than
    the incumbent, oldest first, at most pool_cap.  After a round the replaced incumbent
    (improved_from), else the round's best ascended solution, joins unless it equals the
    incumbent or is already pooled.  Every rank holds the same pool (the round best is
    broadcast by combine_best), so the blend stays independent of the world size (O10)."""
    cand = improved_from if improved_from is not None else round_best
    if cand is None or torch.equal(cand, inc_bits) or any(torch.equal(cand, p) for p in pool):
        return pool
    return (pool + [cand.clone()])[-pool_cap:]


@dataclass
class RoundResult:
    m: int            # survivors on this rank
    T: float          # screening value
    best_key: int     # global best max_key of the ascended survivors (-1: none)
    best_bits: torch.Tensor
    batch_max: int
    mean_sum: int
    mean_count: int


class MultiStart:
    """Diversify -> eval(+gains) -> [all-reduce stats] -> screen -> ascend -> [best record]."""

    def __init__(self, Q: np.ndarray, K: int, lam: float = 0.5, max_flips: int | None = None,
                 device: int | None = None, group=None):
        self.rank, self.world = dist_info(group)
        self.group = group
        self.device = torch.cuda.current_device() if device is None else device
        self.n = int(Q.shape[0])
        self.K = int(K)
        self.block = SHARD_BLOCK_DEFAULT
        self.k_local = shard_count(self.rank, self.K, self.world, self.block)
        self.lam = float(lam)
        self.max_flips = 10 * self.n if max_flips is None else int(max_flips)
        self.qmax = int(np.abs(np.asarray(Q)).max()) if self.n else 0
        # one non-default stream shared by torch (collectives, small ops) and libubqp.so
        self.stream = torch.cuda.Stream(device=self.device)
        torch.cuda.set_stream(self.stream)
        self.u = Ubqp(self.device, stream=self.stream.cuda_stream)
        self.u.set_option(OPT_SHARD_BLOCK, self.block)
        # workspace also holds a polish batch: all ordered pairs of <= 9 elite solutions
        self.u.load_Q(np.ascontiguousarray(Q, dtype=np.int32), max(self.k_local, POLISH_MAX_PAIRS))
        self.W64 = self.u.W64
        dv = torch.device("cuda", self.device)
        kl = max(self.k_local, POLISH_MAX_PAIRS)
        self.stats = torch.zeros(4, dtype=torch.int64, device=dv)
        self.surv = torch.zeros(kl, dtype=torch.int32, device=dv)
        self.f_asc = torch.zeros(kl, dtype=torch.int64, device=dv)
        self.flips = torch.zeros(kl, dtype=torch.int32, device=dv)
        self.bits = torch.zeros((kl, self.W64), dtype=torch.int64, device=dv)
        self.key = torch.zeros(1, dtype=torch.int64, device=dv)
        self.fd_bits = torch.zeros(self.W64, dtype=torch.int64, device=dv)

    # CalculateFirstDerivativeSolution and its value (one-solution eval)
    def first_derivative(self):
        self.u.first_derivative(self.fd_bits)
        self.u.set_batch(self.fd_bits, 1, 0, 1)
        f = torch.zeros(1, dtype=torch.int64, device=self.fd_bits.device)
        self.u.eval_batch(0, f)
        return self.fd_bits.clone(), int(f.item())

    # EvaluateRandomStarts: (sum, count) of K random solutions
    def sample_mean(self, seed: int, K: int | None = None):
        K = self.K if K is None else K
        kl = shard_count(self.rank, K, self.world, self.block)
        self.u.random(seed, kl, self.rank, self.world)
        self.u.eval_batch(0, None, self.stats)
        combine_stats(self.stats, self.group)
        s = self.stats.tolist()
        return s[0], s[1]

    def round(self, seed_bits: torch.Tensor, t0: int, inc_f: int, mean=None,
              parents: torch.Tensor | None = None) -> RoundResult:
        """One batched round.  mean=None -> the batch's own mean (R5).
        parents [P][W64] (device): blend diversification (O4b) instead of Glover (O4)."""
        u = self.u
        if parents is None:
            u.diversify(seed_bits, t0, self.k_local, self.rank, self.world)
        else:
            u.blend(seed_bits, parents, int(parents.shape[0]), t0, self.k_local, self.rank, self.world)
        u.eval_batch(UBQP_EMIT_GAINS, None, self.stats)
        combine_stats(self.stats, self.group)
        ssum, scount, skey, _ = self.stats.tolist()
        batch_max = key_f(skey)
        mean_sum, mean_count = (ssum, scount) if mean is None else mean
        maxv = max(inc_f, batch_max)
        m, T = u.screen(self.lam, mean_sum, mean_count, maxv, self.surv)
        u.ascend(self.surv, m, self.max_flips, self.f_asc, self.flips, self.bits, self.key)
        row = self.bits[0]
        if m > 0 and _collective(self.world):
            k_local = int(self.key.item())
            owner, slot = shard_owner(key_g(k_local), self.world, self.block) if k_local >= 0 else (-1, -1)
            if k_local >= 0 and owner == self.rank:
                i = int(torch.searchsorted(self.surv[:m], torch.tensor([slot], dtype=torch.int32,
                                                                        device=self.surv.device)).item())
                row = self.bits[i]
        best_key, best_bits = combine_best(self.key, row.contiguous(), self.group, self.block)
        if not _collective(self.world) and m > 0:
            best_key = int(self.key.item())
            slot = key_g(best_key)
            i = int(torch.searchsorted(self.surv[:m], torch.tensor([slot], dtype=torch.int32,
                                                                    device=self.surv.device)).item())
            best_bits = self.bits[i].clone()
        return RoundResult(m, T, best_key, best_bits, batch_max, mean_sum, mean_count)

    def polish(self, elite: torch.Tensor):
        """Path relinking over an elite set (NEXT-4, R19): every ordered pair (a, b), a != b,
        relinked from elite[a] toward elite[b] (ubqp_relink), the best interior points
        ascended (ubqp_ascend).  Replicated on every rank (a few dozen walks), so the result
        is the same for any world size.  Returns (f, bits) or None."""
        E = int(elite.shape[0])
        pairs = [(a, b) for a in range(E) for b in range(E) if a != b]
        if not pairs:
            return None
        if len(pairs) > POLISH_MAX_PAIRS:
            raise ValueError(f"polish: at most {POLISH_MAX_PAIRS} pairs")
        dv = elite.device
        ia = torch.tensor([a for a, _ in pairs], device=dv)
        ib = torch.tensor([b for _, b in pairs], device=dv)
        X0 = elite[ia].contiguous()
        Y = elite[ib].contiguous()
        m = len(pairs)
        u = self.u
        u.set_batch(X0, m, 0, 1)
        u.eval_batch(UBQP_EMIT_GAINS)
        slots = torch.arange(m, dtype=torch.int32, device=dv)
        f = torch.zeros(m, dtype=torch.int64, device=dv)
        st = torch.zeros(m, dtype=torch.int32, device=dv)
        bits = torch.zeros((m, self.W64), dtype=torch.int64, device=dv)
        u.relink(Y, m, slots, m, f, st, None, bits, None)
        sel = torch.nonzero(st >= 0).flatten()
        k = int(sel.numel())
        if k == 0:
            return None
        u.set_batch(bits[sel].contiguous(), k, 0, 1)
        u.eval_batch(UBQP_EMIT_GAINS)
        u.ascend(slots[:k], k, self.max_flips, self.f_asc, self.flips, self.bits, self.key)
        key = int(self.key.item())
        i = key_g(key)
        return key_f(key), self.bits[i].clone()

    def run(self, rounds: int, sample_seed: int, t_start: int = 0, lam_policy: str = "fixed",
            div: str = "glover", pool_cap: int = 8, polish_end: bool = False):
        """Figure 2 as batched rounds (O8): pinned sampling mean, first-derivative
        incumbent, rounds of diversify/eval/screen/ascend; strict improvement.
        lam_policy "paper": lambda = Max/Mean = Starting_solution/Mean, clamped to
        (0, 1] with 0.5 when Mean <= 0 or the start's value <= 0 (R7).
        div "blend": once the parent pool is non-empty, rounds blend the incumbent with
        pool[g mod P] (O4b) instead of Glover's generator.  polish_end: after the
        last round, polish(pool + [incumbent]); a strict improvement is recorded as round
        rounds + 1."""
        if polish_end:
            # fail before any round runs (not after all of them): the polish batch holds every
            # ordered pair of pool + incumbent, and ubqp_relink needs (2n-1) qmax < 2^21
            if (pool_cap + 1) * pool_cap > POLISH_MAX_PAIRS:
                raise ValueError(f"polish_end: pool_cap {pool_cap} gives more than {POLISH_MAX_PAIRS} pairs")
            if (2 * self.n - 1) * self.qmax >= (1 << 21):
                raise ValueError("polish_end: path relinking needs (2n-1)*qmax < 2^21 (ubqp_relink E_RANGE)")
        mean = self.sample_mean(sample_seed)
        inc_bits, inc_f = self.first_derivative()
        if lam_policy == "paper":
            self.lam = paper_lambda(mean[0] / mean[1], inc_f)
        traj = [(0, inc_f)]
        pool: list = []
        for r in range(1, rounds + 1):
            parents = torch.stack(pool) if (div == "blend" and pool) else None
            res = self.round(inc_bits, t_start + (r - 1) * self.K, inc_f, mean, parents=parents)
            improved_from = None
            if res.best_key >= 0 and key_f(res.best_key) > inc_f:
                improved_from = inc_bits
                inc_f = key_f(res.best_key)
                inc_bits = res.best_bits.clone()
                traj.append((r, inc_f))
            if div == "blend" or polish_end:
                pool = pool_update(pool, pool_cap, inc_bits, improved_from,
                                   res.best_bits if res.best_key >= 0 else None)
        if polish_end:
            res = self.polish(torch.stack(pool + [inc_bits]))
            if res is not None and res[0] > inc_f:
                inc_f, inc_bits = res
                traj.append((rounds + 1, inc_f))
        return inc_f, inc_bits, traj


# ---------------------------------------------------------------- real-valued Q (R20, R22)
def combine_real_stats(st, group=None):
    """ubqp_stats_real of each rank -> (sum f~ as a Python int, count, max f~ or None): one
    all_gather of the six int64 words per rank, combined exactly on the host (int128 sums)."""
    _, world = dist_info(group)
    lo64 = lambda v: v - (1 << 64) if v >= (1 << 63) else v     # uint64 word -> int64 tensor value
    words = torch.tensor([st.sum_hi, lo64(st.sum_lo), st.count, st.max_hi, lo64(st.max_lo), st.exp],
                         dtype=torch.int64)
    if world > 1:
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        words = words.to(dev)
        out = [torch.zeros_like(words) for _ in range(world)]
        dist.all_gather(out, words, group=group)
        rows = [o.cpu().tolist() for o in out]
    else:
        rows = [words.tolist()]
    i128 = lambda hi, lo: (hi << 64) | (lo & (2**64 - 1))
    total = sum(i128(r[0], r[1]) for r in rows)
    maxes = [i128(r[3], r[4]) for r in rows if r[2] > 0]
    return total, sum(r[2] for r in rows), (max(maxes) if maxes else None)


class MultiStartReal:
    """Figure 2 rounds on a real-valued Q: objective values on the evaluation image (R22:
    x^t Q x correctly rounded for float32 Q), the walk on the walk image (R20).  Mean is the
    exact mean of the sampled values rounded once; Max, T and the best record are binary64.
    Same sharding and exchange pattern as MultiStart."""

    def __init__(self, Q: np.ndarray, K: int, lam: float = 0.5, max_flips: int | None = None,
                 device: int | None = None, group=None):
        from .ubqp import ubqp_stats_real
        self.rank, self.world = dist_info(group)
        self.group = group
        self.device = torch.cuda.current_device() if device is None else device
        self.n = int(Q.shape[0])
        self.K = int(K)
        self.block = SHARD_BLOCK_DEFAULT
        self.k_local = shard_count(self.rank, self.K, self.world, self.block)
        self.lam = float(lam)
        self.max_flips = 10 * self.n if max_flips is None else int(max_flips)
        self.stream = torch.cuda.Stream(device=self.device)
        torch.cuda.set_stream(self.stream)
        self.u = Ubqp(self.device, stream=self.stream.cuda_stream)
        self.u.set_option(OPT_SHARD_BLOCK, self.block)
        self.u.load_Q_real(np.ascontiguousarray(Q), max(self.k_local, 1))
        self.e = self.u.real_exp          # walk image (R20)
        self.w = self.u.eval_exp          # evaluation image (R22)
        self.W64 = self.u.W64
        dv = torch.device("cuda", self.device)
        kl = max(self.k_local, 1)
        self.st = ubqp_stats_real()
        self.surv = torch.zeros(kl, dtype=torch.int32, device=dv)
        self.fa = torch.zeros(kl, dtype=torch.float64, device=dv)
        self.flips = torch.zeros(kl, dtype=torch.int32, device=dv)
        self.bits = torch.zeros((kl, self.W64), dtype=torch.int64, device=dv)
        self.fd_bits = torch.zeros(self.W64, dtype=torch.int64, device=dv)

    def _value(self, fint: int) -> float:
        """2^-w f~ rounded once to binary64"""
        from fractions import Fraction
        return float(Fraction(fint) / (Fraction(2) ** self.w))

    def sample_mean(self, seed: int) -> float:
        from fractions import Fraction
        self.u.random(seed, self.k_local, self.rank, self.world)
        self.u.eval_batch_real(None, self.st)
        total, count, _ = combine_real_stats(self.st, self.group)
        return float(Fraction(total, count) / (Fraction(2) ** self.w))

    def first_derivative(self):
        self.u.first_derivative(self.fd_bits)
        self.u.set_batch(self.fd_bits, 1, 0, 1)
        self.u.eval_batch_real(None, self.st)
        return self.fd_bits.clone(), self._value(self.st.max_fint)

    def round(self, seed_bits, t0: int, inc_f: float, mean: float):
        """-> (m on this rank, T, best f over all ranks or None, its bits)."""
        u = self.u
        u.diversify(seed_bits, t0, self.k_local, self.rank, self.world)
        u.eval_batch_real(None, self.st)
        _, _, bmax = combine_real_stats(self.st, self.group)
        maxv = inc_f if bmax is None else max(inc_f, self._value(bmax))
        m, T = u.screen_real(self.lam, mean, maxv, self.surv)
        best = None
        if m > 0:
            u.ascend_real(self.surv, m, self.max_flips, self.fa, None, self.flips, self.bits)
            fa = self.fa[:m]
            mx = float(fa.max().item())
            i = int(torch.nonzero(fa == mx)[0].item())      # lowest slot = lowest g among ties
            best = (mx, global_index(int(self.surv[i].item()), self.rank, self.world, self.block), i)
        # global best: highest f, then lowest g; the owner broadcasts the bits
        cand = torch.tensor([best[0], float(best[1])] if best else [float("-inf"), float(2**62)], dtype=torch.float64)
        if self.world > 1:
            dev = self.bits.device if dist.get_backend(self.group) == "nccl" else "cpu"
            cand = cand.to(dev)
            out = [torch.zeros_like(cand) for _ in range(self.world)]
            dist.all_gather(out, cand, group=self.group)
            rows = [o.cpu().tolist() for o in out]
        else:
            rows = [cand.tolist()]
        gf, gg = max(rows, key=lambda r: (r[0], -r[1]))
        if gf == float("-inf"):
            return m, T, None, None
        gg = int(gg)
        owner = shard_owner(gg, self.world, self.block)[0]
        row = self.bits[best[2]].clone() if (best and owner == self.rank) else torch.zeros_like(self.bits[0])
        if self.world > 1:
            src = dist.get_global_rank(self.group, owner) if self.group is not None else owner
            if dist.get_backend(self.group) != "nccl":
                row = row.cpu()
            dist.broadcast(row, src=src, group=self.group)
            row = row.to(self.bits.device)
        return m, T, gf, row

    def run(self, rounds: int, sample_seed: int, t_start: int = 0):
        mean = self.sample_mean(sample_seed)
        inc_bits, inc_f = self.first_derivative()
        traj = [(0, inc_f)]
        for r in range(1, rounds + 1):
            _, _, bf, bb = self.round(inc_bits, t_start + (r - 1) * self.K, inc_f, mean)
            if bf is not None and bf > inc_f:
                inc_f, inc_bits = bf, bb.clone()
                traj.append((r, inc_f))
        return inc_f, inc_bits, traj
