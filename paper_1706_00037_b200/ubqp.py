"""Thin Python binding of include/ubqp.h (argument marshalling only).

Every step of the hot path runs in libubqp.so's CUDA kernels; this module only converts
torch tensors / numpy arrays into pointers and error codes into exceptions.  There is no
CPU fallback: if the shared library is missing or cannot be loaded, importing the handle
raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libubqp.so"
_lib = None

UBQP_OK, UBQP_E_INVALID, UBQP_E_NOT_SYMMETRIC, UBQP_E_RANGE, UBQP_E_STATE, UBQP_E_NOMEM, UBQP_E_CUDA = range(7)
UBQP_EMIT_GAINS = 1
Q_N, Q_NPAD, Q_W64, Q_KMAX, Q_KLOCAL, Q_LAUNCHES, Q_STREAM = range(7)

# every entry point declared in include/ubqp.h
EXPORTS = ["ubqp_version", "ubqp_create", "ubqp_destroy", "ubqp_last_error", "ubqp_load_Q",
           "ubqp_diversify", "ubqp_blend", "ubqp_random", "ubqp_first_derivative", "ubqp_set_batch", "ubqp_get_batch", "ubqp_eval_batch",
           "ubqp_get_gains", "ubqp_screen", "ubqp_ascend", "ubqp_relink", "ubqp_sync", "ubqp_query",
           "ubqp_load_Q_real", "ubqp_eval_batch_real", "ubqp_screen_real", "ubqp_ascend_real",
           "ubqp_set_option"]
UBQP_F32, UBQP_F64 = 1, 2
Q_REAL_EXP, Q_IS_REAL, Q_EVAL_EXP, Q_EVAL_LIMBS, Q_NNZ, Q_SPARSE_ROWS, Q_SHARD_BLOCK = 7, 8, 9, 10, 11, 12, 13
Q_ASCENT_LAST = 14
OPT_ASCENT, OPT_EVAL_PAIR, OPT_EVAL_TRI, OPT_SHARD_BLOCK = 0, 1, 2, 3
SHARD_BLOCK_DEFAULT = 2


def global_index(i: int, rank: int, world: int, block: int = SHARD_BLOCK_DEFAULT) -> int:
    """global solution index of slot i on rank `rank` (include/ubqp.h "Sharding")"""
    return (rank + (i // block) * world) * block + i % block


def shard_count(rank: int, K: int, world: int, block: int = SHARD_BLOCK_DEFAULT) -> int:
    """slots of `rank` in a global batch of K"""
    full, rem = divmod(K, world * block)
    return full * block + min(block, max(0, rem - rank * block))


def shard_owner(g: int, world: int, block: int = SHARD_BLOCK_DEFAULT):
    """(rank, slot) holding global solution g"""
    b, o = divmod(g, block)
    r, q = b % world, b // world
    return r, q * block + o


# UBQP_OPT_ASCENT values (include/ubqp.h): automatic, dense CTA, sparse rows, one warp per
# solution, 2-4 warps per solution
ASCENT_AUTO, ASCENT_DENSE, ASCENT_SPARSE, ASCENT_WARP, ASCENT_MW = 0, 1, 2, 3, 4


class UbqpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"ubqp error {code}: {msg}")
        self.code = code


class ubqp_stats_real(ctypes.Structure):
    """statistics of a real-Q batch on the evaluation image (include/ubqp.h): f~ = f 2^exp"""
    _fields_ = [("sum_hi", ctypes.c_int64), ("sum_lo", ctypes.c_uint64), ("count", ctypes.c_int64),
                ("max_hi", ctypes.c_int64), ("max_lo", ctypes.c_uint64), ("exp", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]

    @property
    def sum_fint(self) -> int:
        return (self.sum_hi << 64) | self.sum_lo

    @property
    def max_fint(self) -> int:
        return (self.max_hi << 64) | self.max_lo


class ubqp_stats(ctypes.Structure):
    _fields_ = [("sum", ctypes.c_int64), ("count", ctypes.c_int64), ("max_key", ctypes.c_int64),
                ("reserved", ctypes.c_int64)]


def load_library(path: Path | str | None = None):
    """Load libubqp.so (raises OSError if absent: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    # UBQP_LIB: load another build of the same library (A/B timing of kernel variants)
    p = Path(path) if path else Path(os.environ.get("UBQP_LIB", LIB_PATH))
    if not p.exists():
        raise OSError(f"{p} not built: run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(str(p))
    P, i32, i64, u64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    sig = {
        "ubqp_version": ([], ctypes.c_int),
        "ubqp_create": ([ctypes.c_int, P, ctypes.POINTER(P)], ctypes.c_int),
        "ubqp_destroy": ([P], ctypes.c_int),
        "ubqp_last_error": ([P], ctypes.c_char_p),
        "ubqp_load_Q": ([P, i32, P, i64], ctypes.c_int),
        "ubqp_diversify": ([P, P, i64, i64, i32, i32], ctypes.c_int),
        "ubqp_blend": ([P, P, P, i64, i64, i64, i32, i32], ctypes.c_int),
        "ubqp_random": ([P, u64, i64, i32, i32], ctypes.c_int),
        "ubqp_set_batch": ([P, P, i64, i32, i32], ctypes.c_int),
        "ubqp_get_batch": ([P, P], ctypes.c_int),
        "ubqp_first_derivative": ([P, P], ctypes.c_int),
        "ubqp_eval_batch": ([P, ctypes.c_int, P, P], ctypes.c_int),
        "ubqp_get_gains": ([P, i64, i64, P], ctypes.c_int),
        "ubqp_screen": ([P, dbl, i64, i64, i64, P, P, P], ctypes.c_int),
        "ubqp_ascend": ([P, P, i64, i32, P, P, P, P], ctypes.c_int),
        "ubqp_relink": ([P, P, i64, P, i64, P, P, P, P, P], ctypes.c_int),
        "ubqp_sync": ([P], ctypes.c_int),
        "ubqp_query": ([P, ctypes.c_int, ctypes.POINTER(i64)], ctypes.c_int),
        "ubqp_load_Q_real": ([P, i32, ctypes.c_int, P, i64], ctypes.c_int),
        "ubqp_eval_batch_real": ([P, P, P], ctypes.c_int),
        "ubqp_screen_real": ([P, dbl, dbl, dbl, P, P, P], ctypes.c_int),
        "ubqp_ascend_real": ([P, P, i64, i32, P, P, P, P], ctypes.c_int),
        "ubqp_set_option": ([P, ctypes.c_int, i64], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _ptr(a):
    """data pointer of a torch tensor / numpy array / ctypes object / int; None -> NULL."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous()
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return a.ctypes.data
    return ctypes.addressof(a)


class Ubqp:
    """One handle = (process, device, stream).  Method names follow include/ubqp.h."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = load_library()
        h = ctypes.c_void_p()
        rc = self.lib.ubqp_create(device, ctypes.c_void_p(stream) if stream else None, ctypes.byref(h))
        if rc:
            raise UbqpError(rc, "ubqp_create failed (needs an sm_100 B200 device)")
        self.h = h

    def _ck(self, rc):
        if rc:
            raise UbqpError(rc, self.lib.ubqp_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.ubqp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def query(self, what: int) -> int:
        v = ctypes.c_int64()
        self._ck(self.lib.ubqp_query(self.h, what, ctypes.byref(v)))
        return v.value

    @property
    def n(self):
        return self.query(Q_N)

    @property
    def W64(self):
        return self.query(Q_W64)

    @property
    def launches(self):
        return self.query(Q_LAUNCHES)

    def load_Q(self, Q, k_max: int):
        if isinstance(Q, np.ndarray):
            Q = np.ascontiguousarray(Q, dtype=np.int32)
        n = Q.shape[0]
        self._ck(self.lib.ubqp_load_Q(self.h, n, _ptr(Q), k_max))

    def diversify(self, seed_bits, t0: int, k_local: int, rank: int = 0, world: int = 1):
        self._ck(self.lib.ubqp_diversify(self.h, _ptr(seed_bits), t0, k_local, rank, world))

    def blend(self, seed_bits, parents, n_parents: int, t0: int, k_local: int, rank: int = 0, world: int = 1):
        self._ck(self.lib.ubqp_blend(self.h, _ptr(seed_bits), _ptr(parents), n_parents, t0, k_local, rank, world))

    def random(self, seed: int, k_local: int, rank: int = 0, world: int = 1):
        self._ck(self.lib.ubqp_random(self.h, seed & (2**64 - 1), k_local, rank, world))

    def set_batch(self, bits, k_local: int, rank: int = 0, world: int = 1):
        self._ck(self.lib.ubqp_set_batch(self.h, _ptr(bits), k_local, rank, world))

    def first_derivative(self, bits_out):
        self._ck(self.lib.ubqp_first_derivative(self.h, _ptr(bits_out)))

    def get_batch(self, bits_out):
        self._ck(self.lib.ubqp_get_batch(self.h, _ptr(bits_out)))

    def eval_batch(self, flags: int = 0, f_out=None, stats_out=None):
        self._ck(self.lib.ubqp_eval_batch(self.h, flags, _ptr(f_out), _ptr(stats_out)))

    def get_gains(self, slot0: int, count: int, gains_out):
        self._ck(self.lib.ubqp_get_gains(self.h, slot0, count, _ptr(gains_out)))

    def screen(self, lam: float, mean_sum: int, mean_count: int, max_value: int, surv_out):
        m = ctypes.c_int64()
        T = ctypes.c_double()
        self._ck(self.lib.ubqp_screen(self.h, float(lam), int(mean_sum), int(mean_count), int(max_value),
                                      _ptr(surv_out), ctypes.byref(m), ctypes.byref(T)))
        return m.value, T.value

    def ascend(self, slots, m: int, max_flips: int, f_out=None, flips_out=None, bits_out=None,
               best_key_out=None):
        self._ck(self.lib.ubqp_ascend(self.h, _ptr(slots), m, max_flips, _ptr(f_out), _ptr(flips_out),
                                      _ptr(bits_out), _ptr(best_key_out)))

    def relink(self, guides, n_guides: int, slots, m: int, f_out=None, step_out=None, len_out=None,
               bits_out=None, best_key_out=None):
        self._ck(self.lib.ubqp_relink(self.h, _ptr(guides), n_guides, _ptr(slots), m, _ptr(f_out),
                                      _ptr(step_out), _ptr(len_out), _ptr(bits_out), _ptr(best_key_out)))

    # ---- real-valued Q (a4')
    def load_Q_real(self, Q, k_max: int):
        if isinstance(Q, np.ndarray):
            dt = UBQP_F32 if Q.dtype == np.float32 else UBQP_F64
            Q = np.ascontiguousarray(Q, dtype=np.float32 if dt == UBQP_F32 else np.float64)
        else:
            import torch
            dt = UBQP_F32 if Q.dtype == torch.float32 else UBQP_F64
        self._ck(self.lib.ubqp_load_Q_real(self.h, Q.shape[0], dt, _ptr(Q), k_max))

    @property
    def real_exp(self) -> int:
        """exponent e of the walk image Qt = rint(Q 2^e) (R20)"""
        return self.query(Q_REAL_EXP)

    @property
    def eval_exp(self) -> int:
        """exponent w of the evaluation image (R22)"""
        return self.query(Q_EVAL_EXP)

    @property
    def shard_block(self) -> int:
        return self.query(Q_SHARD_BLOCK)

    @property
    def eval_limbs(self) -> int:
        return self.query(Q_EVAL_LIMBS)

    def set_option(self, what: int, value: int):
        self._ck(self.lib.ubqp_set_option(self.h, what, int(value)))

    def eval_batch_real(self, f_out=None, stats_out=None):
        self._ck(self.lib.ubqp_eval_batch_real(self.h, _ptr(f_out), _ptr(stats_out)))

    def screen_real(self, lam: float, mean: float, max_value: float, surv_out):
        m = ctypes.c_int64()
        T = ctypes.c_double()
        self._ck(self.lib.ubqp_screen_real(self.h, float(lam), float(mean), float(max_value), _ptr(surv_out),
                                           ctypes.byref(m), ctypes.byref(T)))
        return m.value, T.value

    def ascend_real(self, slots, m: int, max_flips: int, f_out=None, fint_out=None, flips_out=None, bits_out=None):
        self._ck(self.lib.ubqp_ascend_real(self.h, _ptr(slots), m, max_flips, _ptr(f_out), _ptr(fint_out),
                                           _ptr(flips_out), _ptr(bits_out)))

    def sync(self):
        self._ck(self.lib.ubqp_sync(self.h))
