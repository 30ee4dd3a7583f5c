"""B200-native (sm_100a) hot path of Lewis's GPU diversified multi-start for UBQP
(arXiv 1706.00037): Glover diversification -> batched xQx + 1-flip gains on int8
tcgen05 tensor cores -> T(lambda) screen -> batched steepest ascent, behind the C-ABI
of include/ubqp.h (libubqp.so).  See DESIGN.md.
"""
from .ubqp import (EXPORTS, UBQP_EMIT_GAINS, Ubqp, UbqpError, load_library, ubqp_stats,  # noqa: F401
                   ubqp_stats_real)

__all__ = ["Ubqp", "UbqpError", "load_library", "ubqp_stats", "ubqp_stats_real", "UBQP_EMIT_GAINS", "EXPORTS"]
