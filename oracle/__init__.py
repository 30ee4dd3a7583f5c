"""CPU oracle for the UBQP hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path in ``paper_1706_00037_b200/``.  See ``oracle/ubqp_oracle.c`` for the
definitions (O1..O10) and their citations into PAPER.md.
"""
from .oracle import *  # noqa: F401,F403
