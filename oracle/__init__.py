"""CPU oracle for the FPE hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2211_06320_b200`` never imports it and shares no code
with it.  See ``oracle/fpe_oracle.c`` for what is computed and which
PAPER.md passages each step follows.
"""
from .oracle import (  # noqa: F401
    NEG_INF_SCALE,
    OraclePoly,
    build,
    drop_for,
    hull,
    lam,
    lib,
    scale,
    scales,
)
