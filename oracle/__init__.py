"""CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_2511_20317_b200``) never imports it.  See ``oracle/oracle.h``.
"""
from .oracle import Oracle, OracleParams, build_oracle, ORACLE_SO  # noqa: F401
