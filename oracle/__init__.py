"""CPU oracle for the MBS hot path — TEST INFRASTRUCTURE ONLY.

Importable only by ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` leg, as the checker or the timed CPU
baseline. Never imported by the product package. Parity is pinned against the
real reference (``tests/golden/``), see ``mbs_oracle.py``.
"""
