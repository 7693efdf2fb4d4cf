"""TEST INFRASTRUCTURE ONLY: CPU oracles for the north-star path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference`` legs) may import this package, and only as the checker
or the timed CPU baseline. The product package ``paper_2012_11077_b200`` never
imports it and has no CPU fallback.
"""
