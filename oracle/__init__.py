"""ORACLE — CPU test infrastructure for the fused-region path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the reported CPU baseline.  The product package never imports it.
"""
