"""Cooperative row family (K3): one thread group per long row, row in registers.

Filled in by the row-normalise work; ``try_generate`` returns None when the
region does not qualify, and the thread-per-row family handles it.
"""

from __future__ import annotations


def try_generate(region):
    return None
