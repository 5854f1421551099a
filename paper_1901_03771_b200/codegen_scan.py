"""Map-scan and keyed-sum families (placeholders until implemented)."""

from __future__ import annotations

from .errors import UnsupportedNodeInFusedStep


def generate(region):
    raise UnsupportedNodeInFusedStep("scan / bincount kernels are not implemented yet")
