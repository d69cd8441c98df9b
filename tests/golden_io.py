"""Loaders for the committed golden vectors (produced by tests/golden/make_golden.py)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def npz(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as f:
        return {k: f[k] for k in f.files}


@lru_cache(maxsize=None)
def meta(name: str) -> dict:
    return json.loads((GOLDEN / f"{name}.json").read_text())


def cases(name: str, leaf: str) -> list[str]:
    """Case prefixes in ``name``.npz that have an entry ``<case>/<leaf>``."""
    return sorted(k[: -len(leaf) - 1] for k in npz(name) if k.endswith("/" + leaf))
