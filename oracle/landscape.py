"""Oracle: synthetic landscape ("fake hardware") scoring (TEST INFRASTRUCTURE ONLY).

Restates ``knobtuner/backends.py``:

* ``hash_unit``          <- backends.py:157-161 (blake2b-64 of "seed:i0,i1,..." -> [-1, 1])
* ``synthetic_runtimes`` <- backends.py:164-174 (Gaussian basins x hash noise, clamped)

Scalar ``math.exp`` is used (not ``np.exp``) so the oracle rounds exactly like the
reference; the squared distances are integers, so their summation order is moot.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np


def hash_unit(seed: int, indices) -> float:
    text = str(seed) + ":" + ",".join(str(int(i)) for i in indices)
    word = int.from_bytes(hashlib.blake2b(text.encode("ascii"), digest_size=8).digest(), "big")
    return 2.0 * (word / 2.0**64) - 1.0


def synthetic_runtimes(landscape: dict, idx: np.ndarray) -> np.ndarray:
    """Runtime per row of an (N, n) index matrix.

    ``landscape`` uses the reference's document keys (backends.py:181-189):
    seed, centers, depths, radii, base_runtime, noise_rel.
    """
    idx = np.asarray(idx, dtype=np.int64)
    base = float(landscape["base_runtime"])
    noise = float(landscape["noise_rel"])
    N = idx.shape[0]
    depth_term = np.zeros(N, dtype=np.float64)
    for center, depth, radius in zip(landscape["centers"], landscape["depths"], landscape["radii"]):
        diff = idx - np.asarray(center, dtype=np.int64)[None, :]
        d2 = (diff * diff).sum(axis=1)  # exact integers
        r2 = float(radius) * float(radius)
        cache: dict[int, float] = {}
        contrib = np.empty(N, dtype=np.float64)
        for row, v in enumerate(d2.tolist()):
            e = cache.get(v)
            if e is None:
                e = float(depth) * math.exp(-float(v) / r2)
                cache[v] = e
            contrib[row] = e
        depth_term += contrib
    runtime = base * (1.0 - depth_term)
    if noise > 0.0:
        seed = int(landscape["seed"])
        u = np.array([hash_unit(seed, row) for row in idx.tolist()], dtype=np.float64)
        runtime = runtime * (1.0 + noise * u)
    return np.maximum(runtime, 0.01 * base)
