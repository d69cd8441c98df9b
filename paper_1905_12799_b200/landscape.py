"""Synthetic landscape scoring on the B200 (K3) — drop-in for the landscape half of
knobtuner/backends.py (backends.py:123-273).

``synthetic_runtime(landscape, config)`` / ``true_fitness`` keep the reference
signatures; ``batch_runtimes`` / ``runtimes_rows`` are the batched engine
paths (used by ``SyntheticBackend`` and the brute-force optimum search).
Landscapes may be the reference's ``SyntheticLandscape`` or its JSON document.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import space as sp


@dataclass(frozen=True)
class SyntheticLandscape:
    """Mirror of backends.py:123-154 (validation included)."""

    seed: int
    space: object
    centers: tuple
    depths: tuple
    radii: tuple
    base_runtime: float = 1.0
    noise_rel: float = 0.0

    def __post_init__(self) -> None:
        if not (len(self.centers) == len(self.depths) == len(self.radii)):
            raise ValueError("centers, depths, and radii must have equal lengths")
        for c in self.centers:
            if len(c) != len(self.space.knobs):
                raise ValueError(f"center {c} does not match the {len(self.space.knobs)}-knob space")
        if any(d <= 0 for d in self.depths) or sum(self.depths) >= 1.0:
            raise ValueError("depths must be positive and sum below 1")
        if any(r <= 0 for r in self.radii):
            raise ValueError("radii must be positive")
        if self.base_runtime <= 0:
            raise ValueError("base_runtime must be positive")
        if not 0.0 <= self.noise_rel < 1.0:
            raise ValueError(f"noise_rel must be in [0, 1), got {self.noise_rel}")


def landscape_from_dict(obj: dict, space) -> SyntheticLandscape:
    return SyntheticLandscape(seed=int(obj["seed"]), space=space,
                              centers=tuple(tuple(int(v) for v in c) for c in obj["centers"]),
                              depths=tuple(float(d) for d in obj["depths"]),
                              radii=tuple(float(r) for r in obj["radii"]),
                              base_runtime=float(obj["base_runtime"]), noise_rel=float(obj["noise_rel"]))


def load_landscape(path, space) -> SyntheticLandscape:
    with open(path, encoding="utf-8") as fh:
        return landscape_from_dict(json.load(fh), space)


class DeviceLandscape:
    def __init__(self, landscape, engine: _lib.Engine):
        n = len(landscape.space.knobs)
        cards = sp.check_engine_space(landscape.space)
        centers = np.ascontiguousarray(np.asarray(landscape.centers, dtype=np.int32).reshape(-1, n))
        depths = np.ascontiguousarray(np.asarray(landscape.depths, dtype=np.float64))
        radii = np.ascontiguousarray(np.asarray(landscape.radii, dtype=np.float64))
        h = _lib.P()
        _lib.call("kt_landscape_create", engine.handle, n, _lib.as_ptr(cards, _lib.C.c_int32), int(centers.shape[0]),
                  _lib.as_ptr(centers, _lib.C.c_int32), _lib.as_ptr(depths, _lib.C.c_double),
                  _lib.as_ptr(radii, _lib.C.c_double), float(landscape.base_runtime), float(landscape.noise_rel),
                  str(landscape.seed).encode("ascii"), _lib.C.byref(h))
        self.handle = h

    def __del__(self):
        try:
            _lib.load().kt_landscape_destroy(self.handle)
        except Exception:
            pass


def device_landscape(landscape, engine: _lib.Engine | None = None) -> DeviceLandscape:
    engine = engine or _lib.engine()
    cache = getattr(landscape, "__dict__", {}).get("_b200_landscape")
    if cache is None:
        cache = {}
        try:
            object.__setattr__(landscape, "_b200_landscape", cache)
        except (AttributeError, TypeError):
            pass
    d = cache.get(engine.device)
    if d is None:
        d = DeviceLandscape(landscape, engine)
        cache[engine.device] = d
    return d


def runtimes_rows(landscape, rows, out=None, engine: _lib.Engine | None = None):
    """Device path: CUDA int64 rows -> CUDA float64 runtimes."""
    import torch

    engine = engine or _lib.engine()
    d = device_landscape(landscape, engine)
    n = int(rows.numel())
    with engine.scope():
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=rows.device)
        _lib.call("kt_score_landscape", engine.handle, d.handle, _lib.ptr(rows), n, _lib.ptr(out))
    return out


def batch_runtimes(landscape, configs) -> list[float]:
    import torch

    if not configs:
        return []
    engine = _lib.engine()
    rows = sp.rows_from_configs(landscape.space, configs)
    with engine.scope():
        t = torch.from_numpy(rows.view(np.int64)).to(f"cuda:{engine.device}")
    return runtimes_rows(landscape, t, engine=engine).cpu().numpy().tolist()


def synthetic_runtime(landscape, config) -> float:
    """backends.py:164-174, one configuration."""
    return batch_runtimes(landscape, [config])[0]


def true_fitness(landscape, config) -> float:
    return 1.0 / synthetic_runtime(landscape, config)


class SyntheticBackend:
    """Pure-function backend over a landscape (backends.py:263-273), scored on the B200."""

    tag = "synthetic"

    def __init__(self, landscape):
        self.landscape = landscape
        self.space = landscape.space

    def batch_runtimes(self, configs) -> list[float]:
        return batch_runtimes(self.landscape, list(configs))


def best_runtime(landscape):
    """Brute-force optimum over the whole lattice (cli.py:77-90 ``_enumerated_oracle``, without the
    10^6 cap of ``enumerate_space``, space.py:20), fused on the device: ranks decoded into rows in the
    space's own row layout, scored, reduced to the first minimum (``kt_landscape_best``).

    Returns (min runtime, argmin as an index tuple); the first minimum in ``enumerate_space`` order
    (last knob fastest) wins ties, like the reference's strict ``<`` scan.
    """
    engine = _lib.engine()
    d = device_landscape(landscape, engine)
    cards = sp.check_engine_space(landscape.space)
    best = _lib.C.c_double(0.0)
    rank = _lib.C.c_int64(-1)
    with engine.scope():
        _lib.call("kt_landscape_best", engine.handle, d.handle, _lib.as_ptr(cards, _lib.C.c_int32),
                  _lib.C.byref(best), _lib.C.byref(rank))
    r = int(rank.value)
    idx = []
    for c in reversed(cards.tolist()):
        idx.append(r % c)
        r //= c
    return float(best.value), tuple(reversed(idx))
