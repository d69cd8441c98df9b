"""Simulated-annealing chains on the B200 (K10) — drop-in for knobtuner/sa.py.

``run_sa_round(params, model, space, starts, seed)`` keeps the reference's
signature, validation, padding, RNG streams and chain-major output
(sa.py:62-122); every chain runs all its steps inside one kernel with the
surrogate forest in shared memory (csrc/sa.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import space as sp
from .cost_model import _check_model, device_forest
from .trajectory import Trajectory


@dataclass(frozen=True)
class SAParams:
    chains: int = 64
    steps_per_round: int = 128
    initial_temperature: float | None = None
    cooling: float = 0.99

    def __post_init__(self) -> None:
        if self.chains < 1:
            raise ValueError(f"chains must be >= 1, got {self.chains}")
        if self.steps_per_round < 1:
            raise ValueError(f"steps_per_round must be >= 1, got {self.steps_per_round}")
        if self.initial_temperature is not None and not self.initial_temperature > 0:
            raise ValueError(f"initial_temperature must be > 0, got {self.initial_temperature}")
        if not 0.0 < self.cooling <= 1.0:
            raise ValueError(f"cooling must be in (0, 1], got {self.cooling}")


def seed_words(seed: int) -> np.ndarray:
    """Little-endian uint32 words of seed & (2^64 - 1) (numpy _int_to_uint32_array)."""
    s = int(seed) & (2**64 - 1)
    words = [s & 0xFFFFFFFF] if s < 2**32 else [s & 0xFFFFFFFF, s >> 32]
    return np.array(words, dtype=np.uint32)


def run_sa_rows(params, model, space, start_rows, seed: int, engine=None):
    """Array path: CUDA int64 start rows -> (rows, scores, step indices) CUDA tensors, chain-major."""
    import torch

    engine = engine or _lib.engine()
    _check_model(model, space)
    cards = sp.check_engine_space(space)
    f = device_forest(model, space, engine)
    if f.neg_prefix.any():
        raise ValueError("featurize requires non-negative knob values")
    cap = params.chains * (params.steps_per_round + 1)
    words = seed_words(seed)
    total = _lib.C.c_int64(0)
    with engine.scope():
        dev = start_rows.device
        rows = torch.empty(cap, dtype=torch.int64, device=dev)
        scores = torch.empty(cap, dtype=torch.float64, device=dev)
        steps = torch.empty(cap, dtype=torch.int32, device=dev)
        has_t = params.initial_temperature is not None
        _lib.call("kt_sa_chains", engine.handle, f.handle, _lib.ptr(start_rows), int(start_rows.numel()),
                  int(params.chains), int(params.steps_per_round), _lib.as_ptr(cards, _lib.C.c_int32),
                  int(cards.size), _lib.as_ptr(words, _lib.C.c_uint32), int(words.size), int(has_t),
                  float(params.initial_temperature) if has_t else 0.0, float(params.cooling), _lib.ptr(rows),
                  _lib.ptr(scores), _lib.ptr(steps), _lib.C.byref(total))
    n = int(total.value)
    return rows[:n], scores[:n], steps[:n]


def run_sa_round(params, model, space, starts, seed: int):
    """Metropolis chains on the surrogate; returns starts plus accepted moves (sa.py:62-122)."""
    import torch

    if not starts:
        raise ValueError("run_sa_round needs at least one start configuration")
    idx = sp.index_matrix(space, starts)  # validate_config on every start (sa.py:76-77)
    engine = _lib.engine()
    used = idx[: params.chains]
    with engine.scope():
        start_rows = torch.from_numpy(sp.pack(used, sp.cardinalities(space)).view(np.int64)).to(f"cuda:{engine.device}")
    rows, scores, steps = run_sa_rows(params, model, space, start_rows, seed, engine=engine)
    cls = type(starts[0]) if hasattr(starts[0], "indices") else sp.Configuration
    return Trajectory(rows, scores, steps, n_knobs=len(space.knobs), config_cls=cls, cards=sp.cardinalities(space))
