"""Adaptive sampling on the B200 — drop-in for knobtuner/sampler.py.

Same names, signatures, error types/messages and (bit-exact) results as the
reference module; the work runs in libknobtuner_b200 (csrc/sampler.cu):

* ``adaptive_sample``  (sampler.py:173-215): dedup (K6) -> knee k-means (K7/K8)
  -> batch assembly, in one engine call.
* ``kmeans`` / ``knee_scan`` (sampler.py:72-148) on lattice points.
* ``mode_config`` (sampler.py:151-158) via the K9 histogram kernel.
* ``round_to_config`` and ``VisitedSet`` are host bookkeeping (<= 63 rows).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import space as sp
from .trajectory import config_class_of, trajectory_rows

KNEE_CONSTANT = 1.1
KNEE_K_MIN = 8
KNEE_K_MAX = 63
KMEANS_MAX_ITERS = 100


class VisitedSet:
    """Measured configurations by exact index equality (sampler.py:26-45), plus packed rows."""

    def __init__(self, configs=None):
        self._seen: set[tuple[int, ...]] = set()
        for c in configs or []:
            self.add(c)

    def add(self, config) -> None:
        self._seen.add(tuple(config.indices))

    def add_all(self, configs) -> None:
        for c in configs:
            self.add(c)

    def __contains__(self, config) -> bool:
        return tuple(config.indices) in self._seen

    def __len__(self) -> int:
        return len(self._seen)


def visited_rows(visited, cards=None) -> np.ndarray:
    """Packed rows of a VisitedSet (ours or the reference's, whose set is ``_seen``)."""
    seen = getattr(visited, "_seen", None)
    if seen is None:
        raise TypeError("visited set must expose its index tuples (VisitedSet._seen)")
    if not seen:
        return np.zeros(0, dtype=np.uint64)
    return sp.pack(np.array(sorted(seen), dtype=np.int64), cards)


@dataclass(frozen=True)
class ClusteringResult:
    centroids: np.ndarray  # (k, d)
    assignment: np.ndarray  # (m,)
    loss: float
    loss_history: tuple


def _lattice_rows(points: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Engine rows (and the per-dimension extents that fix their layout) for lattice
    points; NotImplementedError for anything else."""
    if points.shape[1] > sp.MAX_KNOBS:
        raise NotImplementedError("engine k-means supports at most 8 dimensions")
    if (not np.all(np.isfinite(points)) or np.any(points != np.round(points)) or points.min() < 0
            or points.max() >= sp.MAX_WIDE_CARD):
        raise NotImplementedError(f"engine k-means runs on lattice points (integer coordinates in "
                                  f"[0, {sp.MAX_WIDE_CARD - 1}])")
    idx = points.astype(np.int64)
    cards = (idx.max(axis=0) + 1).astype(np.int32)
    return sp.pack(idx, cards), cards


def _device_points(points):
    import torch

    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    if pts.size == 0:
        raise ValueError("kmeans needs at least one point")
    rows, cards = _lattice_rows(pts)
    eng = _lib.engine()
    with eng.scope():
        d = torch.from_numpy(rows.view(np.int64)).to(f"cuda:{eng.device}")
    return eng, pts, d, cards


def _n_distinct(eng, d) -> int:
    import torch

    m = int(d.numel())
    with eng.scope():
        scratch = torch.empty(m, dtype=torch.int64, device=d.device)
        out = _lib.C.c_int64(0)
        _lib.call("kt_dedup", eng.handle, _lib.ptr(d), m, _lib.ptr(scratch), _lib.C.byref(out))
    return int(out.value)


def kmeans(points, k: int, seed: int) -> ClusteringResult:
    """Lloyd's algorithm with seeded k-means++ starts (sampler.py:72-122), on the device."""
    eng, pts, d, cards = _device_points(points)
    m, n = pts.shape
    nd = _n_distinct(eng, d)
    if not 1 <= k <= nd:
        raise ValueError(f"k={k} out of range [1, {nd}] for {m} points ({nd} distinct)")
    cent = np.zeros((k, n), dtype=np.float64)
    asg = np.zeros(m, dtype=np.int64)
    hist = np.zeros(KMEANS_MAX_ITERS, dtype=np.float64)
    loss = _lib.C.c_double(0.0)
    passes = _lib.C.c_int32(0)
    with eng.scope():
        _lib.call("kt_kmeans", eng.handle, _lib.ptr(d), m, n, _lib.as_ptr(cards, _lib.C.c_int32), int(k),
                  int(seed) & (2**64 - 1),
                  _lib.as_ptr(cent, _lib.C.c_double), _lib.as_ptr(asg, _lib.C.c_int64), _lib.C.byref(loss),
                  _lib.as_ptr(hist, _lib.C.c_double), _lib.C.byref(passes))
    return ClusteringResult(centroids=cent, assignment=asg, loss=float(loss.value),
                            loss_history=tuple(float(x) for x in hist[: passes.value]))


def knee_scan(points, seed: int, knee_constant: float = KNEE_CONSTANT, k_max: int = KNEE_K_MAX):
    """Grow k from 8 until knee_constant * Loss(k) > previous loss (sampler.py:125-148)."""
    eng, pts, d, cards = _device_points(points)
    m, n = pts.shape
    ks = np.zeros(56, dtype=np.int32)
    ls = np.zeros(56, dtype=np.float64)
    cnt = _lib.C.c_int32(0)
    cent = np.zeros((64, n), dtype=np.float64)
    nd = _n_distinct(eng, d)
    if min(k_max, nd) < KNEE_K_MIN:
        raise AssertionError("knee_scan needs at least 8 distinct points")
    # the scan itself runs on the distinct points in first-occurrence order only
    # when they are already distinct; duplicates are valid k-means input too
    with eng.scope():
        _lib.call("kt_knee_scan", eng.handle, _lib.ptr(d), m, n, _lib.as_ptr(cards, _lib.C.c_int32),
                  int(seed) & (2**64 - 1), float(knee_constant),
                  int(min(k_max, nd)), _lib.as_ptr(ks, _lib.C.c_int32), _lib.as_ptr(ls, _lib.C.c_double),
                  _lib.C.byref(cnt), _lib.as_ptr(cent, _lib.C.c_double), None)
    scanned = [(int(ks[i]), float(ls[i])) for i in range(cnt.value)]
    # the chosen k's full result (assignment + loss history) as the reference returns it
    result = kmeans(pts, scanned[-1][0], seed)
    return result, scanned


def mode_config(trajectory, space):
    """Per-knob most frequent index over the trajectory; ties take the smallest (sampler.py:151-158)."""
    eng = _lib.engine()
    cards = sp.check_engine_space(space)
    rows = trajectory_rows(trajectory, space, eng.device)
    out = np.zeros(sp.MAX_KNOBS, dtype=np.int32)
    with eng.scope():
        _lib.call("kt_mode_vote", eng.handle, _lib.ptr(rows), int(rows.numel()), len(space.knobs),
                  _lib.as_ptr(cards, _lib.C.c_int32),
                  _lib.as_ptr(out, _lib.C.c_int32))
    return config_class_of(trajectory)(tuple(int(v) for v in out[: len(space.knobs)]))


def round_to_config(centroid, space):
    """Nearest lattice point; .5 rounds up, out-of-range clamps (sampler.py:161-170)."""
    centroid = np.asarray(centroid, dtype=np.float64)
    if centroid.shape != (len(space.knobs),):
        raise ValueError(f"centroid shape {centroid.shape} does not match {len(space.knobs)} knobs")
    out = []
    for x, card in zip(centroid, space.cardinalities):
        out.append(min(max(int(np.floor(x + 0.5)), 0), card - 1))
    return sp.Configuration(tuple(out))


def adaptive_sample_rows(rows, visited, space, seed: int, knee_constant: float = KNEE_CONSTANT,
                         engine=None, info: _lib.SampleInfo | None = None) -> np.ndarray:
    """Array path: device rows (torch int64) -> batch rows (numpy uint64)."""
    eng = engine or _lib.engine()
    cards = sp.check_engine_space(space)
    vis = visited if isinstance(visited, np.ndarray) else visited_rows(visited, cards)
    vis = np.ascontiguousarray(vis, dtype=np.uint64)
    batch = np.zeros(64, dtype=np.uint64)
    blen = _lib.C.c_int32(0)
    info = info if info is not None else _lib.SampleInfo()
    with eng.scope():
        _lib.call("kt_adaptive_sample", eng.handle, _lib.ptr(rows), int(rows.numel()), int(cards.size),
                  _lib.as_ptr(cards, _lib.C.c_int32), _lib.as_ptr(vis, _lib.C.c_uint64), int(vis.size),
                  int(seed) & (2**64 - 1), float(knee_constant), _lib.as_ptr(batch, _lib.C.c_uint64),
                  _lib.C.byref(blen), _lib.C.byref(info))
    return batch[: blen.value].copy()


def adaptive_sample(trajectory, visited, space, seed: int, knee_constant: float = KNEE_CONSTANT) -> list:
    """Pick the measurement batch for a round from its trajectory (sampler.py:173-215)."""
    eng = _lib.engine()
    rows = trajectory_rows(trajectory, space, eng.device)
    batch = adaptive_sample_rows(rows, visited, space, seed, knee_constant, engine=eng)
    cls = config_class_of(trajectory)
    return [cls(tuple(r)) for r in sp.unpack(batch, len(space.knobs), sp.cardinalities(space)).tolist()]
