"""Oracle: adaptive sampling — dedup, k-means++, Lloyd, knee, mode vote (TEST INFRASTRUCTURE ONLY).

Restates ``knobtuner/sampler.py`` at array level:

* ``distinct_rows``   <- sampler.py:187-192  (first-occurrence dedup of trajectory configs)
* ``plus_plus_init``  <- sampler.py:56-69    (seeded k-means++ starts)
* ``kmeans``          <- sampler.py:72-122   (Lloyd, ties -> lowest cluster, empty-cluster reseed)
* ``knee_scan``       <- sampler.py:125-148  (k = 8.. until knee_constant * L_k > L_{k-1})
* ``mode_vote``       <- sampler.py:151-158  (per-knob bincount argmax, ties -> smallest)
* ``round_centroid``  <- sampler.py:161-170  (floor(x + 0.5), clamped)
* ``adaptive_sample`` <- sampler.py:173-215  (batch assembly with visited/mode replacement)

Inputs are (N, n) integer index matrices and a set of visited index tuples;
outputs are index tuples.  The floating-point expressions are the ones whose
rounding the reference's results depend on (per-row pairwise d^2, pairwise
1-D loss sums, exact integer k-means++ weights), so this module is bit-exact
with the reference — pinned by ``tests/golden``.
"""

from __future__ import annotations

import numpy as np

KNEE_CONSTANT = 1.1
KNEE_K_MIN = 8
KNEE_K_MAX = 63
LLOYD_MAX_ITERS = 100


def seeded_generator(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(int(seed) & (2**64 - 1)))


def distinct_rows(idx: np.ndarray) -> np.ndarray:
    """Distinct rows of ``idx`` in order of first occurrence."""
    idx = np.asarray(idx)
    if idx.shape[0] == 0:
        return idx.copy()
    _, first = np.unique(idx, axis=0, return_index=True)
    return idx[np.sort(first)]


def _sq_dist(points: np.ndarray, c: np.ndarray) -> np.ndarray:
    # per-row sum over the contiguous knob axis: numpy pairwise order
    diff = points - c[None, :]
    return (diff**2).sum(axis=1)


def plus_plus_init(points: np.ndarray, k: int, rng: np.random.Generator) -> np.ndarray:
    m = points.shape[0]
    chosen = np.empty((k, points.shape[1]), dtype=np.float64)
    pick = int(rng.integers(0, m))
    chosen[0] = points[pick]
    weight = _sq_dist(points, chosen[0])
    for j in range(1, k):
        target = rng.random() * float(weight.sum())
        pick = min(int(np.searchsorted(np.cumsum(weight), target, side="right")), m - 1)
        chosen[j] = points[pick]
        weight = np.minimum(weight, _sq_dist(points, chosen[j]))
    return chosen


def kmeans(points, k: int, seed: int, max_iters: int = LLOYD_MAX_ITERS) -> dict:
    """Returns {"centroids", "assignment", "loss", "history"} like ClusteringResult."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    if pts.size == 0:
        raise ValueError("kmeans needs at least one point")
    m = pts.shape[0]
    n_distinct = distinct_rows(pts).shape[0]
    if not 1 <= k <= n_distinct:
        raise ValueError(f"k={k} out of range [1, {n_distinct}] for {m} points ({n_distinct} distinct)")
    centroids = plus_plus_init(pts, k, seeded_generator(seed))

    assignment = np.full(m, -1, dtype=np.int64)
    history: list[float] = []
    for it in range(max_iters):
        dist = np.empty((m, k), dtype=np.float64)
        for j in range(k):
            dist[:, j] = _sq_dist(pts, centroids[j])
        fresh = dist.argmin(axis=1)
        own = dist[np.arange(m), fresh]
        history.append(float(own.sum()))
        if np.array_equal(fresh, assignment):
            break
        assignment = fresh
        if it == max_iters - 1:
            break
        counts = np.bincount(assignment, minlength=k)
        for j in np.flatnonzero(counts):
            centroids[j] = pts[assignment == j].mean(axis=0)
        empty = np.flatnonzero(counts == 0)
        if empty.size:
            far_first = np.argsort(-own, kind="stable")
            used: set[int] = set()
            cursor = 0
            for j in empty:
                while int(far_first[cursor]) in used:
                    cursor += 1
                used.add(int(far_first[cursor]))
                centroids[int(j)] = pts[int(far_first[cursor])]
    return {
        "centroids": centroids,
        "assignment": assignment,
        "loss": history[-1],
        "history": tuple(history),
    }


def knee_scan(points, seed: int, knee_constant: float = KNEE_CONSTANT, k_max: int = KNEE_K_MAX):
    """Returns (result of the breaking / last k, [(k, loss), ...])."""
    pts = np.asarray(points, dtype=np.float64)
    upper = min(k_max, distinct_rows(pts).shape[0])
    previous = np.inf
    curve: list[tuple[int, float]] = []
    result = None
    for k in range(KNEE_K_MIN, upper + 1):
        result = kmeans(pts, k, seed)
        curve.append((k, result["loss"]))
        if knee_constant * result["loss"] > previous:
            break
        previous = result["loss"]
    return result, curve


def mode_vote(idx: np.ndarray, cards) -> tuple[int, ...]:
    idx = np.asarray(idx, dtype=np.int64)
    return tuple(int(np.bincount(idx[:, d], minlength=int(c)).argmax()) for d, c in enumerate(cards))


def round_centroid(centroid: np.ndarray, cards) -> tuple[int, ...]:
    out = []
    for x, c in zip(np.asarray(centroid, dtype=np.float64), cards):
        out.append(min(max(int(np.floor(x + 0.5)), 0), int(c) - 1))
    return tuple(out)


def adaptive_sample(idx: np.ndarray, visited: set, cards, seed: int,
                    knee_constant: float = KNEE_CONSTANT, return_info: bool = False):
    """Batch (list of index tuples) for one round's trajectory matrix ``idx``."""
    idx = np.asarray(idx, dtype=np.int64)
    uniq = distinct_rows(idx)
    info: dict = {"m": int(uniq.shape[0])}
    if uniq.shape[0] <= KNEE_K_MIN:
        batch = [t for t in map(tuple, uniq.tolist()) if t not in visited]
        return (batch, info) if return_info else batch
    result, curve = knee_scan(uniq.astype(np.float64), seed, knee_constant)
    info.update(curve=curve, result=result)
    batch, info["mode"] = assemble_batch(result["centroids"], idx, visited, cards)
    return (batch, info) if return_info else batch


def assemble_batch(centroids, idx: np.ndarray, visited: set, cards):
    """Batch assembly of sampler.py:200-215: round each centroid; a visited one is replaced by the
    trajectory's mode (computed once, lazily); visited modes and repeats are dropped.
    Returns (batch, mode or None when the mode vote never ran)."""
    batch: list[tuple[int, ...]] = []
    taken: set = set()
    mode = None
    for centroid in centroids:
        cand = round_centroid(centroid, cards)
        if cand in visited:
            if mode is None:
                mode = mode_vote(idx, cards)
            cand = mode
            if cand in visited:
                continue
        if cand in taken:
            continue
        taken.add(cand)
        batch.append(cand)
    return batch, mode
