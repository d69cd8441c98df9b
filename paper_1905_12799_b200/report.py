"""Trajectory analysis on the B200 — drop-ins for knobtuner/report.py.

* ``per_step_best(trajectory)`` (report.py:53-69): the round's best surrogate score after each search
  step — a device scatter-max per step index (exact), running max on the host.
* ``convergence_steps_for_round(trajectory, window)`` (report.py:72-74) and ``steps_to_convergence``
  (report.py:23-41) on top of it.
* ``pca_project(configs)`` (report.py:227-253): exact int64 index moments on the device -> mean and
  covariance in float64 -> the reference's seeded power iteration (host, 8x8) -> per-row projections
  on the device.  Projections agree with the reference to float64 rounding (its covariance and
  projections go through BLAS, whose summation order is unspecified).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, errors
from . import space as sp

CONVERGENCE_WINDOW = 8  # report.py:14
POWER_TOL = 1e-9
POWER_MAX_ITERS = 1000


def steps_to_convergence(scores, window: int = CONVERGENCE_WINDOW) -> int:
    """report.py:23-41 (host: at most a few hundred steps)."""
    if len(scores) == 0:
        raise ValueError("steps_to_convergence requires at least one step")
    if window < 1:
        raise ValueError("window must be at least 1")
    best = -np.inf
    last = 0
    for i, s in enumerate(scores, start=1):
        if s > best:
            best = float(s)
            last = i
        if i - last >= window:
            return last
    return len(scores)


def per_step_best(trajectory) -> list[float]:
    """report.py:53-69 for our array-backed Trajectory and for the reference's own (which carries
    ``step_indices`` as a tuple and ``scores()`` / ``entries``; install() rebinds this name)."""
    steps = getattr(trajectory, "_steps", None)
    if steps is None:
        steps = getattr(trajectory, "step_indices", None)
    if steps is None:
        raise ValueError("trajectory does not carry step indices")
    import torch

    eng = _lib.engine()
    dev = f"cuda:{eng.device}"
    with eng.scope():
        st = steps if isinstance(steps, torch.Tensor) else torch.as_tensor(np.asarray(steps))
        st = st.to(dev).to(torch.int32)
        sc = trajectory.scores_device() if hasattr(trajectory, "scores_device") else None
        if sc is None:
            host = (trajectory.scores() if hasattr(trajectory, "scores")
                    else [s for _, s in trajectory.entries])
            sc = torch.as_tensor(np.asarray(host, dtype=np.float64))
        sc = sc.to(dev).to(torch.float64)
    cap = int(st.max().item()) + 1
    best = np.zeros(cap, dtype=np.float64)
    hz = C.c_int32(0)
    with eng.scope():
        _lib.call("kt_step_best", eng.handle, _lib.ptr(sc), _lib.ptr(st), int(st.numel()), cap,
                  _lib.as_ptr(best, C.c_double), C.byref(hz))
    return np.maximum.accumulate(best[: hz.value + 1]).tolist()


def convergence_steps_for_round(trajectory, window: int = CONVERGENCE_WINDOW) -> int:
    return steps_to_convergence(per_step_best(trajectory), window=window)


def _power_iterate(matrix: np.ndarray, rng: np.random.Generator) -> tuple[np.ndarray, float]:
    """Dominant unit eigenvector / eigenvalue of a PSD matrix — the reference's seeded
    iteration (report.py:207-224), same draws and stopping rules."""
    v = rng.standard_normal(matrix.shape[0])
    v /= np.linalg.norm(v)
    for _ in range(POWER_MAX_ITERS):
        w = matrix @ v
        norm = np.linalg.norm(w)
        if norm < POWER_TOL:
            break
        w /= norm
        if np.linalg.norm(w - v) < POWER_TOL or np.linalg.norm(w + v) < POWER_TOL:
            v = w
            break
        v = w
    nz = np.nonzero(np.abs(v) > POWER_TOL)[0]
    if nz.size and v[nz[0]] < 0:
        v = -v
    return v, float(v @ matrix @ v)


def pca_project(configs, cards=None) -> list[tuple[float, float]]:
    """Centre index vectors and project onto the top two principal axes (report.py:227-253).
    ``configs``: Configuration objects (or an (N, n) index matrix)."""
    import torch

    if len(configs) < 2:
        raise ValueError("pca_project requires at least 2 configurations")
    idx = np.asarray(configs if isinstance(configs, np.ndarray) else [c.indices for c in configs], dtype=np.int64)
    N, n = idx.shape
    if n < 2:
        raise ValueError("pca_project requires at least 2 knobs")
    cards = np.asarray(cards if cards is not None else idx.max(axis=0) + 1, dtype=np.int32)
    eng = _lib.engine()
    with eng.scope():
        rows = torch.from_numpy(sp.pack(idx, cards).view(np.int64)).to(f"cuda:{eng.device}")
    sums = np.zeros(n, dtype=np.int64)
    gram = np.zeros(n * n, dtype=np.int64)
    with eng.scope():
        _lib.call("kt_pca_moments", eng.handle, _lib.ptr(rows), N, n, _lib.as_ptr(cards, C.c_int32),
                  _lib.as_ptr(sums, C.c_int64), _lib.as_ptr(gram, C.c_int64))
    mean = sums.astype(np.float64) / float(N)  # exact integer sums: numpy's X.mean(axis=0)
    G = gram.reshape(n, n).astype(np.float64)
    cov = (G - float(N) * np.outer(mean, mean)) / float(N - 1)
    if not np.any(np.abs(cov) > 0.0):
        raise errors.DegenerateVarianceError("all configurations identical: covariance is zero")
    rng = np.random.default_rng(0)
    v1, lam1 = _power_iterate(cov, rng)
    v2, _ = _power_iterate(cov - lam1 * np.outer(v1, v1), rng)
    if abs(np.linalg.norm(v2) - 1.0) > 0.5 or abs(v2 @ v1) > 1e-6:  # rank-1 data (report.py:242-249)
        basis = np.eye(n)
        res = basis - np.outer(basis @ v1, v1)
        pick = int(np.argmax(np.linalg.norm(res, axis=1)))
        v2 = res[pick] / np.linalg.norm(res[pick])
        nz = np.nonzero(np.abs(v2) > POWER_TOL)[0]
        if nz.size and v2[nz[0]] < 0:
            v2 = -v2
    mean_c = np.ascontiguousarray(mean)
    a1, a2 = np.ascontiguousarray(v1, dtype=np.float64), np.ascontiguousarray(v2, dtype=np.float64)
    with eng.scope():
        xs = torch.empty(N, dtype=torch.float64, device=rows.device)
        ys = torch.empty(N, dtype=torch.float64, device=rows.device)
        _lib.call("kt_pca_project", eng.handle, _lib.ptr(rows), N, n, _lib.as_ptr(cards, C.c_int32),
                  _lib.as_ptr(mean_c, C.c_double), _lib.as_ptr(a1, C.c_double), _lib.as_ptr(a2, C.c_double),
                  _lib.ptr(xs), _lib.ptr(ys))
    return list(zip(xs.cpu().numpy().tolist(), ys.cpu().numpy().tolist()))
