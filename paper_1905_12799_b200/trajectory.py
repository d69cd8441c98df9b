"""Array-backed search trajectory (drop-in for knobtuner.agent.Trajectory, agent.py:100-127).

A search round on the B200 produces its trajectory as device arrays (packed
rows, float64 scores, step indices).  Building a million ``Configuration``
objects costs seconds in Python (SURVEY §7 hard part 4), so ``entries`` and
``configs()`` are materialised lazily, only when a pure-Python consumer
(e.g. report.per_step_best) touches them; the engine's own consumers
(``adaptive_sample``, ``_top_unvisited``) read the arrays directly.
"""

from __future__ import annotations

import numpy as np

from . import space as sp


class Trajectory:
    def __init__(self, rows, scores, step_indices=None, n_knobs: int = 0, config_cls=sp.Configuration, cards=None):
        if int(rows.shape[0]) == 0:
            raise ValueError("trajectory is empty")
        if int(scores.shape[0]) != int(rows.shape[0]):
            raise ValueError("rows and scores disagree on length")
        if step_indices is not None and int(step_indices.shape[0]) != int(rows.shape[0]):
            raise ValueError(
                f"step_indices length {int(step_indices.shape[0])} does not match {int(rows.shape[0])} entries")
        self._rows = rows  # torch int64 (device or host) or numpy uint64/int64
        self._scores = scores
        self._steps = step_indices
        self.n_knobs = int(n_knobs)
        self.cards = None if cards is None else np.asarray(cards, dtype=np.int64)  # row layout (space.row_layout)
        self.config_cls = config_cls
        self._entries = None

    # -------------------------------------------------------------- arrays
    def rows_numpy(self) -> np.ndarray:
        r = self._rows
        if hasattr(r, "detach"):
            r = r.detach().cpu().numpy()
        return np.ascontiguousarray(r).view(np.uint64)

    def rows_device(self, device: int):
        import torch

        r = self._rows
        if isinstance(r, torch.Tensor):
            if r.is_cuda and r.device.index == device:
                return r
            return r.to(f"cuda:{device}")
        t = torch.from_numpy(np.ascontiguousarray(r).view(np.int64))
        return t.to(f"cuda:{device}")

    def scores_device(self):
        return self._scores

    def index_matrix(self) -> np.ndarray:
        return sp.unpack(self.rows_numpy(), self.n_knobs, self.cards)

    # --------------------------------------------------- reference interface
    @property
    def step_indices(self):
        if self._steps is None:
            return None
        s = self._steps
        if hasattr(s, "detach"):
            s = s.detach().cpu().numpy()
        return tuple(int(x) for x in np.asarray(s).tolist())

    @property
    def entries(self):
        if self._entries is None:
            scores = self.scores()
            self._entries = tuple(
                (self.config_cls(tuple(r)), float(s)) for r, s in zip(self.index_matrix().tolist(), scores.tolist()))
        return self._entries

    def configs(self) -> list:
        if self._entries is not None:
            return [c for c, _ in self._entries]
        return [self.config_cls(tuple(r)) for r in self.index_matrix().tolist()]

    def scores(self) -> np.ndarray:
        s = self._scores
        if hasattr(s, "detach"):
            s = s.detach().cpu().numpy()
        return np.asarray(s, dtype=np.float64)

    def __len__(self) -> int:
        return int(self._rows.shape[0])


def trajectory_rows(trajectory, space, device: int):
    """Device rows (torch int64) of any trajectory: ours (zero-copy) or the reference's."""
    if isinstance(trajectory, Trajectory):
        return trajectory.rows_device(device)
    import torch

    rows = sp.rows_from_configs(space, trajectory.configs())
    return torch.from_numpy(rows.view(np.int64)).to(f"cuda:{device}")


def config_class_of(trajectory):
    if isinstance(trajectory, Trajectory):
        return trajectory.config_cls
    entries = getattr(trajectory, "entries", None)
    if entries:
        return type(entries[0][0])
    return sp.Configuration
