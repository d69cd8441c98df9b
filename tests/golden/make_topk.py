"""Golden batches of the REFERENCE's _top_unvisited (driver.py:101-115) for kt_top_unvisited.

    python tests/golden/make_topk.py        # writes tests/golden/topk.json

Trajectories with duplicate configurations, quantised scores (many ties), signed zeros, visited
overlap, fewer candidates than the cap and everything visited; sizes 40 .. 60,000 entries.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
CASES = [  # (name, entries, cards, score levels (0 = continuous), visited count, seed)
    ("tiny_all_distinct", 40, [5, 5, 5], 0, 3, 1), ("ties", 2000, [6, 6, 6, 6], 7, 40, 2),
    ("dups_zero", 5000, [4, 4, 3, 3], 3, 100, 3), ("large", 60000, [84, 80, 80, 7, 2, 2, 3, 2], 0, 500, 4),
    ("large_ties", 60000, [30, 30, 30, 3], 11, 2000, 5), ("all_visited", 30, [2, 2], 0, 4, 6),
    ("few_left", 500, [3, 3, 3], 5, 20, 7),
]


def case_inputs(name, n, cards, levels, nvis, seed):
    """(idx, scores, visited idx) of a case, regenerated from its seed (tests import this)."""
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, cards, size=(n, len(cards)))
    if levels:
        scores = (rng.integers(0, levels, size=n) - levels // 2).astype(np.float64)
        scores[rng.random(n) < 0.1] = -0.0
    else:
        scores = rng.standard_normal(n)
    vis_idx = idx[rng.integers(0, n, size=nvis)]
    if name == "all_visited":
        vis_idx = np.indices(cards).reshape(len(cards), -1).T
    return idx, scores, vis_idx


def main() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")  # the reference is imported here only (tests import case_inputs)
    from knobtuner import driver
    from knobtuner.agent import Trajectory
    from knobtuner.sampler import VisitedSet
    from knobtuner.space import Configuration

    out = []
    for case in CASES:
        name = case[0]
        idx, scores, vis_idx = case_inputs(*case)
        tr = Trajectory(entries=tuple((Configuration(tuple(int(v) for v in r)), float(s))
                                      for r, s in zip(idx.tolist(), scores.tolist())))
        visited = VisitedSet([Configuration(tuple(int(v) for v in r)) for r in vis_idx.tolist()])
        batch = driver._top_unvisited(tr, visited, driver.GREEDY_BATCH)
        out.append({"case": list(case), "batch": [list(c.indices) for c in batch]})
        print(name, len(batch))
    (HERE / "topk.json").write_text(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
