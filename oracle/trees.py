"""Oracle: boosted-tree surrogate scoring (TEST INFRASTRUCTURE ONLY).

Restates the scoring half of ``knobtuner/cost_model.py``:

* ``feature_table``     <- cost_model.py:235-249  (log2(1 + knob value) lookup)
* ``featurize_rows``    <- cost_model.py:252-261  (index matrix -> feature matrix)
* ``predict_features``  <- cost_model.py:181-201  (base + sum of one leaf per tree)

Models are handled in the reference's JSON document form
(``CostModel.to_json``, cost_model.py:203-218): ``{"base_score", "feature_count",
"trees": [nested {"feature","threshold","left","right"} | {"value"}]}``.

Summation order (pinned against reference goldens): the per-tree leaf values
are accumulated sequentially in tree order (numpy's axis-0 ``sum`` of the
(trees, rows) matrix), and the base score is added last.
"""

from __future__ import annotations

import numpy as np


def feature_table(knob_values: list[list[int]]) -> tuple[np.ndarray, np.ndarray]:
    """(n, max_card) table of log2(1 + value) and per-knob negative-prefix counts."""
    width = max(len(v) for v in knob_values)
    table = np.zeros((len(knob_values), width), dtype=np.float64)
    negatives = np.zeros(len(knob_values), dtype=np.int64)
    for row, vals in enumerate(knob_values):
        arr = np.asarray(vals, dtype=np.float64)
        negatives[row] = int(np.count_nonzero(arr < 0))
        with np.errstate(invalid="ignore", divide="ignore"):
            table[row, : arr.size] = np.log2(1.0 + arr)
    return table, negatives


def featurize_rows(knob_values: list[list[int]], idx: np.ndarray) -> np.ndarray:
    """Feature matrix for an (N, n) index matrix; rejects negative knob settings."""
    idx = np.asarray(idx, dtype=np.int64)
    table, negatives = feature_table(knob_values)
    if idx.shape[0] and (idx < negatives[None, :]).any():
        raise ValueError("featurize requires non-negative knob values")
    n = len(knob_values)
    return table[np.arange(n)[None, :], idx]


def _route(node: dict, X: np.ndarray, rows: np.ndarray, out: np.ndarray) -> None:
    if "value" in node:
        out[rows] = float(node["value"])
        return
    goes_left = X[rows, int(node["feature"])] <= float(node["threshold"])
    _route(node["left"], X, rows[goes_left], out)
    _route(node["right"], X, rows[~goes_left], out)


def predict_features(model: dict, X: np.ndarray) -> np.ndarray:
    """Surrogate score per feature row (cost_model.py:181-201)."""
    X = np.asarray(X, dtype=np.float64)
    N = X.shape[0]
    base = float(model["base_score"])
    trees = model["trees"]
    if not trees or N == 0:
        return np.full(N, base, dtype=np.float64)
    acc = None
    leaf = np.empty(N, dtype=np.float64)
    all_rows = np.arange(N)
    for tree in trees:
        _route(tree, X, all_rows, leaf)
        if acc is None:
            acc = leaf.copy()
        else:
            acc += leaf
    return np.full(N, base, dtype=np.float64) + acc


def tree_depth(node: dict) -> int:
    if "value" in node:
        return 0
    return 1 + max(tree_depth(node["left"]), tree_depth(node["right"]))
