"""Boosted-tree surrogate scoring on the B200 (K2) — drop-in for the scoring half of
knobtuner/cost_model.py.

* ``CostModel`` / ``Tree``  — mirror of the reference's frozen model types
  (cost_model.py:69-218, JSON format included) so models round-trip.
* ``device_forest(model, space)`` — the model packed for the engine
  (complete-heap trees with integer cut points, see csrc/trees.cu), cached on
  the model object like the reference caches ``_packed_arrays``
  (cost_model.py:157-179).
* ``predict(model, space, configs)`` — same signature, checks, errors and
  bit-exact results as cost_model.py:401-409.
* ``predict_rows(model, space, rows)`` — the array path: device rows in,
  device float64 scores out (no Python objects on the hot path).
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import os

import numpy as np

from . import _lib, errors
from . import space as sp


@dataclass(frozen=True)
class Tree:
    feature: np.ndarray  # (nodes,) int32, -1 = leaf
    threshold: np.ndarray  # (nodes,) float64
    child_left: np.ndarray  # (nodes,) int32
    child_right: np.ndarray  # (nodes,) int32
    value: np.ndarray  # (nodes,) float64

    @classmethod
    def from_dict(cls, obj: dict) -> "Tree":
        cols: dict[str, list] = {"f": [], "t": [], "l": [], "r": [], "v": []}

        def visit(node: dict) -> int:
            me = len(cols["f"])
            for key, init in (("f", -1), ("t", 0.0), ("l", -1), ("r", -1), ("v", 0.0)):
                cols[key].append(init)
            if "value" in node:
                cols["v"][me] = float(node["value"])
            else:
                cols["f"][me] = int(node["feature"])
                cols["t"][me] = float(node["threshold"])
                cols["l"][me] = visit(node["left"])
                cols["r"][me] = visit(node["right"])
            return me

        visit(obj)
        return cls(np.array(cols["f"], dtype=np.int32), np.array(cols["t"], dtype=np.float64),
                   np.array(cols["l"], dtype=np.int32), np.array(cols["r"], dtype=np.int32),
                   np.array(cols["v"], dtype=np.float64))

    def to_dict(self) -> dict:
        def node(i: int) -> dict:
            if self.feature[i] < 0:
                return {"value": float(self.value[i])}
            return {"feature": int(self.feature[i]), "threshold": float(self.threshold[i]),
                    "left": node(int(self.child_left[i])), "right": node(int(self.child_right[i]))}

        return node(0)


@dataclass(frozen=True)
class CostModel:
    trees: tuple
    base_score: float
    feature_count: int

    @classmethod
    def sentinel(cls, feature_count: int, base_score: float = 0.0) -> "CostModel":
        return cls(trees=(), base_score=base_score, feature_count=feature_count)

    @classmethod
    def from_json(cls, text: str) -> "CostModel":
        return cls.from_dict(json.loads(text))

    @classmethod
    def from_dict(cls, obj: dict) -> "CostModel":
        return cls(trees=tuple(Tree.from_dict(t) for t in obj["trees"]), base_score=float(obj["base_score"]),
                   feature_count=int(obj["feature_count"]))

    def to_json(self) -> str:
        return json.dumps({"base_score": self.base_score, "feature_count": self.feature_count,
                           "trees": [t.to_dict() for t in self.trees]}, sort_keys=True)


_TABLES: dict = {}  # knob values -> (table, neg, forest table), read-only arrays


def _tables(space):
    vals = sp.knob_values(space)
    key = tuple(tuple(v) for v in vals)
    hit = _TABLES.get(key)
    if hit is None:
        table, neg = _feature_table(vals)
        ftab = table.copy()
        for j, k in enumerate(neg):  # negative settings are rejected before scoring;
            ftab[j, :k] = -np.inf    # -inf keeps the cut-point search monotone
        for a in (table, neg, ftab):
            a.setflags(write=False)
        if len(_TABLES) > 256:
            _TABLES.clear()
        hit = _TABLES[key] = (table, neg, np.ascontiguousarray(ftab))
    return hit


def feature_table(space) -> tuple[np.ndarray, np.ndarray]:
    """log2(1 + value) lookup and negative-prefix counts (cost_model.py:235-249); cached per
    knob-value tuple, returned read-only."""
    table, neg, _ = _tables(space)
    return table, neg


def _feature_table(vals) -> tuple[np.ndarray, np.ndarray]:
    width = max(len(v) for v in vals)
    table = np.zeros((len(vals), width), dtype=np.float64)
    neg = np.zeros(len(vals), dtype=np.int64)
    for j, v in enumerate(vals):
        a = np.asarray(v, dtype=np.float64)
        neg[j] = int((a < 0).sum())
        with np.errstate(invalid="ignore", divide="ignore"):
            table[j, : a.size] = np.log2(1.0 + a)
    return table, neg


class DeviceForest:
    """kt_forest handle: the model packed for one space on one device."""

    def __init__(self, model, space, engine: _lib.Engine):
        cards = sp.check_engine_space(space)
        _, neg, table = _tables(space)
        trees = list(model.trees)
        flat = getattr(model, "__dict__", {}).get("_b200_flat")  # set by fit(): the same nodes, flat
        if flat is not None:
            node_off, feat, thr, left, right, val = flat
        else:
            offs = [0]
            for t in trees:
                offs.append(offs[-1] + int(np.asarray(t.feature).size))
            cat = lambda attr, dt: (np.ascontiguousarray(np.concatenate([np.asarray(getattr(t, attr), dtype=dt)
                                                                         for t in trees]))
                                    if trees else np.zeros(1, dtype=dt))
            feat, thr = cat("feature", np.int32), cat("threshold", np.float64)
            left, right, val = cat("child_left", np.int32), cat("child_right", np.int32), cat("value", np.float64)
            node_off = np.asarray(offs, dtype=np.int32)
        h = _lib.P()
        _lib.call("kt_forest_create", engine.handle, int(cards.size), _lib.as_ptr(cards, _lib.C.c_int32),
                  _lib.as_ptr(table, _lib.C.c_double), int(table.shape[1]), len(trees),
                  _lib.as_ptr(node_off, _lib.C.c_int32), _lib.as_ptr(feat, _lib.C.c_int32),
                  _lib.as_ptr(thr, _lib.C.c_double), _lib.as_ptr(left, _lib.C.c_int32),
                  _lib.as_ptr(right, _lib.C.c_int32), _lib.as_ptr(val, _lib.C.c_double),
                  float(model.base_score), _lib.C.byref(h))
        self.handle = h
        self.neg_prefix = neg
        self.n_knobs = int(cards.size)
        self.depth = int(_lib.load().kt_forest_depth(h))
        self.device = engine.device

    def __del__(self):
        try:
            _lib.load().kt_forest_destroy(self.handle)
        except Exception:
            pass


def _space_key(space) -> tuple:
    return (space.name, tuple(tuple(v) for v in sp.knob_values(space)))


def device_forest(model, space, engine: _lib.Engine | None = None) -> DeviceForest:
    engine = engine or _lib.engine()
    key = (engine.device, _space_key(space))
    cache = getattr(model, "__dict__", {}).get("_b200_forests")
    if cache is None:
        cache = {}
        try:
            object.__setattr__(model, "_b200_forests", cache)
        except (AttributeError, TypeError):
            pass
    f = cache.get(key)
    if f is None:
        f = DeviceForest(model, space, engine)
        cache[key] = f
    return f


def _check_model(model, space) -> None:
    if model.feature_count != len(space.knobs):
        raise errors.DimensionMismatchError(
            f"model expects {model.feature_count} features, space {space.name!r} has {len(space.knobs)} knobs")


def predict_rows(model, space, rows, out=None, engine: _lib.Engine | None = None):
    """Device path: ``rows`` is a CUDA int64/uint64 tensor of packed rows; returns CUDA float64 scores."""
    import torch

    _check_model(model, space)
    engine = engine or _lib.engine()
    f = device_forest(model, space, engine)
    n = int(rows.numel())
    with engine.scope():
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=rows.device)
        _lib.call("kt_score_trees", engine.handle, f.handle, _lib.ptr(rows), n, _lib.ptr(out))
    return out


def predict(model, space, configs) -> np.ndarray:
    """Surrogate fitness per configuration, in input order (cost_model.py:401-409)."""
    import torch

    _check_model(model, space)
    if not configs:
        return np.empty(0, dtype=np.float64)
    idx = sp.index_matrix(space, configs)
    engine = _lib.engine()
    f = device_forest(model, space, engine)
    if (idx < f.neg_prefix[None, :]).any():
        raise ValueError("featurize requires non-negative knob values")
    rows = torch.from_numpy(sp.pack(idx, sp.cardinalities(space)).view(np.int64)).to(f"cuda:{engine.device}")
    return predict_rows(model, space, rows, engine=engine).cpu().numpy()


# ------------------------------------------------------------------ fit
@dataclass(frozen=True)
class BoostParams:
    """cost_model.py:24-35."""

    rounds: int = 50
    depth: int = 4
    learning_rate: float = 0.3

    def validate(self) -> None:
        if self.rounds < 1:
            raise ValueError(f"rounds must be >= 1, got {self.rounds}")
        if self.depth < 1:
            raise ValueError(f"depth must be >= 1, got {self.depth}")
        if not 0.0 < self.learning_rate <= 1.0:
            raise ValueError(f"learning_rate must be in (0, 1], got {self.learning_rate}")


def _use_device_fit(params, n: int) -> bool:
    """The device engine is opt-in: byte-identical, but the split search's exact float64 cumsums
    are one sequential chain per (node, feature); measured on B200 the single-CTA kernel is at
    parity with the native host engine at the tuning loop's sizes (m = 1,000: 9.0 vs 9.3 ms;
    profiles/r2/fit_device.txt), so the tuning loop keeps the host engine."""
    return os.environ.get("KT_FIT_DEVICE", "") == "1" and int(params.depth) <= 7 and n <= 8


def fit(training, params=BoostParams(), seed: int = 0, engine=None, device: bool | None = None) -> CostModel:
    """Gradient boosting under squared error (fit, cost_model.py:367-398) — native exact-greedy
    restatement (csrc/fit.cu) in numpy's operation order: the model is byte-identical to the
    reference's (its JSON compares equal).  ``training`` is the reference's TrainingSet (or any
    object with ``features`` (m, n) and ``targets`` (m,)); ``seed`` is unused, as in the reference.

    ``device=True`` runs the boosting loop on the GPU (kt_fit_trees_device: one single-CTA
    kernel grows every tree); the default runs the same algorithm natively on the host
    (kt_fit_trees), which measured faster at tuning sizes.  Both give the same bytes.
    """
    params.validate()
    X = np.ascontiguousarray(np.asarray(training.features, dtype=np.float64))
    y = np.ascontiguousarray(np.asarray(training.targets, dtype=np.float64))
    if y.size == 0:
        raise ValueError("training set is empty")
    if X.ndim != 2 or y.ndim != 1 or X.shape[0] != y.shape[0]:
        raise errors.DimensionMismatchError(f"features {X.shape} and targets {y.shape} do not align")
    m, n = X.shape
    per_tree = (1 << (int(params.depth) + 1)) - 1
    cap = int(params.rounds) * per_tree
    feat = np.zeros(cap, dtype=np.int32)
    thr = np.zeros(cap, dtype=np.float64)
    left = np.zeros(cap, dtype=np.int32)
    right = np.zeros(cap, dtype=np.int32)
    val = np.zeros(cap, dtype=np.float64)
    offs = np.zeros(int(params.rounds) + 1, dtype=np.int32)
    base = _lib.C.c_double(0.0)
    C = _lib.C
    args = (_lib.as_ptr(X, C.c_double), _lib.as_ptr(y, C.c_double), m, n, int(params.rounds), int(params.depth),
            float(params.learning_rate), _lib.as_ptr(feat, C.c_int32), _lib.as_ptr(thr, C.c_double),
            _lib.as_ptr(left, C.c_int32), _lib.as_ptr(right, C.c_int32), _lib.as_ptr(val, C.c_double), cap,
            _lib.as_ptr(offs, C.c_int32), C.byref(base))
    if device is None:
        device = _use_device_fit(params, n)
    if device:
        eng = engine if engine is not None else _lib.engine()
        _lib.call("kt_fit_trees_device", eng.handle, *args)
    else:
        _lib.call("kt_fit_trees", *args)
    trees = []
    for r in range(int(params.rounds)):
        a, b = int(offs[r]), int(offs[r + 1])
        # views of the flat node arrays (the model owns them; DeviceForest packs the same arrays)
        trees.append(Tree(feature=feat[a:b], threshold=thr[a:b], child_left=left[a:b], child_right=right[a:b],
                          value=val[a:b]))
    model = CostModel(trees=tuple(trees), base_score=float(base.value), feature_count=n)
    used = int(offs[int(params.rounds)])
    flat = (offs, feat[:used], thr[:used], left[:used], right[:used], val[:used])
    try:  # DeviceForest packs these directly instead of re-concatenating the trees
        object.__setattr__(model, "_b200_flat", flat)
    except (AttributeError, TypeError):
        pass
    return model
