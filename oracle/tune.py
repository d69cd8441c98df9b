"""Oracle: surrogate refit + tuning loop on the host (TEST INFRASTRUCTURE ONLY).

Restates, in numpy:

* ``fit_model``  <- cost_model.py:292-398 (exact greedy boosted trees: canonical lexsort row
  order, per-feature stable orders partitioned down the tree, sequential cumsums, first-max
  split per feature, strictly better gain across features, preorder node ids) -> the model in
  the reference's JSON document form (cost_model.py:203-218).
* ``tune``       <- driver.py:161-243 for the sa / sa+as / random strategies: bootstrap,
  per-round refit (driver.py:142-148), SA round with ``_round_seed`` (driver.py:67-69),
  adaptive sample or greedy top-64 (driver.py:101-115), random fill (driver.py:72-98).

Pinned against the reference's own tune logs (tests/golden/tune.json, tests/test_oracle_tune.py).
Used by bench.py's reference arm for the wall-time-to-95%-best metric.
"""

from __future__ import annotations

import time

import numpy as np

from .landscape import synthetic_runtimes
from .sa import run_sa_round
from .sampler import adaptive_sample
from .trees import feature_table


# ------------------------------------------------------------------ boosted trees
def _node_split(X, resid, orders):
    """Best (feature, threshold) over the node's per-feature orders, or None."""
    chosen = None  # (gain, feature, threshold)
    size = orders[0].size
    for feat, order in enumerate(orders):
        col = X[order, feat]
        res = resid[order]
        cut = np.flatnonzero(col[1:] != col[:-1])
        if cut.size == 0:
            continue
        run_sum = np.cumsum(res)
        run_sq = np.cumsum(res * res)
        tot, tot_sq = run_sum[-1], run_sq[-1]
        n_left = cut + 1
        n_right = size - n_left
        s_left, q_left = run_sum[cut], run_sq[cut]
        left_err = q_left - s_left * s_left / n_left
        right_err = (tot_sq - q_left) - (tot - s_left) ** 2 / n_right
        gain = (tot_sq - tot * tot / size) - left_err - right_err
        at = int(np.argmax(gain))
        if chosen is None or float(gain[at]) > chosen[0]:
            chosen = (float(gain[at]), feat, float((col[cut[at]] + col[cut[at] + 1]) / 2.0))
    return None if chosen is None else chosen[1:]


def _grow_tree(X, resid, max_depth, shrink):
    """One regression tree as the reference's nested dict (preorder growth)."""

    def build(rows, orders, depth):
        part = resid[rows]
        mu = float(part.mean())
        err = float(((part - mu) ** 2).sum())
        split = _node_split(X, resid, orders) if depth < max_depth and err > 0.0 else None
        if split is None:
            return {"value": shrink * mu}
        feat, thr = split
        mask = np.zeros(X.shape[0], dtype=bool)
        mask[rows[X[rows, feat] <= thr]] = True
        left = build(rows[mask[rows]], [o[mask[o]] for o in orders], depth + 1)
        right = build(rows[~mask[rows]], [o[~mask[o]] for o in orders], depth + 1)
        return {"feature": feat, "threshold": thr, "left": left, "right": right}

    rows = np.arange(X.shape[0], dtype=np.int64)
    return build(rows, [np.argsort(X[:, j], kind="stable") for j in range(X.shape[1])], 0)


def _tree_values(node, X):
    out = np.empty(X.shape[0], dtype=np.float64)
    todo = [(node, np.arange(X.shape[0]))]
    while todo:
        nd, rows = todo.pop()
        if "value" in nd:
            out[rows] = nd["value"]
            continue
        go = X[rows, nd["feature"]] <= nd["threshold"]
        todo.append((nd["left"], rows[go]))
        todo.append((nd["right"], rows[~go]))
    return out


def fit_model(features, targets, rounds: int = 50, depth: int = 4, learning_rate: float = 0.3) -> dict:
    X0 = np.asarray(features, dtype=np.float64)
    y0 = np.asarray(targets, dtype=np.float64)
    canon = np.lexsort(np.vstack([y0, X0.T[::-1]]))
    X, y = X0[canon], y0[canon]
    base = float(y.mean())
    pred = np.full(y.shape, base)
    trees = []
    for _ in range(rounds):
        tree = _grow_tree(X, y - pred, depth, learning_rate)
        pred += _tree_values(tree, X)
        trees.append(tree)
    return {"base_score": base, "feature_count": int(X.shape[1]), "trees": trees}


# ------------------------------------------------------------------ tuning loop
def _round_seed(seed, r):
    return int(np.random.SeedSequence(seed & (2**64 - 1), spawn_key=(r,)).generate_state(1, dtype=np.uint64)[0])


def _draw(cards, rng):
    return tuple(int(rng.integers(0, c)) for c in cards)


def _fresh(cards, visited, count, rng):
    if count <= 0:
        return []
    out, seen, tries = [], set(), 0
    while len(out) < count and tries < max(200, 20 * count):
        tries += 1
        c = _draw(cards, rng)
        if c not in seen and c not in visited:
            seen.add(c)
            out.append(c)
    if len(out) < count and int(np.prod(cards)) <= 10**6:
        grid = [t for t in map(tuple, np.indices(tuple(cards)).reshape(len(cards), -1).T.tolist())
                if t not in visited and t not in seen]
        k = min(count - len(out), len(grid))
        if k > 0:
            out += [grid[int(i)] for i in rng.choice(len(grid), size=k, replace=False)]
    return out


def tune(knob_values, landscape: dict, strategy: str, budget: int, seed: int = 0, bootstrap: int = 64,
         chains: int = 64, steps: int = 128, clock=time.perf_counter, stop_fitness: float | None = None):
    """Returns (configs, runtimes, trace[(seconds, measurements, best fitness)], rounds); stops early
    once best-so-far fitness reaches ``stop_fitness`` (the wall-time-to-95% harness)."""
    if strategy not in ("sa", "sa+as", "random"):
        raise ValueError("oracle tune covers the sa, sa+as and random strategies")
    cards = [len(v) for v in knob_values]
    table, _ = feature_table(knob_values)
    rng = np.random.default_rng(np.random.SeedSequence(seed & (2**64 - 1), spawn_key=(0xD21,)))
    visited, configs, runtimes, trace = set(), [], [], []
    t0, best = clock(), 0.0

    def measure(batch):
        nonlocal best
        rt = synthetic_runtimes(landscape, np.asarray(batch, dtype=np.int64))
        configs.extend(batch)
        runtimes.extend(rt.tolist())
        visited.update(batch)
        best = max(best, float(np.max(1.0 / rt)))
        trace.append((clock() - t0, len(configs), best))

    rounds = 0
    first = _fresh(cards, visited, min(bootstrap, budget), rng)
    if first:
        measure(first)
        rounds = 1
    while len(configs) < budget and not (stop_fitness is not None and best >= stop_fitness):
        left = budget - len(configs)
        batch = []
        if strategy != "random":
            idx = np.asarray(configs, dtype=np.int64)
            model = fit_model(table[np.arange(len(cards)), idx], 1.0 / np.asarray(runtimes))
            starts = [_draw(cards, rng) for _ in range(chains)]
            t_idx, t_sc, _ = run_sa_round(model, knob_values, starts, _round_seed(seed, rounds), chains, steps)
            if strategy == "sa+as":
                batch = adaptive_sample(t_idx, visited, cards, _round_seed(seed, rounds))
            else:
                seen, cand, sc = set(), [], []
                for t, s in zip(map(tuple, t_idx.tolist()), t_sc.tolist()):
                    if t not in seen and t not in visited:
                        seen.add(t)
                        cand.append(t)
                        sc.append(s)
                batch = [cand[int(i)] for i in np.argsort(-np.asarray(sc), kind="stable")[:64]]
        if not batch:
            batch = _fresh(cards, visited, min(64, left), rng)
        if not batch:
            break
        measure(batch[:left])
        rounds += 1
    return configs, runtimes, trace, rounds


def top_unvisited(idx, scores, visited: set, cap: int = 64) -> list:
    """driver.py:101-115 (_top_unvisited): first occurrence of every unvisited configuration, stable
    sort by -score, first ``cap``."""
    configs, sc, seen = [], [], set()
    for t, s in zip(map(tuple, np.asarray(idx, dtype=np.int64).tolist()), np.asarray(scores).tolist()):
        if t in seen or t in visited:
            continue
        seen.add(t)
        configs.append(t)
        sc.append(s)
    if not configs:
        return []
    order = np.argsort(-np.asarray(sc, dtype=np.float64), kind="stable")
    return [configs[int(i)] for i in order[:cap]]
