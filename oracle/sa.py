"""Oracle: simulated-annealing chains on the surrogate (TEST INFRASTRUCTURE ONLY).

Restates ``knobtuner/sa.py:45-122`` (``_propose_into`` + ``run_sa_round``) at
array level.  Each chain owns ``default_rng(SeedSequence(seed).spawn(chains)[c])``;
per step it draws ``integers(0, n)`` (knob), ``integers(0, 2)`` (sign) and —
only when the proposal lowers the score — ``random()`` for Metropolis.
Starts shorter than ``chains`` are padded from the parent generator
(``random_config``: ``integers(0, card)`` per knob, space.py:212-214).
"""

from __future__ import annotations

import math

import numpy as np

from .trees import feature_table, predict_features

TEMPERATURE_STD_FLOOR = 1e-12


def run_sa_round(model: dict, knob_values: list[list[int]], starts, seed: int,
                 chains: int = 64, steps: int = 128, initial_temperature=None,
                 cooling: float = 0.99):
    """Returns (entries_idx (E, n) int64, scores (E,), step_indices (E,)), chain-major."""
    cards = np.array([len(v) for v in knob_values], dtype=np.int64)
    n = cards.size
    parent = np.random.SeedSequence(int(seed) & (2**64 - 1))
    pad = np.random.default_rng(parent)
    walkers = [np.random.default_rng(s) for s in parent.spawn(chains)]

    rows = [tuple(int(i) for i in s) for s in list(starts)[:chains]]
    while len(rows) < chains:
        rows.append(tuple(int(pad.integers(0, c)) for c in cards))
    cur = np.array(rows, dtype=np.int64)

    table, neg = feature_table(knob_values)
    if neg.any():
        raise ValueError("featurize requires non-negative knob values")
    knob_axis = np.arange(n)
    score = predict_features(model, table[knob_axis[None, :], cur]).tolist()

    if initial_temperature is not None:
        temp = float(initial_temperature)
    else:
        spread = float(np.std(score))
        temp = spread if spread > TEMPERATURE_STD_FLOOR else 1.0

    kept_rows = [[tuple(r)] for r in cur.tolist()]
    kept_score = [[s] for s in score]
    kept_step = [[0] for _ in range(chains)]
    prop = np.empty_like(cur)
    for step in range(1, steps + 1):
        prop[:] = cur
        for c, g in enumerate(walkers):
            knob = int(g.integers(0, n))
            sign = int(g.integers(0, 2)) * 2 - 1
            prop[c, knob] = min(max(prop[c, knob] + sign, 0), cards[knob] - 1)
        prop_score = predict_features(model, table[knob_axis[None, :], prop])
        for c, g in enumerate(walkers):
            delta = float(prop_score[c]) - score[c]
            if delta >= 0.0 or g.random() < math.exp(delta / temp):
                cur[c] = prop[c]
                score[c] = float(prop_score[c])
                kept_rows[c].append(tuple(int(i) for i in prop[c]))
                kept_score[c].append(score[c])
                kept_step[c].append(step)
        temp *= cooling

    flat_rows = [r for chain in kept_rows for r in chain]
    flat_score = [s for chain in kept_score for s in chain]
    flat_step = [s for chain in kept_step for s in chain]
    return (np.array(flat_rows, dtype=np.int64).reshape(-1, n),
            np.array(flat_score, dtype=np.float64),
            np.array(flat_step, dtype=np.int64))
