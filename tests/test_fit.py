"""Surrogate refit: kt_fit_trees (host code in the engine library, no
device work) vs the reference's fit — byte-identical model JSON on the golden cases produced
by running the reference (tests/golden/make_fit.py)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_fit import case_inputs  # noqa: E402

import paper_1905_12799_b200 as kt  # noqa: E402
from paper_1905_12799_b200 import _lib  # noqa: E402

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "fit.json").read_text())


class _TS:
    def __init__(self, X, y):
        self.features, self.targets = X, y


def _lib_or_skip():
    try:
        _lib.load()
    except _lib.EngineUnavailable as ex:  # pragma: no cover
        pytest.skip(str(ex))


@pytest.mark.parametrize("case", GOLD, ids=lambda c: f"m{c['m']}_n{c['n']}_{c['targets']}")
def test_fit_byte_identical_to_reference(case):
    _lib_or_skip()
    X, y = case_inputs(case["seed"], case["m"], case["n"], case["levels"], case["targets"])
    model = kt.fit(_TS(X, y), kt.BoostParams(case["rounds"], case["depth"], case["lr"]))
    assert model.to_json() == case["model"]
    # row order must not matter (canonical lexsort order inside)
    perm = np.random.default_rng(1).permutation(len(y))
    assert kt.fit(_TS(X[perm], y[perm]), kt.BoostParams(case["rounds"], case["depth"], case["lr"])).to_json() == \
        case["model"]


def test_fit_errors():
    _lib_or_skip()
    with pytest.raises(ValueError, match="empty"):
        kt.fit(_TS(np.zeros((0, 2)), np.zeros(0)))
    with pytest.raises(ValueError, match="rounds"):
        kt.fit(_TS(np.zeros((3, 2)), np.zeros(3)), kt.BoostParams(rounds=0))
    with pytest.raises(ValueError, match="learning_rate"):
        kt.fit(_TS(np.zeros((3, 2)), np.zeros(3)), kt.BoostParams(learning_rate=0.0))
