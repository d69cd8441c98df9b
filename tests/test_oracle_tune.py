"""The oracle's refit + tuning loop (oracle/tune.py) pinned to the reference: byte-identical
models on the fit goldens, and the reference driver's exact measurement logs (CPU only)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_fit import case_inputs  # noqa: E402

from oracle import tune as otune  # noqa: E402

GOLDEN = Path(__file__).resolve().parent / "golden"
FIT = json.loads((GOLDEN / "fit.json").read_text())
TUNE = json.loads((GOLDEN / "tune.json").read_text())


@pytest.mark.parametrize("case", FIT[:8], ids=lambda c: f"m{c['m']}_n{c['n']}")
def test_oracle_fit_matches_reference(case):
    X, y = case_inputs(case["seed"], case["m"], case["n"], case["levels"], case["targets"])
    model = otune.fit_model(X, y, case["rounds"], case["depth"], case["lr"])
    assert json.dumps(model, sort_keys=True) == case["model"]


@pytest.mark.parametrize("case", [c for c in TUNE["cases"] if c["strategy"] != "rl+as" and "fail_mod" not in c],
                         ids=lambda c: c["strategy"])
def test_oracle_tune_matches_reference_driver(case):
    values = [k["values"] for k in TUNE["space"]["knobs"]]
    configs, runtimes, trace, rounds = otune.tune(values, case["landscape"], case["strategy"], case["budget"],
                                                  case["seed"])
    assert configs == [tuple(x) for x in case["indices"]]
    assert runtimes == case["runtimes"]
    assert rounds == case["rounds"]
    assert [t[1] for t in trace][-1] == case["budget"]
    assert np.all(np.diff([t[2] for t in trace]) >= 0)


TOPK = json.loads((GOLDEN / "topk.json").read_text())


@pytest.mark.parametrize("g", TOPK, ids=lambda g: g["case"][0])
def test_oracle_top_unvisited_matches_reference(g):
    sys.path.insert(0, str(GOLDEN))
    from make_topk import case_inputs

    idx, scores, vis = case_inputs(*g["case"])
    got = otune.top_unvisited(idx, scores, {tuple(r) for r in vis.tolist()}, 64)
    assert [list(t) for t in got] == g["batch"]
