"""Device-resident tuning loop (tune.py) vs the reference driver (tests/golden/tune.json).

sa+as / sa / random, replaying the reference's measured runtimes (its ``replay:`` backend idea):
every measured configuration equals the reference's tune log — the loop, its RNG streams, the
refit, the SA chains and the adaptive sampler agree bit for bit.  With the on-device K3
landscape (glibc's exp restated bit-exactly) the whole run, runtimes included, equals the
reference's log too.  rl+as: the bootstrap and the first search round's batch are exact; later
rounds follow the PPO update, which the north star holds to the TF32 tier, so only the
budget accounting is checked there.
"""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_12799_b200 as kt  # noqa: E402
from golden_io import GOLDEN  # noqa: E402
from paper_1905_12799_b200 import tune  # noqa: E402
from paper_1905_12799_b200.landscape import landscape_from_dict  # noqa: E402

G = json.loads((GOLDEN / "tune.json").read_text())
SPACE = kt.space_from_dict(G["space"])


CLEAN = [c for c in G["cases"] if "fail_mod" not in c]
FAILING = [c for c in G["cases"] if "fail_mod" in c]


@pytest.mark.parametrize("case", FAILING, ids=lambda c: f"{c['strategy']}_fail{c['fail_mod']}_{c['fail_value']}")
def test_tune_with_failed_measurements_matches_reference(case):
    """Failed measurements (inf / non-positive runtimes) follow MeasurementRecord: excluded from the
    refit, fitness 0, runtime inf — the run equals the reference driver's log (make_tune.py)."""
    land = landscape_from_dict(case["landscape"], SPACE)
    want = [tuple(x) for x in case["indices"]]
    table = dict(zip(want, case["runtimes"]))
    mod, bad = case["fail_mod"], float(case["fail_value"])
    run = tune.tune_rows(SPACE, land, case["strategy"], case["budget"], case["seed"],
                         runtimes=lambda batch: [bad if sum(t) % mod == 0 else table[t] for t in batch])
    assert run.configs == want
    assert run.rounds == case["rounds"]
    assert [r == float("inf") for r in run.runtimes] == case["failed"]
    assert any(case["failed"])


@pytest.mark.parametrize("case", CLEAN, ids=lambda c: f"{c['strategy']}_b{c['budget']}_s{c['seed']}")
def test_tune_matches_reference_driver(case):
    land = landscape_from_dict(case["landscape"], SPACE)
    want = [tuple(x) for x in case["indices"]]
    table = dict(zip(want, case["runtimes"]))
    run = tune.tune_rows(SPACE, land, case["strategy"], case["budget"], case["seed"],
                         runtimes=lambda batch: [table[t] for t in batch])
    assert len(run.configs) == case["budget"] == len(want)
    if case["strategy"] == "rl+as":
        first = 64 + 1  # bootstrap + at least the first search round's first batch entry
        assert run.configs[:first] == want[:first]
        return
    assert run.configs == want
    assert run.rounds == case["rounds"]
    # the on-device landscape: bit-exact runtimes, so the unreplayed run is the reference's log
    dev = tune.tune_rows(SPACE, land, case["strategy"], case["budget"], case["seed"])
    assert dev.configs == want
    assert [float(x).hex() for x in dev.runtimes] == [float(x).hex() for x in case["runtimes"]]


def test_wall_to_95_trace():
    case = CLEAN[0]
    land = landscape_from_dict(case["landscape"], SPACE)
    best_rt, _ = kt.best_runtime(land)
    f_star = 1.0 / best_rt
    run = tune.tune_rows(SPACE, land, "sa+as", 1000, seed=0)
    t95 = run.wall_to_fraction(f_star, 0.95)
    assert run.best_fitness <= f_star * (1 + 1e-12)
    bests = [b for _, _, b in run.trace]
    assert bests == sorted(bests)
    if t95 is not None:
        assert 0.0 < t95 <= run.seconds


TOPK = json.loads((GOLDEN / "topk.json").read_text())


def _topk_inputs(case):
    import sys

    sys.path.insert(0, str(GOLDEN))
    from make_topk import case_inputs

    return case_inputs(*case)


@pytest.mark.parametrize("g", TOPK, ids=lambda g: g["case"][0])
def test_top_unvisited_vs_reference(g):
    """kt_top_unvisited == the reference's _top_unvisited (driver.py:101-115) on its own goldens:
    duplicates, score ties, signed zeros, visited overlap, short and empty batches."""
    from paper_1905_12799_b200 import space as sp

    idx, scores, vis = _topk_inputs(g["case"])
    cards = np.array(g["case"][2])
    tr = kt.Trajectory(torch.from_numpy(sp.pack(idx, cards).view(np.int64)).cuda(), torch.from_numpy(scores).cuda(),
                       n_knobs=cards.size, cards=cards)
    visited = kt.VisitedSet([kt.Configuration(tuple(r)) for r in vis.tolist()])
    got = tune.top_unvisited(tr, visited, 64)
    assert [list(c.indices) for c in got] == g["batch"]

    class RefShaped:  # the reference's Trajectory: entries of (Configuration, score)
        def __init__(self, entries):
            self.entries = entries

        def configs(self):
            return [c for c, _ in self.entries]

    ref_tr = RefShaped(tuple((kt.Configuration(tuple(r)), float(s)) for r, s in zip(idx.tolist(), scores.tolist())))
    assert [list(c.indices) for c in tune.top_unvisited(ref_tr, visited, 64)] == g["batch"]


@pytest.mark.parametrize("n", [1, 511, 1 << 20])
def test_top_unvisited_large_vs_oracle(n):
    from oracle import tune as otune
    from paper_1905_12799_b200 import space as sp

    rng = np.random.default_rng(n)
    cards = np.array([84, 80, 80, 7, 2, 2, 3, 2])
    idx = rng.integers(0, cards, size=(n, 8))
    idx[n // 2:] = idx[: n - n // 2]  # every second half row repeats the first half
    scores = np.round(rng.standard_normal(n), 2)  # ties
    vis = idx[rng.integers(0, n, size=min(n, 300))]
    visited = {tuple(r) for r in vis.tolist()}
    got = tune.top_unvisited_rows(torch.from_numpy(sp.pack(idx).view(np.int64)).cuda(),
                                  torch.from_numpy(scores).cuda(), sp.pack(np.array(sorted(visited))), 64)
    assert [tuple(r) for r in sp.unpack(got, 8).tolist()] == otune.top_unvisited(idx, scores, visited, 64)
