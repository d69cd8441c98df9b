"""Device-resident tuning loop (tune.py) vs the reference driver (tests/golden/tune.json).

sa+as / sa / random, replaying the reference's measured runtimes (its ``replay:`` backend idea):
every measured configuration equals the reference's tune log — the loop, its RNG streams, the
refit, the SA chains and the adaptive sampler agree bit for bit.  With the on-device K3
landscape the runtimes agree to <= 1 ulp (CUDA vs glibc exp) and the runs agree until the
first such difference feeds a refit.  rl+as: the bootstrap and the first search round's batch are exact; later
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


@pytest.mark.parametrize("case", G["cases"], ids=lambda c: f"{c['strategy']}_b{c['budget']}_s{c['seed']}")
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
    # the on-device landscape: same measurements until the first last-bit runtime difference
    dev = tune.tune_rows(SPACE, land, case["strategy"], case["budget"], case["seed"])
    got = np.array(dev.runtimes[:64])
    assert dev.configs[:64] == want[:64]
    assert np.max(np.abs(got - np.array(case["runtimes"][:64])) / got) <= 1e-12


def test_wall_to_95_trace():
    case = G["cases"][0]
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
