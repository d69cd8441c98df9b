"""Golden tuning runs produced by the REFERENCE driver (driver.tune, driver.py:161-243).

    python tests/golden/make_tune.py       # writes tests/golden/tune.json

Each case records the reference's measurement sequence (index tuples + runtimes) for the
bench_grid4d fixture space and one of its landscapes; the GPU test replays the same task
through paper_1905_12799_b200.tune.tune_rows and compares measurement for measurement.
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from knobtuner import driver  # noqa: E402
from knobtuner.agent import AgentHyperparams  # noqa: E402
from knobtuner.sa import SAParams  # noqa: E402
from knobtuner.space import parse_space  # noqa: E402

HERE = Path(__file__).resolve().parent
PKG = Path("/root/reference/pkg")
CASES = [("sa+as", 0, 300, 0), ("sa", 1, 200, 3), ("random", 2, 150, 1), ("rl+as", 0, 200, 0)]
# failure injection (MeasurementRecord semantics, backends.py:54-71): configurations whose index sum
# is divisible by `mod` measure as `bad` (inf or a non-positive runtime)
FAIL_CASES = [("sa+as", 3, 300, 2, 5, "inf"), ("sa", 4, 200, 1, 4, "-1.0")]


def failing(backend, mod: int, bad: float):
    class Failing:
        tag = "failing-synthetic"
        space = backend.space

        def batch_runtimes(self, configs):
            rts = backend.batch_runtimes(configs)
            return [bad if sum(c.indices) % mod == 0 else r for c, r in zip(configs, rts)]

    return Failing()


def main() -> None:
    space_json = json.loads((PKG / "spaces" / "bench_grid4d.json").read_text())
    space = parse_space(json.dumps(space_json))
    out = []
    for strategy, land, budget, seed in CASES:
        lpath = PKG / "landscapes" / f"bench_grid4d_s{land}.json"
        task = driver.TuningTask(space=space, backend_spec=f"synthetic:{lpath}", strategy=strategy, budget=budget,
                                 seed=seed, agent_params=AgentHyperparams(), sa_params=SAParams())
        with tempfile.TemporaryDirectory() as d:
            res = driver.tune(task, d)
            lines = [json.loads(x) for x in (Path(d) / driver.LOG_FILENAME).read_text().splitlines()]
        out.append({"strategy": strategy, "landscape": json.loads(lpath.read_text()), "budget": budget, "seed": seed,
                    "indices": [ln["indices"] for ln in lines], "runtimes": [ln["runtime_s"] for ln in lines],
                    "rounds": res.rounds})
        print(strategy, len(lines), res.rounds, res.best_runtime_s)
    for strategy, land, budget, seed, mod, bad in FAIL_CASES:
        lpath = PKG / "landscapes" / f"bench_grid4d_s{land}.json"
        task = driver.TuningTask(space=space, backend_spec=f"synthetic:{lpath}", strategy=strategy, budget=budget,
                                 seed=seed, agent_params=AgentHyperparams(), sa_params=SAParams())
        backend = failing(driver.make_backend(task.backend_spec, space), mod, float(bad))
        with tempfile.TemporaryDirectory() as d:
            res = driver.tune(task, d, backend=backend)
            lines = [json.loads(x) for x in (Path(d) / driver.LOG_FILENAME).read_text().splitlines()]
        out.append({"strategy": strategy, "landscape": json.loads(lpath.read_text()), "budget": budget, "seed": seed,
                    "fail_mod": mod, "fail_value": bad,
                    "indices": [ln["indices"] for ln in lines], "runtimes": [ln["runtime_s"] for ln in lines],
                    "failed": [ln["failed"] for ln in lines], "rounds": res.rounds})
        print(strategy, "fail", mod, len(lines), res.rounds, sum(ln["failed"] for ln in lines))
    (HERE / "tune.json").write_text(json.dumps({"space": space_json, "cases": out}) + "\n")


if __name__ == "__main__":
    main()
