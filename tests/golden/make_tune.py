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
    (HERE / "tune.json").write_text(json.dumps({"space": space_json, "cases": out}) + "\n")


if __name__ == "__main__":
    main()
