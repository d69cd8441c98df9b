"""Achieved error of the tcgen05 (3xTF32) PPO update against the float64 oracle, per call on
identical inputs (test_gpu_rl.py::test_large_round_vs_oracle's setup): one 4096-episode round on
the Table-1 space and one on an AlexNet task.  Prints one JSON line; written to gpurun_out/.

    python tools/ppo_error.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main() -> None:
    import torch

    import paper_1905_12799_b200 as kt
    from oracle import agent as oagent
    from paper_1905_12799_b200.agent import PARAM_KEYS, _flat
    from test_gpu_rl import _unflat, oracle_from, space_of

    models = json.loads((ROOT / "tests" / "golden" / "models.json").read_text())
    cases = [("table1", models["table1"]["values"], models["table1"]["model"])]
    for t in (0, 2):
        doc = json.loads((ROOT / "data" / "models" / f"alexnet_task{t}.json").read_text())
        cases.append((f"alexnet_task{t}", doc["values"], doc["model"]))
    out = {}
    for name, values, mdoc in cases:
        space = space_of(values)
        model = kt.CostModel.from_dict(mdoc)
        hyper = kt.AgentHyperparams(episodes_per_round=4096)
        agent = kt.init_agent(space, hyper, seed=21)
        ref = oracle_from(agent)
        cards = np.array(space.cardinalities)
        starts = np.random.default_rng(4).integers(0, cards, size=(4096, cards.size))
        before = _flat(agent.params)
        rows = torch.from_numpy(kt.pack(starts, cards).view(np.int64)).cuda()
        kt.run_search_rows(agent, model, space, rows)
        oagent.search_round(ref, mdoc, values, starts, hyper.to_dict())
        want = np.concatenate([ref["params"][k].ravel() for k in PARAM_KEYS])
        after = _flat(agent.params)
        d_got, d_want = after - before, want - before
        X = np.random.default_rng(0).random((4096, cards.size))
        lg, vg, _ = oagent.forward(_unflat(after, agent.params), X)
        lw, vw, _ = oagent.forward(_unflat(want, agent.params), X)
        pg, pw = np.exp(oagent.log_softmax(lg)), np.exp(oagent.log_softmax(lw))
        out[name] = {
            "param_update_max_abs_err_over_lr": float(np.max(np.abs(d_got - d_want)) / 1e-3),
            "param_update_rel_err": float(np.linalg.norm(d_got - d_want) / np.linalg.norm(d_want)),
            "probs_max_rel_err": float(np.max(np.abs(pg - pw) / pw)),
            "values_max_rel_err": float(np.max(np.abs(vg - vw) / np.maximum(np.abs(vw), 1.0))),
            "params_max_rel_err": float(np.max(np.abs(after - want) / np.maximum(np.abs(want), 1e-3))),
        }
    line = json.dumps(out)
    print(line)
    d = ROOT / "gpurun_out"
    d.mkdir(exist_ok=True)
    (d / "ppo_error.json").write_text(line + "\n")


if __name__ == "__main__":
    main()
