"""Concurrent engines (one host thread each) on one GPU: which stage fails?  (GPU)
    python tools/concurrency_probe.py search|sample|both [threads] [iters]"""
import sys
import threading
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1905_12799_b200 as kt  # noqa: E402
from tools.bench_rl import AGENTS, task_docs  # noqa: E402

mode = sys.argv[1]
nth = int(sys.argv[2]) if len(sys.argv) > 2 else 5
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
docs = task_docs()
engines = [kt.engine(0)] + [kt._lib.Engine(0) for _ in range(nth - 1)]
tasks = []
for i in range(nth):
    d = docs[i % len(docs)]
    space = kt.space_from_dict({"name": d["space"], "knobs": [{"name": f"k{j}", "values": v}
                                                               for j, v in enumerate(d["values"])]})
    model = kt.CostModel.from_dict(d["model"])
    agent = kt.init_agent(space, kt.AgentHyperparams(episodes_per_round=AGENTS), seed=i)
    cards = np.array(space.cardinalities)
    starts = torch.from_numpy(kt.space.pack(np.random.default_rng(i).integers(0, cards, size=(AGENTS, cards.size)),
                                            cards).view(np.int64)).cuda()
    rows = None
    if "cold" not in sys.argv:  # warm: device objects created serially first
        rows, _, _ = kt.run_search_rows(agent, model, space, starts, engine=engines[0])
        rows = rows.clone()
    tasks.append((space, model, agent, starts, rows))
torch.cuda.synchronize()
errs = []


def body(i):
    space, model, agent, starts, rows0 = tasks[i]
    e = engines[i]
    try:
        with torch.cuda.stream(e.stream):
            for it in range(iters):
                if mode in ("search", "both") or rows0 is None:
                    rows, _, _ = kt.run_search_rows(agent, model, space, starts, engine=e)
                else:
                    rows = rows0
                if mode in ("sample", "both"):
                    kt.adaptive_sample_rows(rows, np.zeros(0, np.uint64), space, seed=it, engine=e)
        e.synchronize()
    except BaseException as ex:
        errs.append(f"thread {i}: {ex}")


th = [threading.Thread(target=body, args=(i,)) for i in range(nth)]
for t in th:
    t.start()
for t in th:
    t.join()
print(mode, "OK" if not errs else errs[:2])
