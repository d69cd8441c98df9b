"""Where the RL step's time goes: per task, host wall time of run_search_rows and adaptive_sample_rows
next to their device time (CUDA events on the engine stream) and the engine's per-kernel busy time.

    python tools/rl_step_probe.py [--steps 5]
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import bench_rl
    import paper_1905_12799_b200 as kt

    sp = kt.space
    eng = kt.engine(0)
    tasks = []
    for i, d in enumerate(bench_rl.task_docs()):
        space = kt.space_from_dict({"name": d["space"], "knobs": [{"name": f"k{j}", "values": v}
                                                                   for j, v in enumerate(d["values"])]})
        model = kt.CostModel.from_dict(d["model"])
        agent = kt.init_agent(space, kt.AgentHyperparams(episodes_per_round=bench_rl.AGENTS), seed=i)
        cards = np.array(space.cardinalities)
        starts = torch.from_numpy(sp.pack(np.random.default_rng(i).integers(0, cards, size=(bench_rl.AGENTS, cards.size)),
                                          cards).view(np.int64)).cuda()
        tasks.append((space, model, agent, starts))
    vis = np.zeros(0, dtype=np.uint64)

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        with eng.scope():
            e.record(eng.stream)
        return e

    for s in range(args.steps + 2):
        rec = []
        torch.cuda.synchronize()
        t_step = time.perf_counter()
        e_step = ev()
        for space, model, agent, starts in tasks:
            e0 = ev()
            h0 = time.perf_counter()
            rows, _, _ = kt.run_search_rows(agent, model, space, starts, engine=eng)
            h1 = time.perf_counter()
            e1 = ev()
            kt.adaptive_sample_rows(rows, vis, space, seed=s, engine=eng)
            h2 = time.perf_counter()
            e2 = ev()
            rec.append((h1 - h0, h2 - h1, e0, e1, e2))
        e_end = ev()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t_step
        if s < 2:
            continue
        print(f"step {s}: wall {wall * 1e3:.2f} ms, device {e_step.elapsed_time(e_end):.2f} ms")
        for i, (hs, ha, e0, e1, e2) in enumerate(rec):
            print(f"  task {i}: search host {hs * 1e3:6.2f} dev {e0.elapsed_time(e1):6.2f} | "
                  f"sample host {ha * 1e3:6.2f} dev {e1.elapsed_time(e2):6.2f} ms")
    eng.set_timing(True)
    eng.kernel_stats(reset=True)
    for space, model, agent, starts in tasks:
        rows, _, _ = kt.run_search_rows(agent, model, space, starts, engine=eng)
        kt.adaptive_sample_rows(rows, vis, space, seed=99, engine=eng)
    stats = eng.kernel_stats(reset=True)
    busy = sum(ms for _, ms in stats.values())
    print(f"kernel busy per step: {busy:.2f} ms")


if __name__ == "__main__":
    main()
