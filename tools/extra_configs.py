"""The BASELINE configs beyond the headline, measured inside the default bench.py run (rank 0,
one GPU) so the driver's own run records them: a short version of tools/sweep.py plus two-step
runs of the RL (configs[1]) and 12-task ResNet-18 (configs[3]) workloads.

Each entry: candidates/s over CUDA-event-timed steps after one warm-up step, L2 flushed between
steps (same methodology as the headline).  ~20-40 s in all.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _timed(eng, torch, flush, fn, steps):
    ms = []
    out = None
    for s in range(steps + 1):
        flush.fill_(float(s))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with eng.scope():
            a.record(eng.stream)
        out = fn(s)
        with eng.scope():
            b.record(eng.stream)
        torch.cuda.synchronize()
        if s:
            ms.append(a.elapsed_time(b))
    return float(np.median(ms)), out


def run_all(kt, torch, steps: int = 2, local_rank: int = 0, clock=None) -> dict:
    from paper_1905_12799_b200 import space as sp
    from paper_1905_12799_b200 import workloads as wl
    from tools import bench_c4, bench_rl

    t_start = time.time()
    eng = kt.engine(local_rank)
    dev = f"cuda:{local_rank}"
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    doc = json.loads((ROOT / "data" / "models" / "s2_resnet18.json").read_text())
    space = kt.space_from_dict({"name": doc["space"], "knobs": [{"name": f"k{i}", "values": v}
                                                                  for i, v in enumerate(doc["values"])]})
    model = kt.CostModel.from_dict(doc["model"])
    cards = np.array(space.cardinalities)
    vis = np.zeros(0, dtype=np.uint64)
    out = {"note": "rank 0, one GPU; median of CUDA-event-timed steps after a warm-up step, L2 flushed between "
                   "steps; candidates = trajectory entries scored + clustered per step"}

    # configs[4]: SA chains (K10, 128 steps, S2 surrogate) + adaptive sampling, N = chains x 129
    sweep = []
    for chains in (8, 512, 8192):
        params = kt.SAParams(chains=chains, steps_per_round=128)
        starts = torch.from_numpy(sp.pack(np.random.default_rng(chains).integers(0, cards, size=(chains, 8)))
                                  .view(np.int64)).to(dev)
        info = kt._lib.SampleInfo()

        def sa_step(s, params=params, starts=starts, info=info):
            rows, _, _ = kt.run_sa_rows(params, model, space, starts, seed=100 + s, engine=eng)
            kt.adaptive_sample_rows(rows, vis, space, seed=200 + s, engine=eng, info=info)
            return int(rows.numel())

        ms, n = _timed(eng, torch, flush, sa_step, steps)
        sweep.append({"chains": chains, "candidates": n, "distinct": int(info.n_distinct),
                      "knee_k": int(info.chosen_k), "ms_per_step": ms, "candidates_per_s": n / (ms / 1e3)})
    out["c5_sa_as_sweep"] = sweep

    # configs[2]: VGG-16 conv tasks, 256K uniform candidates per step (first two layer spaces)
    vgg = []
    for t in wl.VGG16_TASKS[:2]:
        vspace = sp.space_from_dict(t.space_dict())
        vcards = np.array(vspace.cardinalities)
        rng = np.random.default_rng(7)
        tr_idx = rng.integers(0, vcards, size=(500, vcards.size))
        table, _ = kt.cost_model.feature_table(vspace)
        X = table[np.arange(vcards.size), tr_idx]
        y = 1.0 / (0.5 + np.abs(np.sin(X.sum(axis=1))))

        class _TS:
            features, targets = X, y

        vmodel = kt.fit(_TS, kt.BoostParams())
        rows = torch.from_numpy(sp.pack(rng.integers(0, vcards, size=(1 << 18, vcards.size)), vcards)
                                .view(np.int64)).to(dev)
        info = kt._lib.SampleInfo()

        def vgg_step(s, vmodel=vmodel, vspace=vspace, rows=rows, info=info):
            kt.predict_rows(vmodel, vspace, rows, engine=eng)
            kt.adaptive_sample_rows(rows, vis, vspace, seed=300 + s, engine=eng, info=info)
            return 1 << 18

        ms, n = _timed(eng, torch, flush, vgg_step, steps)
        vgg.append({"task": t.name, "candidates": n, "knee_k": int(info.chosen_k), "ms_per_step": ms,
                    "candidates_per_s": n / (ms / 1e3)})
    out["c3_vgg16_256k"] = vgg

    # configs[1] and configs[3] through their bench modules (two steps after one warm-up)
    args = argparse.Namespace(steps=steps, warmup=1, no_cpu_baseline=True, rl_serial=False)

    class _NoClock:
        def __init__(self, *_a):
            pass

        def __enter__(self):
            return self

        def __exit__(self, *_a):
            return False

        def summary(self):
            return None

    helpers = {"barrier": torch.cuda.synchronize, "clock": clock or _NoClock}
    for key, mod in (("c1_alexnet_rl", bench_rl), ("c4_resnet18_12tasks", bench_c4)):
        line = mod.run(args, 0, 1, local_rank, kt, torch, None, helpers)
        out[key] = {"candidates_per_s": line["value"], "ms_per_step": line["ms_per_step"],
                    "workload": line["config"]["workload"][:160]}
    out["seconds"] = round(time.time() - t_start, 1)
    return out


if __name__ == "__main__":
    import torch

    import paper_1905_12799_b200 as kt

    print(json.dumps(run_all(kt, torch)))
