"""BASELINE configs beyond the headline line, measured on one B200 (writes one JSON document).

* configs[4] — AutoTVM-style simulated annealing + adaptive sampling sweep: per step, SA chains
  (K10, 128 steps each, on the S2 ResNet-18 surrogate) produce N = chains x 129 trajectory entries,
  which adaptive_sample clusters (K6-K9).  N from ~1K to ~16M.
* configs[2] — VGG-16 conv tasks with 256K uniform candidates per step: predict + adaptive_sample
  (knee k-means over k in 8..64) for each of VGG-16's 9 layer spaces (surrogate fitted on the
  fly with the native refit on 500 random configurations of a generated landscape).

    python tools/sweep.py [--out gpurun_out/sweep.json] [--steps 3]

Timing: CUDA events on the engine stream around each step after one warm-up step, L2 flushed
between steps; candidates/s = N / step time.
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


def timed(eng, torch, flush, fn, steps):
    ms = []
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


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_1905_12799_b200 as kt
    from paper_1905_12799_b200 import space as sp
    from paper_1905_12799_b200 import workloads as wl

    eng = kt.engine(0)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
    doc = json.loads((ROOT / "data" / "models" / "s2_resnet18.json").read_text())
    space = kt.space_from_dict({"name": doc["space"], "knobs": [{"name": f"k{i}", "values": v}
                                                                  for i, v in enumerate(doc["values"])]})
    model = kt.CostModel.from_dict(doc["model"])
    cards = np.array(space.cardinalities)
    vis = np.zeros(0, dtype=np.uint64)
    result = {"device": torch.cuda.get_device_name(0), "sa_as_sweep": [], "vgg16_256k": []}

    # ---- configs[4]: SA + AS sweep
    for chains in (8, 64, 512, 4096, 32768, 131072):
        params = kt.SAParams(chains=chains, steps_per_round=128)
        starts = torch.from_numpy(sp.pack(np.random.default_rng(chains).integers(0, cards, size=(chains, 8)))
                                  .view(np.int64)).cuda()
        info = kt._lib.SampleInfo()

        def sa_step(s):
            rows, scores, steps = kt.run_sa_rows(params, model, space, starts, seed=100 + s, engine=eng)
            batch = kt.adaptive_sample_rows(rows, vis, space, seed=200 + s, engine=eng, info=info)
            return int(rows.numel()), batch

        ms, (n, batch) = timed(eng, torch, flush, sa_step, args.steps)
        result["sa_as_sweep"].append({"chains": chains, "steps_per_chain": 128, "candidates": n,
                                      "distinct": int(info.n_distinct), "knee_k": int(info.chosen_k),
                                      "ms_per_step": ms, "candidates_per_s": n / (ms / 1e3)})
        print(result["sa_as_sweep"][-1], flush=True)

    # ---- configs[2]: VGG-16 tasks, 256K candidates per step
    for t in wl.VGG16_TASKS:
        vspace = sp.space_from_dict(t.space_dict())
        vcards = np.array(vspace.cardinalities)
        rng = np.random.default_rng(7)
        tr_idx = rng.integers(0, vcards, size=(500, vcards.size))
        table, _ = kt.cost_model.feature_table(vspace)
        X = table[np.arange(vcards.size), tr_idx]
        y = 1.0 / (0.5 + np.abs(np.sin(X.sum(axis=1))))  # smooth synthetic fitness surface

        class _TS:
            features, targets = X, y

        vmodel = kt.fit(_TS, kt.BoostParams())
        rows = torch.from_numpy(sp.pack(rng.integers(0, vcards, size=(1 << 18, vcards.size)), vcards)
                                .view(np.int64)).cuda()
        info = kt._lib.SampleInfo()

        def vgg_step(s):
            kt.predict_rows(vmodel, vspace, rows, engine=eng)
            return kt.adaptive_sample_rows(rows, vis, vspace, seed=300 + s, engine=eng, info=info)

        ms, _ = timed(eng, torch, flush, vgg_step, args.steps)
        result["vgg16_256k"].append({"task": t.name, "cards": vcards.tolist(), "candidates": 1 << 18,
                                     "distinct": int(info.n_distinct), "knee_k": int(info.chosen_k),
                                     "scanned_k": [int(info.scanned_k[i]) for i in range(info.n_scanned)],
                                     "ms_per_step": ms, "candidates_per_s": (1 << 18) / (ms / 1e3)})
        print(result["vgg16_256k"][-1], flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(result, indent=1) + "\n")


if __name__ == "__main__":
    t0 = time.time()
    main()
    print(f"sweep done in {time.time() - t0:.1f} s")
