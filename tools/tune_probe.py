"""Where does a tuning round's time go?  One sa+as tune on bench_grid4d landscape 0 with engine
kernel timing on, plus host-side wall time per stage."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_1905_12799_b200 as kt  # noqa: E402
from paper_1905_12799_b200 import tune  # noqa: E402
from paper_1905_12799_b200.landscape import landscape_from_dict  # noqa: E402

fx = json.loads((ROOT / "data" / "landscapes" / "bench_grid4d.json").read_text())
space = kt.space_from_dict(fx["space"])
land = landscape_from_dict(fx["landscapes"][0], space)
eng = kt.engine(0)
tune.tune_rows(space, land, "sa+as", 200, 1)  # warm
stage = {"fit": 0.0, "sa": 0.0, "as": 0.0, "measure": 0.0}
orig = {"fit": tune.fit, "sa": tune.run_sa_rows, "as": tune.adaptive_sample_rows, "measure": tune.runtimes_rows}


def wrap(name):
    def f(*a, **k):
        import torch
        t = time.perf_counter()
        out = orig[name](*a, **k)
        torch.cuda.synchronize()
        stage[name] += time.perf_counter() - t
        return out
    return f


tune.fit, tune.run_sa_rows, tune.adaptive_sample_rows, tune.runtimes_rows = (wrap(n) for n in ("fit", "sa", "as", "measure"))
eng.set_timing(True)
eng.kernel_stats(reset=True)
t0 = time.perf_counter()
run = tune.tune_rows(space, land, "sa+as", 1000, 0)
total = time.perf_counter() - t0
print(f"rounds {run.rounds} total {total*1e3:.1f} ms; per stage (ms):", {k: round(v * 1e3, 1) for k, v in stage.items()})
print({k: (c, round(ms, 2)) for k, (c, ms) in eng.kernel_stats(reset=True).items()})
