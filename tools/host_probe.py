"""Host-side cost of one headline step (predict_rows + adaptive_sample_rows) on the B200:
wall time vs device time, and a cProfile of the Python layer."""
import cProfile
import json
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_12799_b200 as kt  # noqa: E402
from paper_1905_12799_b200 import space as sp  # noqa: E402

doc = json.loads((ROOT / "data" / "models" / "s2_resnet18.json").read_text())
space = kt.space_from_dict({"name": "s2", "knobs": [{"name": f"k{i}", "values": v} for i, v in enumerate(doc["values"])]})
model = kt.CostModel.from_dict(doc["model"])
cards = np.array(space.cardinalities)
rows = torch.from_numpy(sp.pack(np.random.default_rng(0).integers(0, cards, size=(1 << 20, 8))).view(np.int64)).cuda()
eng = kt.engine(0)
out = torch.empty(1 << 20, dtype=torch.float64, device="cuda")
vis = np.zeros(0, dtype=np.uint64)


def step(s):
    kt.predict_rows(model, space, rows, out=out, engine=eng)
    return kt.adaptive_sample_rows(rows, vis, space, 7 + s, engine=eng)


for s in range(3):
    step(s)
torch.cuda.synchronize()
t = time.perf_counter()
for s in range(20):
    step(s)
torch.cuda.synchronize()
print(f"wall per step {(time.perf_counter() - t) / 20 * 1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for s in range(20):
    step(s)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
