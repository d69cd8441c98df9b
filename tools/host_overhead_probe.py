"""Host-side overhead of one headline step (GPU): cProfile of 20 predict + adaptive_sample steps on
the 1M-candidate S2 input, plus the wall time per step against the engine's kernel time."""
import cProfile
import json
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1905_12799_b200 as kt  # noqa: E402
from paper_1905_12799_b200 import space as sp  # noqa: E402

doc = json.loads((ROOT / "data/models/s2_resnet18.json").read_text())
space = kt.space_from_dict({"name": "s2", "knobs": [{"name": f"k{i}", "values": v} for i, v in enumerate(doc["values"])]})
model = kt.CostModel.from_dict(doc["model"])
cards = np.array(space.cardinalities)
idx = np.random.default_rng(0).integers(0, cards, size=(1 << 20, 8))
rows = torch.from_numpy(sp.pack(idx).view(np.int64)).cuda()
out = torch.empty(1 << 20, dtype=torch.float64, device="cuda")
eng = kt.engine(0)
vis = sp.pack(idx[:2])


def step(s):
    kt.predict_rows(model, space, rows, out=out, engine=eng)
    return kt.adaptive_sample_rows(rows, vis, space, 1000 + s, engine=eng)


for s in range(3):
    step(s)
torch.cuda.synchronize()
t = time.perf_counter()
for s in range(20):
    step(s)
torch.cuda.synchronize()
wall = (time.perf_counter() - t) / 20
eng.set_timing(True)
eng.kernel_stats(reset=True)
for s in range(5):
    step(s)
st = eng.kernel_stats(reset=True)
eng.set_timing(False)
kern = sum(ms for _, ms in st.values()) / 5
print(f"wall per step {wall * 1e3:.3f} ms, kernel time per step {kern:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for s in range(20):
    step(s)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)

# idle gaps of the engine stream between consecutive kernels (KT_GAP_TRACE=1 to enable)
import os  # noqa: E402

if os.environ.get("KT_GAP_TRACE"):
    eng.set_timing(True)
    eng.kernel_stats(reset=True)
    for s in range(10):
        step(s)
    st = eng.kernel_stats(reset=True)
    eng.set_timing(False)
    print("per step (ms):")
    for k, (c, ms) in sorted(st.items(), key=lambda kv: -kv[1][1])[:24]:
        print(f"  {k:34s} {c / 10:5.1f}x {ms / 10:8.4f}")
