"""Time K2 (predict_rows) on 1M uniform S2 candidates: median of 20 launches (CUDA events)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1905_12799_b200 as kt  # noqa: E402

doc = json.loads((ROOT / "data/models/s2_resnet18.json").read_text())
space = kt.space_from_dict({"name": "s2", "knobs": [{"name": f"k{i}", "values": v} for i, v in enumerate(doc["values"])]})
model = kt.CostModel.from_dict(doc["model"])
idx = np.random.default_rng(0).integers(0, np.array(space.cardinalities), size=(1 << 20, 8))
rows = torch.from_numpy(kt.pack(idx).view(np.int64)).cuda()
eng = kt.engine(0)
out = torch.empty(rows.numel(), dtype=torch.float64, device="cuda")
ms = []
for r in range(25):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with eng.scope():
        a.record(eng.stream)
    kt.predict_rows(model, space, rows, out=out, engine=eng)
    with eng.scope():
        b.record(eng.stream)
    torch.cuda.synchronize()
    if r >= 5:
        ms.append(a.elapsed_time(b))
print(f"score_trees 1M: {np.median(ms) * 1e3:.1f} us, checksum {float(out.sum()):.17g}")
