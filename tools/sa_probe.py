"""One tuning-round SA launch (64 chains x 128 steps on the S2 surrogate) for ncu: python tools/sa_probe.py"""
import json
import sys
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
chains = int(sys.argv[1]) if len(sys.argv) > 1 else 64
starts = torch.from_numpy(sp.pack(np.random.default_rng(1).integers(0, cards, size=(chains, 8))).view(np.int64)).cuda()
eng = kt.engine(0)
for s in range(3):
    rows, _, _ = kt.run_sa_rows(kt.SAParams(chains=chains, steps_per_round=128), model, space, starts, seed=5 + s,
                                engine=eng)
torch.cuda.synchronize()
print("entries", int(rows.numel()))
