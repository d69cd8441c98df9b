"""Time one adaptive_sample on N uniform S2 candidates and print engine kernel stats (GPU)."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1905_12799_b200 as kt
from paper_1905_12799_b200 import space as sp
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
doc = json.loads((ROOT / "data/models/s2_resnet18.json").read_text())
space = kt.space_from_dict({"name": "s2", "knobs": [{"name": f"k{i}", "values": v} for i, v in enumerate(doc["values"])]})
idx = np.random.default_rng(0).integers(0, np.array(space.cardinalities), size=(N, 8))
rows = torch.from_numpy(sp.pack(idx).view(np.int64)).cuda()
eng = kt.engine(0)
for rep in range(3):
    eng.set_timing(True)
    info = kt._lib.SampleInfo()
    t = time.perf_counter()
    kt.adaptive_sample_rows(rows, np.zeros(0, np.uint64), space, 7, engine=eng, info=info)
    dt = time.perf_counter() - t
    st = eng.kernel_stats(reset=True)
    print(f"rep {rep}: {dt*1e3:.2f} ms wall, k={info.chosen_k}, passes={info.lloyd_passes}",
          {k: round(v[1], 3) for k, v in st.items()})
