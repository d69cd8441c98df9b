"""Time one PPO search round (K1+K2+K4+K5) with E agents on the S2 space (GPU)."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1905_12799_b200 as kt
E = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
doc = json.loads((ROOT / "data/models/s2_resnet18.json").read_text())
space = kt.space_from_dict({"name": "s2", "knobs": [{"name": f"k{i}", "values": v} for i, v in enumerate(doc["values"])]})
model = kt.CostModel.from_dict(doc["model"])
agent = kt.init_agent(space, kt.AgentHyperparams(episodes_per_round=E), seed=0)
idx = np.random.default_rng(0).integers(0, np.array(space.cardinalities), size=(E, 8))
rows = torch.from_numpy(kt.pack(idx).view(np.int64)).cuda()
eng = kt.engine(0)
for rep in range(3):
    eng.set_timing(True)
    info = kt._lib.RoundInfo()
    torch.cuda.synchronize(); t = time.perf_counter()
    out = kt.run_search_rows(agent, model, space, rows, engine=eng, info=info)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    st = eng.kernel_stats(reset=True)
    top = sorted(st.items(), key=lambda kv: -kv[1][1])[:8]
    print(f"rep {rep}: {dt*1e3:.1f} ms wall, T={info.steps} N={info.entries}",
          {k: (c, round(ms, 3)) for k, (c, ms) in top})
