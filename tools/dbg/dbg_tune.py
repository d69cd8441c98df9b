import json, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_1905_12799_b200 as kt
from paper_1905_12799_b200 import tune, space as sp
from paper_1905_12799_b200.landscape import landscape_from_dict, runtimes_rows
G = json.load(open("tests/golden/tune.json")); SPACE = kt.space_from_dict(G["space"])
case = G["cases"][0]
land = landscape_from_dict(case["landscape"], SPACE)
cards = np.array(SPACE.cardinalities)
idx = np.array(case["indices"])
rows = torch.from_numpy(sp.pack(idx, cards).view(np.int64)).cuda()
rt = runtimes_rows(land, rows).cpu().numpy()
ref = np.array(case["runtimes"])
print("runtime mismatches (bitwise):", int((rt != ref).sum()), "max rel", float(np.max(np.abs(rt-ref)/ref)))
bad = np.nonzero(rt != ref)[0]; print("first bad idx", bad[:10])
run = tune.tune_rows(SPACE, land, "sa+as", 300, 0)
print("rounds", run.rounds, "sizes", [t[1] for t in run.trace][:20])
