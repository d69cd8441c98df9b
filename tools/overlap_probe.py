"""Does scoring (K2) overlap the sampler's dedup / k-means++ phase when it runs on a second engine?

Headline step (predict + adaptive_sample on 1M S2 candidates, visited set on), CUDA-event timed:
  serial      both on one engine (bench.py's value leg)
  overlapped  predict on engine B, adaptive_sample on engine A, both released by one start event
              and joined before the end event (the cooperative Lloyd launch waits for any SM K2
              still holds)
usage: python tools/overlap_probe.py [steps]
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch

    import paper_1905_12799_b200 as kt
    from paper_1905_12799_b200 import _lib
    from paper_1905_12799_b200 import space as sp

    K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    doc = json.loads((ROOT / "data/models/s2_resnet18.json").read_text())
    space = kt.space_from_dict({"name": "s2", "knobs": [{"name": f"k{i}", "values": v} for i, v in enumerate(doc["values"])]})
    model = kt.CostModel.from_dict(doc["model"])
    cards = np.array(space.cardinalities)
    N = 1 << 20
    sets = [torch.from_numpy(sp.pack(np.random.default_rng(s).integers(0, cards, size=(N, 8))).view(np.int64)).cuda()
            for s in range(4)]
    A = kt.engine(0)
    B = _lib.Engine(0)
    out = torch.empty(N, dtype=torch.float64, device="cuda")
    vis = np.zeros(0, np.uint64)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    s0, sa, sb = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for mode in ("serial", "overlapped", "serial", "overlapped"):
        ms = []
        for s in range(K + 2):
            flush.fill_(float(s))
            torch.cuda.synchronize()
            rows = sets[s % 4]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s0):
                e0.record(s0)
            if mode == "serial":
                with torch.cuda.stream(s0):
                    kt.predict_rows(model, space, rows, out=out, engine=A)
                    kt.adaptive_sample_rows(rows, vis, space, 1000 + s, engine=A)
            else:
                sb.wait_stream(s0)
                sa.wait_stream(s0)
                with torch.cuda.stream(sb):
                    kt.predict_rows(model, space, rows, out=out, engine=B)
                with torch.cuda.stream(sa):
                    kt.adaptive_sample_rows(rows, vis, space, 1000 + s, engine=A)
                s0.wait_stream(sa)
                s0.wait_stream(sb)
            with torch.cuda.stream(s0):
                e1.record(s0)
            torch.cuda.synchronize()
            if s >= 2:
                ms.append(e0.elapsed_time(e1))
        res.setdefault(mode, []).append(float(np.median(ms)))
        print(mode, "median %.4f ms/step" % np.median(ms), flush=True)


if __name__ == "__main__":
    main()
