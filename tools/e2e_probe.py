"""Where the headline's end-to-end leg loses time against the device-resident leg.

Runs the headline step (predict + adaptive_sample on 1M S2 candidates, mode vote on) as one
continuous CUDA-event-timed region of K steps in variants:
  full      pinned-host rows H2D + scores D2H (bench.py's e2e loop)
  no_d2h    H2D only
  resident  rows already on the device, no copies (same continuous region)
  flushed   resident, 512 MiB L2 flush between steps inside the region (bench.py's value leg
            keeps the flush outside its per-step events)
  chunked   full, the scores' D2H split into 16 copies
  zerocopy  H2D rows; predict writes the scores straight into pinned host memory (UVA), no D2H
  prio      full, the engine on a high-priority stream and the D2H on a low-priority one
  late      full, but step s's scores D2H is issued once step s's clustering has returned
usage: python tools/e2e_probe.py [steps]
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch

    import bench
    import paper_1905_12799_b200 as kt
    from paper_1905_12799_b200 import space as sp

    K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    eng = kt.engine(0)
    doc = bench.load_model()
    space = kt.space_from_dict({"name": doc["space"], "knobs": [{"name": f"k{i}", "values": v}
                                                                  for i, v in enumerate(doc["values"])]})
    model = kt.CostModel.from_dict(doc["model"])
    cards = np.array(space.cardinalities)
    N = 1 << 20
    host = [torch.from_numpy(sp.pack(bench.candidates(N, s, cards)).view(np.int64)).pin_memory() for s in range(4)]
    dev = [h.to("cuda:0") for h in host]
    vis = {}
    for s in range(K):
        kt.predict_rows(model, space, dev[s % 4], engine=eng)
        nv = kt.adaptive_sample_rows(dev[s % 4], np.zeros(0, np.uint64), space, 2000 + s, engine=eng)
        vis[s] = bench.bench_visited_rows(nv, host[s % 4].numpy())
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
    copy_stream, d2h_plain = torch.cuda.Stream(), torch.cuda.Stream()
    lo_stream, hi_stream = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
    eng_stream0 = eng.stream
    bufs = [torch.empty(N, dtype=torch.int64, device="cuda:0") for _ in range(3)]
    sbufs = [torch.empty(N, dtype=torch.float64, device="cuda:0") for _ in range(2)]
    hs = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(2)]

    def run(variant: str) -> float:
        ready = [torch.cuda.Event() for _ in range(3)]
        scored = [torch.cuda.Event() for _ in range(2)]
        drained = [torch.cuda.Event() for _ in range(2)]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        copies = variant in ("full", "no_d2h", "chunked", "zerocopy", "prio", "late")
        d2h = variant in ("full", "chunked", "prio", "late")
        d2h_stream = lo_stream if variant == "prio" else d2h_plain
        eng.set_stream(hi_stream if variant == "prio" else eng_stream0)

        def rows(s):
            return bufs[s % 3] if copies else dev[s % 4]

        def upload(s):
            if copies:
                with torch.cuda.stream(copy_stream):
                    bufs[s % 3].copy_(host[s % 4], non_blocking=True)
                    ready[s % 3].record(copy_stream)

        def score(s):
            i = s % 2
            if copies:
                eng.stream.wait_event(ready[s % 3])
            if s >= 2 and (d2h or variant == "zerocopy"):
                eng.stream.wait_event(drained[i])
            if variant == "zerocopy":
                kt.predict_rows(model, space, rows(s), out=hs[i], engine=eng)
                with eng.scope():
                    drained[i].record(eng.stream)
                return
            kt.predict_rows(model, space, rows(s), out=sbufs[i], engine=eng)
            if d2h:
                with eng.scope():
                    scored[i].record(eng.stream)
                if variant != "late":
                    drain(s)

        def drain(s):
            i = s % 2
            if True:
                with torch.cuda.stream(d2h_stream):
                    d2h_stream.wait_event(scored[i])
                    if variant == "chunked":
                        for c in range(16):
                            sl = slice(c * (N // 16), (c + 1) * (N // 16))
                            hs[i][sl].copy_(sbufs[i][sl], non_blocking=True)
                    else:
                        hs[i].copy_(sbufs[i], non_blocking=True)
                    drained[i].record(d2h_stream)

        torch.cuda.synchronize()
        with eng.scope():
            a.record(eng.stream)
        for s in range(min(2, K)):
            upload(s)
        score(0)
        for s in range(K):
            if s + 1 < K:
                score(s + 1)
            if s + 2 < K:
                upload(s + 2)
            kt.adaptive_sample_rows(rows(s), vis[s], space, 2000 + s, engine=eng)
            if variant == "late":
                drain(s)
            if variant == "flushed":
                with eng.scope():
                    flush.fill_(float(s))
        with eng.scope():
            eng.stream.wait_stream(copy_stream)
            eng.stream.wait_stream(d2h_stream)
            b.record(eng.stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / K

    for v in ("full", "no_d2h", "resident", "flushed", "chunked", "zerocopy", "prio", "late", "full", "resident"):
        run(v)  # warm
        ms = sorted(run(v) for _ in range(3))[1]
        print(f"{v:10s} {ms:.4f} ms/step  {N / ms * 1e3:.3e} cand/s")


if __name__ == "__main__":
    main()
