"""Where a wall-to-95% tuning round spends its time (bench.py's metric 2 loop, tune.tune_rows).

Wraps the per-round calls of tune.tune_rows (refit, SA round, adaptive sample, K3 measurement)
with host timers; a second pass synchronises the device after each call so device time is
attributed to the call that queued it.  Prints per-call totals over the five landscapes.
usage: python tools/w95_probe.py [--sync]
"""

from __future__ import annotations

import collections
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    import torch

    import bench
    import paper_1905_12799_b200 as kt
    from paper_1905_12799_b200 import tune
    from paper_1905_12799_b200.landscape import landscape_from_dict

    fx = bench.w95_fixture()
    space = kt.space_from_dict(fx["space"])
    eng = kt.engine(0)
    for sync in (False, True):
        acc = collections.defaultdict(lambda: [0, 0.0])
        orig = {}
        from paper_1905_12799_b200 import sa as sa_mod
        targets = [(tune, n) for n in ("fit", "run_sa_rows", "adaptive_sample_rows", "runtimes_rows",
                                       "random_unvisited")] + [(sa_mod, "device_forest")]
        for mod, name in targets:
            fn = getattr(mod, name)
            orig[(mod, name)] = fn

            def wrapped(*a, _fn=fn, _name=name, **k):
                t = time.perf_counter()
                out = _fn(*a, **k)
                if sync:
                    torch.cuda.synchronize()
                acc[_name][0] += 1
                acc[_name][1] += time.perf_counter() - t
                return out

            setattr(mod, name, wrapped)
        try:
            tune.tune_rows(space, landscape_from_dict(fx["landscapes"][0], space), bench.W95_STRATEGY, 100, 1,
                           engine=eng)
            acc.clear()
            total = 0.0
            rounds = 0
            for doc in fx["landscapes"]:
                land = landscape_from_dict(doc, space)
                fs = 1.0 / kt.best_runtime(land)[0]
                t = time.perf_counter()
                run = tune.tune_rows(space, land, bench.W95_STRATEGY, bench.W95_BUDGET, bench.W95_SEED, engine=eng,
                                     stop_fitness=0.95 * fs)
                total += time.perf_counter() - t
                rounds += run.rounds
        finally:
            for (mod, name), fn in orig.items():
                setattr(mod, name, fn)
        print(f"sync={sync}: {total * 1e3:.2f} ms over 5 landscapes, {rounds} rounds "
              f"({total / rounds * 1e6:.0f} us/round)")
        for name, (cnt, sec) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
            print(f"  {name:22s} {cnt:4d} calls {sec * 1e3:8.2f} ms  {sec / max(cnt, 1) * 1e6:8.1f} us/call")
        other = total - sum(v[1] for k, v in acc.items() if k != "device_forest")
        print(f"  {'(loop body / host)':22s}           {other * 1e3:8.2f} ms")

    # kernel time per round (engine CUDA-event timing; serialises launches, so only the split counts)
    lands = [landscape_from_dict(doc, space) for doc in fx["landscapes"]]
    fstars = [1.0 / kt.best_runtime(land)[0] for land in lands]
    eng.set_timing(True)
    eng.kernel_stats(reset=True)
    rounds = 0
    for land, fs in zip(lands, fstars):
        run = tune.tune_rows(space, land, bench.W95_STRATEGY, bench.W95_BUDGET, bench.W95_SEED, engine=eng,
                             stop_fitness=0.95 * fs)
        rounds += run.rounds
    stats = eng.kernel_stats(reset=True)
    eng.set_timing(False)
    tot = sum(v[1] for v in stats.values())
    print(f"kernels: {tot:.2f} ms over {rounds} rounds ({tot / rounds * 1e3:.0f} us/round)")
    for name, (cnt, ms) in sorted(stats.items(), key=lambda kv: -kv[1][1]):
        print(f"  {name:28s} {cnt:5d} launches {ms:8.3f} ms  {ms / cnt * 1e3:8.1f} us/launch")


if __name__ == "__main__":
    main()
