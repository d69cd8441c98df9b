"""bench.py --workload c4: configs[3] — ResNet-18's 12 tuning tasks, 1M candidates per task per step,
placed over the ranks with shard.place_tasks (whole tasks round-robin; the remainder tasks split into
candidate shards over groups of ranks, whose adaptive_sample runs sharded: NCCL all-gather of the
candidate rows, one int64 all-reduce per Lloyd pass).  One rank runs all 12 tasks.

Per task the surrogate is the native refit (kt.fit) on 500 random configurations of a smooth synthetic
fitness surface (deterministic per task); candidates are uniform over the task's space.  value = 12M
candidates per step / step time (max over ranks).
"""

from __future__ import annotations

import numpy as np

N_CAND = 1 << 20


def build_tasks(kt, sp, wl):
    tasks = []
    for ti, t in enumerate(wl.RESNET18_TASKS):
        space = sp.space_from_dict(t.space_dict())
        cards = np.array(space.cardinalities)
        rng = np.random.default_rng(10 + ti)
        table, _ = kt.cost_model.feature_table(space)
        tr = rng.integers(0, cards, size=(500, cards.size))
        X = table[np.arange(cards.size), tr]

        class _TS:
            features = X
            targets = 1.0 / (0.5 + np.abs(np.sin(X.sum(axis=1) + ti)))

        model = kt.fit(_TS, kt.BoostParams())
        cand = sp.pack(rng.integers(0, cards, size=(N_CAND, cards.size)), cards)
        tasks.append((t.name, space, model, cand))
    return tasks


def run(args, rank: int, world: int, local_rank: int, kt, torch, dist, helpers) -> dict | None:
    from paper_1905_12799_b200 import shard
    from paper_1905_12799_b200 import space as sp
    from paper_1905_12799_b200 import workloads as wl

    eng = kt.engine(local_rank)
    dev = f"cuda:{local_rank}"
    tasks = build_tasks(kt, sp, wl)
    plan = shard.place_tasks(len(tasks), world)
    groups = {}
    if world > 1:  # every rank creates every shard group, in the same order
        for p in plan:
            for _, _, n_sh, grp in p.shards:
                if n_sh > 1 and grp not in groups:
                    groups[grp] = None
        for grp in list(groups):
            groups[grp] = dist.new_group(ranks=list(grp))
    mine = []
    for task, i, n_sh, grp in plan[rank].shards:
        name, space, model, cand = tasks[task]
        lo, hi = shard.shard_range(len(cand), i, n_sh)
        rows = torch.from_numpy(cand[lo:hi].view(np.int64)).to(dev)
        mine.append((name, space, model, rows, n_sh, groups.get(grp)))
    vis = np.zeros(0, dtype=np.uint64)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    outs = [torch.empty(m[3].numel(), dtype=torch.float64, device=dev) for m in mine]

    def step(s):
        for (name, space, model, rows, n_sh, pg), out in zip(mine, outs):
            kt.predict_rows(model, space, rows, out=out, engine=eng)
            if n_sh == 1:
                kt.adaptive_sample_rows(rows, vis, space, seed=1000 + s, engine=eng)
            else:
                shard.adaptive_sample_sharded(rows, vis, space, seed=1000 + s, group=pg)

    for w in range(args.warmup):
        step(w)
    helpers["barrier"]()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = eng.launches
    with helpers["clock"](local_rank) as clk:
        for s in range(args.steps):
            flush.fill_(float(s))
            helpers["barrier"]()  # every step starts together (sharded tasks exchange inside it)
            with eng.scope():
                ev[s][0].record(eng.stream)
            step(s)
            with eng.scope():
                ev[s][1].record(eng.stream)
        helpers["barrier"]()
    launches = eng.launches - launches0
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / 1e3], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t = float(t[0])
    if rank != 0:
        return None
    total = len(tasks) * N_CAND * args.steps
    value = total / t
    return {
        "metric": "candidate configs scored+clustered/sec per tuning step", "value": value, "unit": "candidates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "configs[3]: ResNet-18's 12 tasks x 1,048,576 uniform candidates per task per step "
                               "(predict + adaptive_sample); tasks placed by shard.place_tasks, remainder tasks "
                               "candidate-sharded with sharded k-means",
                   "candidates_per_step": len(tasks) * N_CAND, "parallelism": f"{world} ranks",
                   "placement_rank0": [list(x[:3]) for x in plan[0].shards],
                   "l2": "flushed between steps (512 MiB write, outside the timed events)"},
        "e2e": None, "gpu_launches": int(launches), "clocks": clk.summary(),
    }
