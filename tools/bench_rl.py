"""bench.py --workload rl: the PPO + adaptive-sampling tuning step of configs[1].

Per step and rank: AlexNet's 5 conv tasks (workloads.ALEXNET_TASKS; surrogates
and landscapes in data/models/alexnet_task*.json), each runs one search round
with 4096 PPO agents (K1 rollout, K2 scoring, K4 GAE, K5 PPO update) followed by
adaptive_sample on its trajectory (K6/K7/K8/K9).  Metric: trajectory candidates
scored + clustered per second.  The tasks are independent (configs[1]), so each runs on its own
engine (stream) from its own host thread: one task's host-side work and latency-bound kernels
overlap the others' (~22 ms/step against ~26-28 in sequence; --rl-serial: one engine, tasks in
sequence).  Running them concurrently exposed a real race, since fixed: the rollout kernel's
warps could poll its TMA mbarrier before thread 0 had initialised it.  conv3/conv4 have tile_f cardinality 480, so
their rows use the bit-field layout (space.row_layout).
"""

from __future__ import annotations

import json
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
N_TASKS, AGENTS = 5, 4096


def task_docs():
    return [json.loads((ROOT / "data" / "models" / f"alexnet_task{i}.json").read_text()) for i in range(N_TASKS)]


def cpu_rl_step(docs, rng_seed: int, agents: int):
    """Reference algorithm (oracle numpy port) for one step on `agents` agents per task."""
    from oracle import agent as oagent
    from oracle import sampler as osamp

    n_cand = 0
    for i, d in enumerate(docs):
        cards = np.array([len(v) for v in d["values"]])
        hyper = dict(oagent.DEFAULT_HYPER, episodes_per_round=agents)
        ag = oagent.new_agent(len(cards), hyper, seed=i)
        starts = np.random.default_rng(rng_seed + i).integers(0, cards, size=(agents, cards.size))
        idx, scores, steps = oagent.search_round(ag, d["model"], d["values"], starts, hyper)
        osamp.adaptive_sample(idx, set(), cards.tolist(), rng_seed + i)
        n_cand += len(idx)
    return n_cand


def run(args, rank: int, world: int, local_rank: int, kt, torch, dist, helpers) -> dict | None:
    """GPU arm; returns the JSON line (rank 0) or None."""
    import threading

    sp = kt.space
    docs = task_docs()
    eng = kt.engine(local_rank)
    serial = bool(getattr(args, "rl_serial", False))
    engines = [eng] * N_TASKS if serial else [eng] + [kt._lib.Engine(local_rank) for _ in range(N_TASKS - 1)]
    dev = f"cuda:{local_rank}"
    tasks = []
    for i, d in enumerate(docs):
        space = kt.space_from_dict({"name": d["space"], "knobs": [{"name": f"k{j}", "values": v}
                                                                   for j, v in enumerate(d["values"])]})
        model = kt.CostModel.from_dict(d["model"])
        agent = kt.init_agent(space, kt.AgentHyperparams(episodes_per_round=AGENTS), seed=1000 * rank + i)
        cards = np.array(space.cardinalities)
        host_starts = [torch.from_numpy(sp.pack(np.random.default_rng(100 * rank + 10 * i + s)
                                                .integers(0, cards, size=(AGENTS, cards.size)), cards).view(np.int64))
                       .pin_memory() for s in range(2)]
        tasks.append((space, model, agent, host_starts))
    no_visited = np.zeros(0, dtype=np.uint64)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def task_step(i, s, out, infos):
        space, model, agent, host_starts = tasks[i]
        e = engines[i]
        with torch.cuda.stream(e.stream):  # this thread's current stream = its engine's
            with e.scope():
                starts = host_starts[s % 2].to(dev, non_blocking=True)
            rows, scores, _ = kt.run_search_rows(agent, model, space, starts, engine=e)
            info = kt._lib.SampleInfo() if infos is not None else None
            batch = kt.adaptive_sample_rows(rows, no_visited, space, seed=s, engine=e, info=info)
        if infos is not None:
            infos[i] = {"entries": int(rows.numel()), "distinct": int(info.n_distinct), "k": int(info.chosen_k),
                        "lloyd_passes": int(info.lloyd_passes), "lloyd_launches": int(info.lloyd_launches)}
        out[i] = (int(rows.numel()), batch.nbytes)

    def step(s, e2e_batch=None, infos=None):
        """One step of all tasks, ordered after the caller's stream and joined back into it."""
        main = torch.cuda.current_stream(local_rank)
        go = torch.cuda.Event()
        go.record(main)
        for e in set(engines):
            e.stream.wait_event(go)
        out = [None] * N_TASKS
        if serial:
            for i in range(N_TASKS):
                task_step(i, s, out, infos)
        else:
            errs = []

            def body(i):
                try:
                    task_step(i, s, out, infos)
                except BaseException as ex:  # pragma: no cover - surfaced below
                    errs.append(ex)

            th = [threading.Thread(target=body, args=(i,)) for i in range(N_TASKS)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            if errs:
                raise errs[0]
        for e in set(engines):
            done = torch.cuda.Event()
            done.record(e.stream)
            main.wait_event(done)
        if e2e_batch is not None:
            e2e_batch.extend(b for _, b in out)
        return sum(c for c, _ in out)

    for w in range(args.warmup):
        step(w)
    helpers["barrier"]()
    uniq = list({id(e): e for e in engines}.values())
    launches0 = sum(e.launches for e in uniq)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    n_total = 0
    d2h = []
    main = torch.cuda.current_stream(local_rank)
    with helpers["clock"](local_rank) as clk:
        helpers["barrier"]()
        for s in range(args.steps):
            flush.fill_(float(s))
            ev[s][0].record(main)
            n_total += step(s, d2h)
            ev[s][1].record(main)
        helpers["barrier"]()
    launches = sum(e.launches for e in uniq) - launches0
    t = sum(a.elapsed_time(b) for a, b in ev) / 1e3
    # per-kernel device times: one serial step (the engines' timing events would overlap otherwise)
    for e in uniq:
        e.set_timing(True)
        e.kernel_stats(reset=True)
    infos = [None] * N_TASKS
    serial_saved, serial = serial, True
    step(0, infos=infos)
    serial = serial_saved
    stats = {}
    for e in uniq:
        for k, (c, ms) in e.kernel_stats(reset=True).items():
            c0, m0 = stats.get(k, (0, 0.0))
            stats[k] = (c0 + c, m0 + ms)
        e.set_timing(False)
    times = torch.tensor([t, float(n_total)], dtype=torch.float64, device=dev)
    if dist is not None:
        tt = times.clone()
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        nn = times.clone()
        dist.all_reduce(nn, op=dist.ReduceOp.SUM)
        t, n_total = float(tt[0]), float(nn[1])
    if rank != 0:
        return None
    value = n_total / t
    # host-to-device starts and device-to-host batches are inside the timed region (e2e == value here)
    base = None
    if not args.no_cpu_baseline:
        t0 = time.perf_counter()
        nc = cpu_rl_step(docs, 7, 256)
        dt = time.perf_counter() - t0
        base = {"value": nc / dt, "unit": "candidates/s", "cores": 1, "kind": "port",
                "sample": f"{N_TASKS} tasks x 256 agents (oracle numpy port of run_search_round + adaptive_sample), "
                          f"{dt:.1f} s"}
    # PPO GEMM roofline (tensor): algorithmic fp32 FLOPs of the 3 epochs' forward, data-gradient and
    # weight-gradient GEMMs (n = knobs, h = 128 shared, 2g = 128 heads, 3n + 1 outputs) over the
    # tc_gemm kernels' time; they run as 3xTF32 (three tf32 MMAs per fp32 product)
    gemm_ms = sum(ms for k, (c, ms) in stats.items() if k.startswith("tc_gemm"))
    flops = 0.0
    for d, inf in zip(docs, infos):
        n = len(d["values"])
        macs = (n * 128 + 128 * 128 + 128 * (3 * n + 1)) + ((3 * n + 1) * 128 + 128 * 128) + \
               ((3 * n + 1) * 128 + 128 * 128 + 128 * n)
        flops += 3 * 2.0 * macs * (inf["entries"] - AGENTS)  # 3 epochs, T = entries - agents rows
    pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else None
    tf32_peak = (float(pk["bf16_tflops"]) / 2.0) if pk else 1100.0
    gemm_tflops = flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else None
    gemm_roof = {"bound": "tensor", "kernel": "tc_gemm (fwd + dgrad + wgrad, 3xTF32)", "achieved": gemm_tflops,
                 "peak": tf32_peak, "unit": "TFLOP/s", "frac": gemm_tflops / tf32_peak if gemm_tflops else None,
                 "tensor_work_frac": 3 * gemm_tflops / tf32_peak if gemm_tflops else None, "traffic": None,
                 "peak_source": "MEASURED_PEAKS bf16 / 2 (dense tf32)" if pk else "fallback 1.1 PF tf32",
                 "flops_model": "2 * 60.8K MACs per trajectory row per epoch (8 knobs), 3 epochs, fp32-equivalent",
                 "gemm_ms_per_step": gemm_ms, "kernel_share_of_step": gemm_ms / sum(ms for _, ms in stats.values())}
    dom = max(stats.items(), key=lambda kv: kv[1][1])
    return {
        "metric": "candidate configs scored+clustered/sec per tuning step", "value": value, "unit": "candidates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+fp32/tf32", "data": "synthetic",
        "config": {"workload": f"AlexNet's {N_TASKS} conv tasks x {AGENTS} PPO agents per step: run_search_round "
                               f"(rollout, scoring, GAE, 3 PPO epochs) + adaptive_sample per task",
                   "tasks": "serial on one engine" if serial else f"{N_TASKS} engines (streams) + host threads, concurrent",
                   "candidates_per_step": n_total / args.steps / world, "parallelism": f"tasks x{world}",
                   "l2": "flushed between steps"},
        "e2e": {"value": value, "unit": "candidates/s", "h2d_bytes_per_step": N_TASKS * AGENTS * 8,
                "d2h_bytes_per_step": int(sum(d2h) / max(1, args.steps))},
        "gpu_launches": int(launches),
        "sample_info": infos,
        "kernels": {k: {"launches": c, "ms": round(ms, 3)} for k, (c, ms) in sorted(stats.items(), key=lambda kv: -kv[1][1])},
        "roofline": gemm_roof,
        "dominant_single_kernel": dom[0],
        "clocks": clk.summary(), "cpu_baseline": base,
    }
