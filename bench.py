#!/usr/bin/env python
"""Benchmark: candidate configs scored + clustered per second per tuning step (BASELINE.json metric).

Step = one pass of the search-step hot path over one batch of candidates of
the ResNet-18 3x3 64->64 56x56 conv space (S2, 90.3M configs):
    K2 surrogate scoring (50 depth-4 boosted trees)  ->  K6 first-occurrence dedup
    ->  K7/K8 knee k-means (k = 8, 9, ... until the knee)  ->  K9 mode / batch assembly
exactly as predict() + adaptive_sample() compute it in the reference.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--candidates 1048576]

N>1 runs under torchrun: one process per GPU, each rank tunes its own task
(weak scaling, no data-path collective); time = max over ranks.
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "candidate configs scored+clustered/sec per tuning step"
UNIT = "candidates/s"
WORKLOAD = ("resnet18.c2_3x3_64x64_56 space (S2: 84x80x80x7x2x2x3x2 = 90,316,800 configs); per step {n} "
            "uniform candidates -> K2 boosted-tree scores (50 trees, depth 4) + K6 dedup + K7/K8 knee k-means "
            "(k=8..knee, seeded) + K9 mode vote + batch (predict + adaptive_sample); visited set per step = two of "
            "the step's own rounded centroids (measured in an earlier round) + 62 earlier measurements, so batch "
            "assembly takes the reference's mode branch (sampler.py:203-209) every step")
GOLDEN = ROOT / "tests" / "golden" / "bench_golden.json"
TRAFFIC_ROUND = "r2"  # profiles/<round>/traffic.json: ncu --set full DRAM bytes per launch


def load_model():
    doc = json.loads((ROOT / "data" / "models" / "s2_resnet18.json").read_text())
    return doc


def candidates(n: int, seed: int, cards: np.ndarray) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, cards, size=(n, cards.size))


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------- CPU side
def bench_visited_rows(batch_rows: np.ndarray, cand_rows: np.ndarray) -> np.ndarray:
    """The step's visited set (packed rows): the first two configurations of the step's own batch
    without a visited set (rounded centroids 0 and 1, as if measured in an earlier round) and the
    first 62 candidates, first occurrence kept — tests/golden/make_bench_golden.py:bench_visited."""
    out, seen = [], set()
    for r in list(np.asarray(batch_rows, dtype=np.uint64)[:2]) + list(np.asarray(cand_rows).view(np.uint64)[:62]):
        if int(r) not in seen:
            seen.add(int(r))
            out.append(int(r))
    return np.array(out, dtype=np.uint64)


def cpu_step(doc, idx: np.ndarray, seed: int, visited_rows: bool = True):
    from oracle import sampler as osamp
    from oracle import trees as otrees

    cards = [len(v) for v in doc["values"]]
    scores = otrees.predict_features(doc["model"], otrees.featurize_rows(doc["values"], idx))
    batch, info = osamp.adaptive_sample(idx, set(), cards, seed, return_info=True)
    if visited_rows and "result" in info:  # same visited construction as the GPU arm: mode branch
        visited = {tuple(b) for b in batch[:2]} | {tuple(r) for r in idx[:62].tolist()}
        batch, _ = osamp.assemble_batch(info["result"]["centroids"], idx, visited, cards)
    return scores, batch


def cpu_baseline(doc, cards, n_sample: int, reps: int = 1, full: int = 0) -> dict:
    idx = candidates(n_sample, 12345, cards)
    t0 = time.perf_counter()
    for r in range(reps):
        cpu_step(doc, idx, 7 + r)
    dt = (time.perf_counter() - t0) / reps
    out = {"value": n_sample / dt, "unit": UNIT, "cores": 1, "kind": "port",
           "sample": f"{n_sample} uniform S2 candidates per step (oracle/ numpy restatement of "
                     f"predict_features + adaptive_sample, single-threaded), {reps} step(s), {dt:.2f} s/step"}
    if full:
        out["full_size"] = cpu_full_size(doc, cards, full)
    return out


def cpu_full_size(doc, cards, n: int) -> dict:
    """One step of the headline workload at its full size through the port on one core (~2 min)."""
    idx = candidates(n, 0, cards)
    t0 = time.perf_counter()
    cpu_step(doc, idx, 1000)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "port", "candidates": n, "seconds": dt,
            "sample": f"one full headline step: {n} uniform S2 candidates (rank 0's first set, seed 1000), "
                      f"oracle numpy port, single-threaded"}


# ------------------------------------------------- wall time to 95% best (metric 2)
W95_STRATEGY, W95_BUDGET, W95_SEED = "sa+as", 1000, 0


def w95_fixture():
    return json.loads((ROOT / "data" / "landscapes" / "bench_grid4d.json").read_text())


def f_star(land_doc, values) -> float:
    """1 / enumerated optimum runtime (the 10^4-config fixture space is brute-forced on the host)."""
    from oracle.landscape import synthetic_runtimes  # bench reference arm / baseline leg only

    grid = np.indices(tuple(len(v) for v in values)).reshape(len(values), -1).T
    return 1.0 / float(np.min(synthetic_runtimes(land_doc, grid)))


def w95_summary(per: list, impl: str, cores: int) -> dict:
    reached = [r["seconds_to_95"] for r in per if r["seconds_to_95"] is not None]
    return {"metric": "wall time to 95% best", "unit": "s", "higher_is_better": False,
            "value": float(np.mean(reached)) if reached else None, "reached": f"{len(reached)}/{len(per)}",
            "strategy": W95_STRATEGY, "budget": W95_BUDGET, "seed": W95_SEED,
            "workload": "reference fixture space bench_grid4d (10^4 configs) x its 5 synthetic landscapes; f* = "
                        "enumerated optimum; value = mean over landscapes of seconds from tune start until best-so-far "
                        "fitness >= 0.95 f* (the tune stops there)", "impl": impl, "cores": cores, "per_landscape": per}


def w95_ours(engine) -> dict:
    import paper_1905_12799_b200 as kt
    from paper_1905_12799_b200 import tune
    from paper_1905_12799_b200.landscape import landscape_from_dict

    fx = w95_fixture()
    space = kt.space_from_dict(fx["space"])
    tune.tune_rows(space, landscape_from_dict(fx["landscapes"][0], space), W95_STRATEGY, 100, 1, engine=engine)  # warm
    per = []
    for i, doc in enumerate(fx["landscapes"]):
        land = landscape_from_dict(doc, space)
        fs = 1.0 / kt.best_runtime(land)[0]
        run = tune.tune_rows(space, land, W95_STRATEGY, W95_BUDGET, W95_SEED, engine=engine, stop_fitness=0.95 * fs)
        per.append({"landscape": i, "seconds_to_95": run.wall_to_fraction(fs, 0.95), "tune_seconds": run.seconds,
                    "rounds": run.rounds, "best_over_fstar": run.best_fitness / fs,
                    "measurements_to_95": next((m for _, m, b in run.trace if b >= 0.95 * fs), None)})
    return w95_summary(per, "ours (B200)", 1)


def _w95_ref_job(i):
    from oracle import tune as otune

    fx = w95_fixture()
    values = [k["values"] for k in fx["space"]["knobs"]]
    doc = fx["landscapes"][i]
    fs = f_star(doc, values)
    configs, rts, trace, rounds = otune.tune(values, doc, W95_STRATEGY, W95_BUDGET, W95_SEED, stop_fitness=0.95 * fs)
    t95 = next((t for t, _, b in trace if b >= 0.95 * fs), None)
    return {"landscape": i, "seconds_to_95": t95, "tune_seconds": trace[-1][0], "rounds": rounds,
            "best_over_fstar": max(1.0 / r for r in rts) / fs,
            "measurements_to_95": next((m for _, m, b in trace if b >= 0.95 * fs), None)}


def w95_reference() -> dict:
    import multiprocessing as mp

    n = len(w95_fixture()["landscapes"])
    with mp.get_context("fork").Pool(n) as pool:
        per = pool.map(_w95_ref_job, range(n))
    return w95_summary(per, "reference algorithm (oracle numpy port), one host process per landscape", n)


def _ref_job(job):
    n, cand_seed, seed = job
    doc = load_model()
    cards = np.array([len(v) for v in doc["values"]])
    cpu_step(doc, candidates(n, cand_seed, cards), seed)


def run_reference(args, rank: int, world: int) -> None:
    """--impl reference: the reference's CPU algorithm (oracle port; the reference itself is pure Python
    and /root/reference does not exist on the GPU box) on the host cores, rank 0 only."""
    if rank != 0:
        return
    import multiprocessing as mp

    doc = load_model()
    cards = np.array([len(v) for v in doc["values"]])
    n = args.ref_sample
    procs = args.ref_procs or len(os.sched_getaffinity(0))
    cpu_step(doc, candidates(n, 1, cards), 100)  # warm caches / imports in the parent
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_ref_job, [(n, 100 + w, 100 + w) for w in range(max(args.warmup, 1) * procs)][:procs])
        t0 = time.perf_counter()
        pool.map(_ref_job, [(n, 1000 + s, 200 + s) for s in range(args.steps * procs)])
        wall = time.perf_counter() - t0
    dt = wall / args.steps  # wall time per round of `procs` concurrent steps
    value = n * procs / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD.format(n=n), "candidates_per_step": n,
                   "parallelism": f"{procs} host processes, one independent task each",
                   "same_config": False,
                   "sample_vs_headline": f"bounded sample: {n} of the headline's {args.candidates} candidates per step "
                                         f"(the port's per-candidate rate falls as the size grows, so this favours "
                                         f"the CPU); cpu_baseline.full_size is one step at the headline size"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": f"{n} uniform S2 candidates per step per process, oracle numpy port "
                                   f"(predict_features + adaptive_sample), {procs} processes x {args.steps} steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu_full:  # one full-size step (the GPU arm's per-step workload) on one core
        line["cpu_baseline"]["full_size"] = cpu_full_size(doc, cards, args.candidates)
    if not args.no_wall95:
        line["wall_to_95"] = w95_reference()
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU side
def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch

    import paper_1905_12799_b200 as kt
    from paper_1905_12799_b200 import space as sp

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    eng = kt.engine(local_rank)
    doc = load_model()
    space = kt.space_from_dict({"name": doc["space"], "knobs": [{"name": f"k{i}", "values": v}
                                                                  for i, v in enumerate(doc["values"])]})
    model = kt.CostModel.from_dict(doc["model"])
    cards = np.array(space.cardinalities)
    N = args.candidates
    no_visited = np.zeros(0, dtype=np.uint64)

    # inputs: one distinct candidate set per step (and per rank), pinned on the host and resident on the device
    n_sets = max(2, min(args.steps, 4))
    host_sets = []
    for s in range(n_sets):
        rows = sp.pack(candidates(N, 10_000 * rank + s, cards)).view(np.int64)
        host_sets.append(torch.from_numpy(rows).pin_memory())
    dev = f"cuda:{local_rank}"
    dev_sets = [h.to(dev) for h in host_sets]
    scores_buf = torch.empty(N, dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step(rows_dev, seed, visited=no_visited, info=None, out=scores_buf):
        kt.predict_rows(model, space, rows_dev, out=out, engine=eng)
        return kt.adaptive_sample_rows(rows_dev, visited, space, seed, engine=eng, info=info)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    # untimed: each step's visited set, built from the same step computed without one ("an earlier
    # round measured two of these centroids"), so every timed step runs the mode vote (K9)
    visited_for = {}
    for base in (1000, 2000):
        for s in range(args.steps):
            nv = step(dev_sets[s % n_sets], base + s)
            visited_for[base + s] = bench_visited_rows(nv, host_sets[s % n_sets].numpy())
    for w in range(args.warmup):
        step(dev_sets[w % n_sets], 1000 + w, visited_for[1000 + w % args.steps])

    # parity self-check (untimed) on rank 0's first set against the oracle golden of this exact step
    parity = None
    if rank == 0 and N == 1 << 20 and GOLDEN.exists():
        g = json.loads(GOLDEN.read_text())["s2"]
        pinfo = kt._lib.SampleInfo()
        b0 = sp.unpack(step(dev_sets[0], g["seed"], info=pinfo), 8).tolist()
        curve = [[pinfo.scanned_k[i], float(pinfo.scanned_loss[i]).hex()] for i in range(pinfo.n_scanned)]
        vis = sp.pack(np.array(g["visited"], dtype=np.int64))
        vinfo = kt._lib.SampleInfo()
        b1 = sp.unpack(step(dev_sets[0], g["seed"], vis, info=vinfo), 8).tolist()
        checks = {"distinct": pinfo.n_distinct == g["m"], "curve": curve == g["curve"], "batch": b0 == g["batch"],
                  "batch_with_visited": b1 == g["batch_visited"], "mode_vote_ran": bool(vinfo.used_mode)}
        parity = {"ok": all(checks.values()), **checks,
                  "golden": "tests/golden/bench_golden.json[s2] (oracle, candidate seed 0, adaptive_sample seed 1000)"}
    barrier()

    # ---- timed region 1: device-resident inputs (value)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = eng.launches
    infos = []
    with ClockSampler(local_rank) as clk:
        barrier()
        for s in range(args.steps):
            flush.fill_(float(s))  # L2 flush, outside the timed events
            with eng.scope():
                ev[s][0].record(eng.stream)
            info = kt._lib.SampleInfo()
            step(dev_sets[s % n_sets], 1000 + s, visited_for[1000 + s], info)
            with eng.scope():
                ev[s][1].record(eng.stream)
            infos.append(info)
        barrier()
    launches = eng.launches - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_total = sum(step_ms) / 1e3

    # ---- timed region 2: end to end through the public API with host buffers.  One continuous
    # region over K steps: every step's candidate rows come from pinned host memory (a fresh H2D
    # copy, never reused on the device), its float64 scores (predict's return value, 8 B per
    # candidate) and its batch go back to the host.  Pipelined as a tuning service runs it: step
    # s+1's scoring is queued on the engine stream ahead of step s's clustering (so the GPU scores
    # while the host returns from one adaptive_sample and launches the next), the H2D of step s+2
    # runs on one copy stream and the scores' D2H on another; rows are triple-buffered, scores
    # double-buffered, every reuse ordered by events.  (Scoring on a second engine concurrently
    # with the clustering was measured slower: the resident Lloyd launch waits for the SMs the
    # scoring kernel holds.)
    copy_stream = torch.cuda.Stream(device=dev)  # H2D of upcoming steps' candidates
    d2h_stream = torch.cuda.Stream(device=dev)   # D2H of the scores
    bufs = [torch.empty(N, dtype=torch.int64, device=dev) for _ in range(3)]
    sbufs = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(2)]
    host_scores = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(3)]    # rows of a step on the device
    scored = [torch.cuda.Event() for _ in range(2)]
    drained = [torch.cuda.Event() for _ in range(2)]  # scores of a step copied out: sbufs free again
    e2e_start, e2e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def upload(s):  # bufs[s % 3] was last read by step s-3, whose clustering has returned
        with torch.cuda.stream(copy_stream):
            bufs[s % 3].copy_(host_sets[s % n_sets], non_blocking=True)
            ready[s % 3].record(copy_stream)

    def score(s):
        i = s % 2
        eng.stream.wait_event(ready[s % 3])
        if s >= 2:
            eng.stream.wait_event(drained[i])
        kt.predict_rows(model, space, bufs[s % 3], out=sbufs[i], engine=eng)
        with eng.scope():
            scored[i].record(eng.stream)
        with torch.cuda.stream(d2h_stream):  # the D2H overlaps the clustering queued behind it
            d2h_stream.wait_event(scored[i])
            host_scores[i].copy_(sbufs[i], non_blocking=True)
            drained[i].record(d2h_stream)

    d2h = 0
    barrier()
    flush.fill_(-1.0)
    torch.cuda.synchronize()
    e2e_start.record(copy_stream)
    for s in range(min(2, args.steps)):
        upload(s)
    score(0)
    for s in range(args.steps):
        if s + 1 < args.steps:
            score(s + 1)
        if s + 2 < args.steps:
            upload(s + 2)
        batch = kt.adaptive_sample_rows(bufs[s % 3], visited_for[2000 + s], space, 2000 + s, engine=eng)
        d2h += batch.nbytes + N * 8
    with eng.scope():
        eng.stream.wait_stream(copy_stream)
        eng.stream.wait_stream(d2h_stream)
        e2e_end.record(eng.stream)
    barrier()
    t_e2e = e2e_start.elapsed_time(e2e_end) / 1e3

    # ---- instrumented pass: per-kernel CUDA-event durations (roofline)
    eng.set_timing(True)
    eng.kernel_stats(reset=True)
    kinfo = []
    for s in range(args.steps):
        flush.fill_(float(s))
        info = kt._lib.SampleInfo()
        step(dev_sets[s % n_sets], 1000 + s, visited_for[1000 + s], info)
        kinfo.append(info)
    stats = eng.kernel_stats(reset=True)
    eng.set_timing(False)

    times = torch.tensor([t_total, t_e2e], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    t_total, t_e2e = float(times[0]), float(times[1])
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    K = args.steps
    value = world * N * K / t_total
    e2e_value = world * N * K / t_e2e
    pk = peaks()
    # dominant kernel and its algorithmic bytes per launch
    dom = max(stats.items(), key=lambda kv: kv[1][1])
    dom_name, (dom_count, dom_ms) = dom
    if dom_name == "lloyd":
        alg_bytes = sum(i.lloyd_bytes for i in kinfo)
        note = ("SURVEY §8(d) K8: (n + 1) B per distinct point per Lloyd pass per active k (8 B row + 1 B assignment); "
                "the resident kernel keeps state in shared memory, so DRAM traffic is far below this")
    elif dom_name == "score_trees":
        alg_bytes = K * N * 16
        note = "8 B row read + 8 B float64 score written per candidate"
    else:
        alg_bytes = None
        note = "no byte model"
    achieved = (alg_bytes / dom_count) / (dom_ms / dom_count / 1e3) / 1e9 if alg_bytes else None
    # DRAM traffic per launch of the same kernel from the committed ncu --set full capture
    tr_doc = ROOT / "profiles" / TRAFFIC_ROUND / "traffic.json"
    traffic = None
    if tr_doc.exists():
        traffic = json.loads(tr_doc.read_text())["kernels"].get(dom_name, {}).get("dram_bytes_per_launch")
    kernel_table = {k: {"launches": c, "ms_total": round(ms, 4), "ms_per_step": round(ms / K, 4)}
                    for k, (c, ms) in sorted(stats.items(), key=lambda kv: -kv[1][1])}
    base = None
    if not args.no_cpu_baseline and world == 1:  # the CPU baseline is reported at N = 1 only
        base = cpu_baseline(doc, cards, args.cpu_sample, full=0 if args.no_cpu_full else N)
    chosen = sorted({i.chosen_k for i in infos})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": t_total / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD.format(n=N), "candidates_per_step": N, "parallelism": f"tasks x{world} (1 per GPU)",
                   "l2": "value: flushed between steps (512 MiB write, outside the timed events); e2e: one continuous "
                                "region, every step's rows a fresh H2D copy from pinned host memory (overlapped with "
                                "the previous step on a copy stream)",
                   "distinct_per_step": int(np.mean([i.n_distinct for i in infos])), "knee_k": chosen,
                   "mode_vote_steps": int(sum(i.used_mode for i in infos)),
                   "lloyd_passes_per_step": float(np.mean([i.lloyd_passes for i in infos]))},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": N * 8, "d2h_bytes_per_step": d2h // K},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": (achieved / pk["hbm_gbs"]) if achieved else None, "traffic": traffic,
                     "traffic_source": f"profiles/{TRAFFIC_ROUND}/traffic.json (ncu --set full, bytes per launch)",
                     "alg_bytes_per_launch": (alg_bytes / dom_count) if alg_bytes else None,
                     "peak_source": pk["source"], "bytes_model": note,
                     "kernel_share_of_step": dom_ms / sum(ms for _, ms in stats.values())},
        "kernels": kernel_table,
        "clocks": clk.summary(),
        "cpu_baseline": base,
        "parity": parity,
    }
    if not args.no_wall95 and world == 1:  # metric 2 is a single-task, single-GPU number
        line["wall_to_95"] = w95_ours(eng)
    if not args.no_extra_configs and world == 1:  # configs[1..4] beside the headline (after its timing)
        from tools import extra_configs

        try:
            line["other_configs"] = extra_configs.run_all(kt, torch, steps=2, local_rank=local_rank)
        except Exception as ex:  # informational: never lose the headline line over it
            line["other_configs"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_rl(args, rank: int, world: int, local_rank: int) -> None:
    import torch

    import paper_1905_12799_b200 as kt
    from tools import bench_rl

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    line = bench_rl.run(args, rank, world, local_rank, kt, torch, dist, {"barrier": barrier, "clock": ClockSampler})
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_c4(args, rank: int, world: int, local_rank: int) -> None:
    import torch

    import paper_1905_12799_b200 as kt
    from tools import bench_c4

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    line = bench_c4.run(args, rank, world, local_rank, kt, torch, dist, {"barrier": barrier, "clock": ClockSampler})
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--candidates", type=int, default=1 << 20)
    ap.add_argument("--cpu-sample", type=int, default=32768)
    ap.add_argument("--ref-sample", type=int, default=16384)
    ap.add_argument("--ref-procs", type=int, default=0, help="host processes for --impl reference (0: all cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-full", action="store_true", help="skip the one full-size (1M) CPU step (~2 min)")
    ap.add_argument("--no-wall95", action="store_true", help="skip the wall-time-to-95%%-best tune runs")
    ap.add_argument("--no-extra-configs", action="store_true",
                    help="skip the short runs of BASELINE configs[1..4] reported beside the headline")
    ap.add_argument("--rl-serial", action="store_true",
                    help="--workload rl: the 5 tasks in sequence on one engine (default: 5 engines, 5 host threads)")
    ap.add_argument("--workload", choices=("s2", "rl", "c4"), default="s2",
                    help="s2: the headline scored+clustered step; rl: 5 tasks x 4096 PPO agents per step; "
                         "c4: ResNet-18's 12 tasks x 1M candidates placed over the ranks (configs[3])")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload == "rl":
        run_rl(args, rank, world, local_rank)
    elif args.workload == "c4":
        run_c4(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
