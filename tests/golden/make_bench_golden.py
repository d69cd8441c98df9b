"""Bit-exact goldens for the BENCHMARKED configurations, produced by the pinned oracle
(oracle/sampler.py, checked against the reference itself by tests/test_oracle.py).

    python tests/golden/make_bench_golden.py [s2] [c5]    # ~2 min (s2) / ~10 min (c5)

* ``s2``: bench.py's headline step on rank 0's first candidate set — 1,048,576 uniform S2
  candidates (seed 0), adaptive_sample seed 1000 — with and without the visited set the bench
  uses (two of the step's own rounded centroids, as if measured in an earlier round, plus the
  first 62 candidates), which sends batch assembly through the mode vote (K9).
* ``c5``: configs[4]'s large end, 4,194,304 uniform S2 candidates (seed 4), seed 77: about 4M
  distinct points, beyond the resident Lloyd kernel (streaming kernel).

Inputs are regenerated from the seeds; only seeds and outputs are committed (bench_golden.json).
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import sampler as osamp  # noqa: E402

CASES = {"s2": (1 << 20, 0, 1000), "c5": (1 << 22, 4, 77)}  # (candidates, candidate seed, sample seed)


def candidates(n: int, seed: int, cards: np.ndarray) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, cards, size=(n, cards.size))  # == bench.candidates


def bench_visited(batch: list, idx: np.ndarray) -> list:
    """bench.py's visited set for a step: batch[:2] of the same step without visited + idx[:62]."""
    seen, out = set(), []
    for t in list(batch[:2]) + [tuple(r) for r in idx[:62].tolist()]:
        if t not in seen:
            seen.add(t)
            out.append(t)
    return out


def run(name: str, cards: np.ndarray) -> dict:
    n, cseed, seed = CASES[name]
    idx = candidates(n, cseed, cards)
    t0 = time.perf_counter()
    batch, info = osamp.adaptive_sample(idx, set(), cards.tolist(), seed, return_info=True)
    res = info["result"]
    visited = bench_visited(batch, idx)
    vbatch, mode = osamp.assemble_batch(res["centroids"], idx, set(visited), cards.tolist())
    print(name, f"{time.perf_counter() - t0:.1f} s", info["m"], info["curve"], len(batch), mode)
    return {
        "n": n, "cand_seed": cseed, "seed": seed, "m": info["m"],
        "batch": [list(b) for b in batch],
        "curve": [[k, float(v).hex()] for k, v in info["curve"]],
        "assignment_sha256": hashlib.sha256(np.asarray(res["assignment"], dtype=np.int64).tobytes()).hexdigest(),
        "centroids": [[float(x).hex() for x in c] for c in res["centroids"]],
        "visited": [list(t) for t in visited], "batch_visited": [list(b) for b in vbatch],
        "mode": None if mode is None else list(mode),
    }


def main() -> None:
    doc = json.loads((ROOT / "data" / "models" / "s2_resnet18.json").read_text())
    cards = np.array([len(v) for v in doc["values"]])
    path = HERE / "bench_golden.json"
    out = json.loads(path.read_text()) if path.exists() else {}
    for name in (sys.argv[1:] or list(CASES)):
        out[name] = run(name, cards)
        path.write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
