"""Large-size golden cases for the k-means / adaptive-sample path (resident Lloyd kernel, many tiles).

The oracle (oracle/sampler.py, pinned bit-exact to the reference by tests/test_oracle.py) is run
here on seeded uniform candidates of the S2 ResNet-18 space; only the seeds and the outputs are
committed (tests/golden/large.json), the inputs are regenerated from the seeds by the tests.

    python tests/golden/make_large.py
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import sampler as osamp  # noqa: E402

CASES = [(262144, 5, 13), (131072, 6, 21)]  # (candidates, candidate seed, adaptive_sample seed)


def candidates(n: int, seed: int, cards: np.ndarray) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, cards, size=(n, cards.size))


def main() -> None:
    doc = json.loads((ROOT / "data" / "models" / "s2_resnet18.json").read_text())
    cards = np.array([len(v) for v in doc["values"]])
    out = {}
    for n, cseed, seed in CASES:
        idx = candidates(n, cseed, cards)
        batch, info = osamp.adaptive_sample(idx, set(), cards.tolist(), seed, return_info=True)
        res = info["result"]
        out[f"{n}_{cseed}_{seed}"] = {
            "n": n, "cand_seed": cseed, "seed": seed, "m": info["m"],
            "batch": [list(b) for b in batch],
            "curve": [[k, float(l).hex()] for k, l in info["curve"]],
            "assignment_sha256": hashlib.sha256(np.asarray(res["assignment"], dtype=np.int64).tobytes()).hexdigest(),
            "centroids": [[float(x).hex() for x in c] for c in res["centroids"]],
        }
        print(n, len(batch), info["curve"])
    (HERE / "large.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
