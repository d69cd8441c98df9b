"""Golden brute-force optima produced by the REFERENCE's own enumeration (cli.py:77-90
``_enumerated_oracle``: enumerate_space + synthetic_runtime, strict ``<`` scan) and sampled
runtimes (backends.py:164-174), for the fused device argmin ``kt_landscape_best`` and K3.

    python tests/golden/make_best.py      # writes tests/golden/best.json (~1 min)

Cases: the fixture space bench_grid4d x its 5 landscapes; conv_gpu_table1 (49,000 configs) with
gen_landscape(seed=1); and a bit-field ("wide") space whose first knob has 480 settings (AlexNet
conv3/4 ``tile_f``) within the reference's 10^6 enumeration cap, with gen_landscape(seed=3).
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from knobtuner import cli  # noqa: E402
from knobtuner.backends import gen_landscape, landscape_to_dict, synthetic_runtime  # noqa: E402
from knobtuner.space import Configuration, parse_space  # noqa: E402

HERE = Path(__file__).resolve().parent
PKG = Path("/root/reference/pkg")
WIDE = {"name": "wide_alexnet_like", "knobs": [
    {"name": "tile_f", "values": list(range(480))}, {"name": "tile_y", "values": list(range(9))},
    {"name": "tile_x", "values": list(range(5))}, {"name": "tile_rc", "values": list(range(4))},
    {"name": "unroll_explicit", "values": [0, 1]}, {"name": "auto_unroll_max_step", "values": [0, 512, 1500]}]}


def case(space_doc: dict, land_doc: dict, name: str, n_sample: int = 2000) -> dict:
    space = parse_space(json.dumps(space_doc))
    with tempfile.TemporaryDirectory() as d:
        sp_path, l_path = Path(d) / "space.json", Path(d) / "land.json"
        sp_path.write_text(json.dumps(space_doc))
        l_path.write_text(json.dumps(land_doc))
        best_idx, best_rt = cli._enumerated_oracle(str(sp_path), f"synthetic:{l_path}")
        from knobtuner.backends import load_landscape

        land = load_landscape(l_path, space)
    rng = np.random.default_rng(len(name))
    idx = rng.integers(0, np.array(space.cardinalities), size=(n_sample, len(space.cardinalities)))
    rts = [synthetic_runtime(land, Configuration(tuple(int(v) for v in r))) for r in idx.tolist()]
    print(name, best_idx, best_rt)
    return {"name": name, "space": space_doc, "landscape": land_doc, "best_indices": best_idx,
            "best_runtime": float(best_rt).hex(), "sample_idx": idx.tolist(), "sample_runtime": [x.hex() for x in rts]}


def main() -> None:
    out = []
    grid = json.loads((PKG / "spaces" / "bench_grid4d.json").read_text())
    for s in range(5):
        out.append(case(grid, json.loads((PKG / "landscapes" / f"bench_grid4d_s{s}.json").read_text()), f"grid4d_s{s}"))
    table1 = json.loads((PKG / "spaces" / "conv_gpu_table1.json").read_text())
    out.append(case(table1, landscape_to_dict(gen_landscape(parse_space(json.dumps(table1)), 1)), "table1_seed1"))
    out.append(case(WIDE, landscape_to_dict(gen_landscape(parse_space(json.dumps(WIDE)), 3)), "wide_seed3"))
    (HERE / "best.json").write_text(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
