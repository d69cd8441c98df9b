"""Device vs host surrogate refit at the tuning budget: kernel time (engine stats) and wall (GPU)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import paper_1905_12799_b200 as kt  # noqa: E402
from make_fit import case_inputs  # noqa: E402


class _TS:
    def __init__(self, X, y):
        self.features, self.targets = X, y


m = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
X, y = case_inputs(7, m, 8, 30, "rand")
eng = kt.engine(0)
for rep in range(3):
    eng.set_timing(True)
    t = time.perf_counter()
    kt.fit(_TS(X, y), kt.BoostParams(), device=True)
    dt = time.perf_counter() - t
    st = eng.kernel_stats(reset=True)
    t = time.perf_counter()
    kt.fit(_TS(X, y), kt.BoostParams(), device=False)
    dh = time.perf_counter() - t
    print(f"m={m} rep {rep}: device wall {dt*1e3:.2f} ms (kernels {({k: round(v[1], 3) for k, v in st.items()})}), "
          f"host {dh*1e3:.2f} ms")
