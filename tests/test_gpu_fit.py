"""Device surrogate refit: kt_fit_trees_device grows every tree in one
single-CTA CUDA kernel — byte-identical model JSON to the REFERENCE's fit (golden cases from
tests/golden/make_fit.py, cost_model.py:367-398) and to the host engine on random,
tie-heavy, constant and duplicate-row training sets at every supported depth."""

import json
import sys
import time
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_fit import case_inputs  # noqa: E402

import paper_1905_12799_b200 as kt  # noqa: E402

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "fit.json").read_text())


class _TS:
    def __init__(self, X, y):
        self.features, self.targets = X, y


@pytest.mark.parametrize("mode", ["auto", "global"])
@pytest.mark.parametrize("case", GOLD, ids=lambda c: f"m{c['m']}_n{c['n']}_{c['targets']}")
def test_device_fit_byte_identical_to_reference(case, mode, monkeypatch):
    if mode == "global":
        monkeypatch.setenv("KT_FIT_GLOBAL", "1")
    X, y = case_inputs(case["seed"], case["m"], case["n"], case["levels"], case["targets"])
    params = kt.BoostParams(case["rounds"], case["depth"], case["lr"])
    before = kt.engine().launches
    model = kt.fit(_TS(X, y), params, device=True)
    assert kt.engine().launches > before  # the CUDA kernel ran
    assert model.to_json() == case["model"]
    perm = np.random.default_rng(1).permutation(len(y))
    assert kt.fit(_TS(X[perm], y[perm]), params, device=True).to_json() == case["model"]


@pytest.mark.parametrize("seed,m,n,levels,depth", [
    (11, 1, 1, 2, 1), (12, 3, 2, 2, 7), (13, 17, 8, 2, 3), (14, 257, 5, 9, 7), (15, 640, 8, 64, 5),
    (16, 4096, 8, 30, 4), (17, 1000, 2, 3, 6), (18, 5000, 8, 200, 4)])
@pytest.mark.parametrize("kind", ["rand", "ties", "const", "dups"])
@pytest.mark.parametrize("mode", ["auto", "global"])
def test_device_fit_matches_host(seed, m, n, levels, depth, kind, mode, monkeypatch):
    """auto: the shared-memory kernel for m up to ~1300 rows (else the global one);
    global: KT_FIT_GLOBAL forces the global-memory kernel."""
    if mode == "global":
        monkeypatch.setenv("KT_FIT_GLOBAL", "1")
    if kind == "dups":
        Xb, yb = case_inputs(seed, (m + 3) // 4, n, levels, "rand")
        X, y = np.tile(Xb, (4, 1))[:m], np.tile(yb, 4)[:m]
    else:
        X, y = case_inputs(seed, m, n, levels, kind)
    params = kt.BoostParams(20, depth, 0.3)
    dev = kt.fit(_TS(X, y), params, device=True)
    host = kt.fit(_TS(X, y), params, device=False)
    assert dev.to_json() == host.to_json()


def test_device_fit_errors_and_auto_path():
    with pytest.raises(ValueError, match="empty"):
        kt.fit(_TS(np.zeros((0, 2)), np.zeros(0)), device=True)
    with pytest.raises(NotImplementedError, match="depth"):
        kt.fit(_TS(np.zeros((3, 2)), np.zeros(3)), kt.BoostParams(depth=8), device=True)
    X, y = case_inputs(3, 300, 8, 10, "rand")
    before = kt.engine().launches
    kt.fit(_TS(X, y))  # default: the native host engine (faster at tuning sizes)
    assert kt.engine().launches == before


def test_device_fit_timing_report():
    """Not a gate: prints device vs host refit time at the tuning budget (1000 records)."""
    X, y = case_inputs(7, 1000, 8, 30, "rand")
    params = kt.BoostParams()
    for dev in (True, False):
        kt.fit(_TS(X, y), params, device=dev)
        t = time.perf_counter()
        for _ in range(5):
            kt.fit(_TS(X, y), params, device=dev)
        print(f"fit m=1000 n=8 {'device' if dev else 'host'}: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms")
