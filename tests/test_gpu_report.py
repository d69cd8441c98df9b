"""Trajectory analysis on the device vs the reference's report.py
(tests/golden/report.json): per_step_best and convergence steps exact, PCA projections
to float64 rounding (the reference's covariance / projections go through BLAS)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_report import case_inputs  # noqa: E402

import paper_1905_12799_b200 as kt  # noqa: E402
from paper_1905_12799_b200 import report  # noqa: E402
from paper_1905_12799_b200 import space as sp  # noqa: E402

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "report.json").read_text())


@pytest.mark.parametrize("case", GOLD, ids=lambda c: f"N{c['N']}_n{c['n']}")
def test_report_vs_reference(case):
    idx, scores, steps = case_inputs(case["seed"], case["N"], case["S"], case["n"], case["card"])
    cards = np.full(case["n"], case["card"], dtype=np.int64)
    tr = kt.Trajectory(torch.from_numpy(sp.pack(idx, cards).view(np.int64)).cuda(),
                       torch.from_numpy(scores).cuda(), torch.from_numpy(steps.astype(np.int32)).cuda(),
                       n_knobs=case["n"], cards=cards)
    assert [float(x).hex() for x in report.per_step_best(tr)] == case["per_step_best"]
    assert report.convergence_steps_for_round(tr) == case["convergence"]
    got = np.array(report.pca_project(idx, cards=cards))
    want = np.array(case["pca"])
    scale = np.max(np.abs(want))
    assert np.max(np.abs(got - want)) <= 1e-9 * scale


def test_report_errors():
    with pytest.raises(ValueError, match="at least 2 configurations"):
        report.pca_project(np.zeros((1, 3), dtype=np.int64))
    with pytest.raises(ValueError, match="at least 2 knobs"):
        report.pca_project(np.zeros((4, 1), dtype=np.int64))
    with pytest.raises(kt.errors.DegenerateVarianceError):
        report.pca_project(np.ones((5, 3), dtype=np.int64))
    tr = kt.Trajectory(torch.zeros(3, dtype=torch.int64).cuda(), torch.zeros(3, dtype=torch.float64).cuda(), None,
                       n_knobs=2)
    with pytest.raises(ValueError, match="step indices"):
        report.per_step_best(tr)


def test_per_step_best_accepts_reference_trajectory():
    """install() rebinds knobtuner.report.per_step_best: the reference's own Trajectory (a frozen
    dataclass with ``entries`` and a ``step_indices`` tuple, agent.py:100-127) must work too."""
    from dataclasses import dataclass

    @dataclass(frozen=True)
    class RefConfiguration:
        indices: tuple

    @dataclass(frozen=True)
    class RefTrajectory:
        entries: tuple
        step_indices: tuple | None = None

        def configs(self):
            return [c for c, _ in self.entries]

        def scores(self):
            return np.array([s for _, s in self.entries], dtype=np.float64)

    case = GOLD[0]
    idx, scores, steps = case_inputs(case["seed"], case["N"], case["S"], case["n"], case["card"])
    tr = RefTrajectory(tuple((RefConfiguration(tuple(r)), float(s)) for r, s in zip(idx.tolist(), scores.tolist())),
                       tuple(int(s) for s in steps.tolist()))
    assert [float(x).hex() for x in report.per_step_best(tr)] == case["per_step_best"]
    assert report.convergence_steps_for_round(tr) == case["convergence"]
    with pytest.raises(ValueError, match="step indices"):
        report.per_step_best(RefTrajectory(tr.entries, None))
