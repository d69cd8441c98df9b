"""Parity of the CUDA path on spaces whose knobs exceed 255 settings (bit-field rows).

AlexNet's conv3/conv4 tasks (configs[1]) have tile_f cardinality 480, and the
synthetic ``wide8`` space packs 8 knobs into 41 bits; rows use the bit-field
layout of ``space.row_layout`` / ``row_fmt``.  Same bars as the byte layout:
bit-exact trees, k-means, mode, SA and trajectories; runtimes within 1e-12;
the PPO update at the TF32 tier.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_12799_b200 as kt  # noqa: E402
from golden_io import meta, npz  # noqa: E402
from oracle import agent as oagent  # noqa: E402
from oracle import sa as osa  # noqa: E402
from oracle import sampler as osamp  # noqa: E402
from oracle import trees as otrees  # noqa: E402
from paper_1905_12799_b200 import space as sp  # noqa: E402
from paper_1905_12799_b200.agent import _flat  # noqa: E402

W = meta("wide")
G = npz("wide")


def space_of(values, name="wide"):
    return kt.DesignSpace(name, tuple(kt.KnobDef(f"k{i}", tuple(v)) for i, v in enumerate(values)))


def dev_rows(idx, cards):
    return torch.from_numpy(sp.pack(np.asarray(idx), cards).view(np.int64)).cuda()


def model_of(name):
    m = W["models"][name]
    return space_of(m["values"]), kt.CostModel.from_dict(m["model"]), m


@pytest.fixture(scope="module", autouse=True)
def _engine_loaded():
    kt.engine(0)


@pytest.mark.parametrize("name", ["alexnet2", "alexnet3", "wide8"])
def test_wide_predict_bit_exact(name):
    space, model, _ = model_of(name)
    idx = G[f"predict/{name}/idx"]
    got = kt.predict_rows(model, space, dev_rows(idx, space.cardinalities)).cpu().numpy()
    assert np.array_equal(got, G[f"predict/{name}/scores"])
    configs = [kt.Configuration(tuple(r)) for r in idx[:50].tolist()]
    assert np.array_equal(kt.predict(model, space, configs), G[f"predict/{name}/scores"][:50])


def test_wide_predict_random_vs_oracle():
    space, model, m = model_of("alexnet3")
    idx = np.random.default_rng(3).integers(0, np.array(space.cardinalities), size=(100_003, 8))
    got = kt.predict_rows(model, space, dev_rows(idx, space.cardinalities)).cpu().numpy()
    want = otrees.predict_features(m["model"], otrees.featurize_rows(m["values"], idx))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name", ["alexnet3", "wide8"])
def test_wide_landscape(name):
    space, _, m = model_of(name)
    land = kt.landscape.landscape_from_dict(m["landscape"], space)
    idx = G[f"landscape/{name}/idx"]
    got = kt.runtimes_rows(land, dev_rows(idx, space.cardinalities)).cpu().numpy()
    want = G[f"landscape/{name}/runtime"]
    assert np.array_equal(got, want)  # bit-exact (glibc's exp restated on the device)


@pytest.mark.parametrize("name", sorted(W["adaptive"]))
def test_wide_adaptive_sample_and_mode(name):
    md = W["adaptive"][name]
    cards = md["cards"]
    space = space_of([list(range(c)) for c in cards])
    idx = G[f"adaptive/{name}/idx"]
    traj = kt.Trajectory(dev_rows(idx, cards), torch.zeros(len(idx), dtype=torch.float64, device="cuda"),
                         n_knobs=len(cards), cards=cards)
    visited = kt.VisitedSet([kt.Configuration(tuple(r)) for r in G[f"adaptive/{name}/visited"].tolist()])
    batch = kt.adaptive_sample(traj, visited, space, md["seed"])
    assert [c.indices for c in batch] == [tuple(r) for r in G[f"adaptive/{name}/batch"].tolist()]
    assert kt.mode_config(traj, space).indices == tuple(G[f"adaptive/{name}/mode"].tolist())


@pytest.mark.parametrize("pack", ["pack3", "pack5"])
@pytest.mark.parametrize("seed", [0, 1])
def test_wide_adaptive_sample_vs_oracle(seed, pack, monkeypatch):
    """Bit-field rows under both resident delta encodings (3-word packed deltas when the block's
    points allow, the 5-word fallback forced by KT_LLOYD_PACK5)."""
    if pack == "pack5":
        monkeypatch.setenv("KT_LLOYD_PACK5", "1")
    space, _, _ = model_of("alexnet3")
    cards = space.cardinalities
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, np.array(cards), size=(30_000, 8))
    idx = np.vstack([idx, idx[:3000]])
    visited = {tuple(r) for r in idx[rng.integers(0, len(idx), size=40)].tolist()}
    got = kt.adaptive_sample_rows(dev_rows(idx, cards), sp.pack(np.array(sorted(visited)), cards), space, seed=seed + 5)
    want = osamp.adaptive_sample(idx, visited, cards, seed + 5)
    assert [tuple(r) for r in sp.unpack(got, 8, cards).tolist()] == want


def test_wide_kmeans_points_vs_oracle():
    """kmeans/knee on float lattice points with coordinates > 255 (layout from the point extents)."""
    rng = np.random.default_rng(11)
    pts = np.unique(rng.integers(0, [480, 9, 300, 4], size=(2500, 4)), axis=0)
    pts = pts[rng.permutation(len(pts))].astype(np.float64)
    res = kt.kmeans(pts, 9, seed=4)
    want = osamp.kmeans(pts, 9, 4)
    assert np.array_equal(res.centroids, want["centroids"])
    assert np.array_equal(res.assignment, want["assignment"])
    assert res.loss == want["loss"]
    _, scanned = kt.knee_scan(pts, seed=6)
    _, want_scanned = osamp.knee_scan(pts, 6)
    assert scanned == want_scanned


@pytest.mark.parametrize("name", sorted(W["sa"]))
def test_wide_sa(name):
    md = W["sa"][name]
    space, model, _ = model_of(md["model"])
    params = kt.SAParams(chains=md["chains"], steps_per_round=md["steps"],
                         initial_temperature=md["initial_temperature"], cooling=md["cooling"])
    starts = [kt.Configuration(tuple(r)) for r in G[f"sa/{name}/starts"].tolist()]
    tr = kt.run_sa_round(params, model, space, starts, md["seed"])
    assert np.array_equal(tr.index_matrix(), G[f"sa/{name}/idx"])
    assert np.array_equal(tr.scores(), G[f"sa/{name}/scores"])
    assert tr.step_indices == tuple(G[f"sa/{name}/steps"].tolist())


def test_wide_sa_large_vs_oracle():
    space, model, m = model_of("alexnet3")
    idx = np.random.default_rng(8).integers(0, np.array(space.cardinalities), size=(700, 8))
    tr = kt.run_sa_round(kt.SAParams(chains=1024, steps_per_round=40), model, space,
                         [kt.Configuration(tuple(r)) for r in idx.tolist()], seed=99)
    o_idx, o_sc, o_st = osa.run_sa_round(m["model"], m["values"], idx, 99, chains=1024, steps=40)
    assert np.array_equal(tr.index_matrix(), o_idx)
    assert np.array_equal(tr.scores(), o_sc)
    assert np.array_equal(np.array(tr.step_indices), o_st)


def test_wide_search_round():
    md = W["rl"]["alexnet3"]
    space, model, _ = model_of("alexnet3")
    hyper = kt.AgentHyperparams.from_dict(md["hyper"])
    agent = kt.init_agent(space, hyper, seed=md["seed"])
    assert np.array_equal(_flat(agent.params), G["rl/alexnet3/params0"])
    before = _flat(agent.params)
    starts = [kt.Configuration(tuple(r)) for r in G["rl/alexnet3/starts"].tolist()]
    tr = kt.run_search_round(agent, model, space, starts)
    assert np.array_equal(tr.index_matrix(), G["rl/alexnet3/idx"])
    assert np.array_equal(tr.scores(), G["rl/alexnet3/scores"])
    assert tr.step_indices == tuple(G["rl/alexnet3/steps"].tolist())
    # PPO update at the TF32 tier: each parameter moved like the reference's (within 5% of lr)
    got, want = _flat(agent.params) - before, G["rl/alexnet3/params"] - before
    assert np.max(np.abs(got - want)) < 5e-2 * hyper.adam_step_size
    assert oagent is not None
