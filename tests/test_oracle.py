"""Pin the CPU oracle (oracle/) to the reference: golden vectors + the reference's known answers.

CPU-only; these are the checks that make the oracle trustworthy before it is
used to judge the CUDA path.
"""

import math

import numpy as np
import pytest

from golden_io import cases, meta, npz
from oracle import agent as oagent
from oracle import landscape as oland
from oracle import sa as osa
from oracle import sampler as osamp
from oracle import trees as otrees


def models():
    import json
    from golden_io import GOLDEN

    return json.loads((GOLDEN / "models.json").read_text())


# ---------------------------------------------------------------- trees
@pytest.mark.parametrize("name", sorted(models()))
def test_predict_matches_reference(name):
    m = models()[name]
    g = npz("predict")
    X = otrees.featurize_rows(m["values"], g[f"{name}/idx"])
    got = otrees.predict_features(m["model"], X)
    assert np.array_equal(got, g[f"{name}/scores"])  # bit-exact


def test_featurize_known_answers():
    # reference test_cost_model.py:52-63 (values 1 and 3 -> 1, 2; 0 -> 0; 7 -> 3)
    assert otrees.featurize_rows([[1], [3]], [[0, 0]]).tolist() == [[1.0, 2.0]]
    assert otrees.featurize_rows([[0, 1]], [[0]]).tolist() == [[0.0]]
    assert otrees.featurize_rows([[7]], [[0]]).tolist() == [[3.0]]
    with pytest.raises(ValueError):
        otrees.featurize_rows([[-2, 1]], [[0]])


# ---------------------------------------------------------------- landscape
@pytest.mark.parametrize("name", sorted(meta("landscapes")))
def test_landscape_matches_reference(name):
    d = meta("landscapes")[name]
    g = npz("landscape")
    got = oland.synthetic_runtimes(d["landscape"], g[f"{name}/idx"])
    assert np.array_equal(got, g[f"{name}/runtime"])


def test_landscape_known_answers():
    # reference test_backends.py:112-120
    at_center = {"seed": 0, "centers": [[4]], "depths": [0.9], "radii": [2.0], "base_runtime": 2.0, "noise_rel": 0.0}
    assert oland.synthetic_runtimes(at_center, [[4]])[0] == pytest.approx(0.2, rel=1e-12)
    far = {"seed": 0, "centers": [[0]], "depths": [0.9], "radii": [0.5], "base_runtime": 1.0, "noise_rel": 0.0}
    assert oland.synthetic_runtimes(far, [[9]])[0] == pytest.approx(1.0, rel=1e-12)


# ---------------------------------------------------------------- sampler
@pytest.mark.parametrize("name", cases("kmeans", "points"))
def test_kmeans_matches_reference(name):
    g = npz("kmeans")
    k, seed = (int(x) for x in g[f"{name}/meta"])
    res = osamp.kmeans(g[f"{name}/points"], k, seed)
    assert np.array_equal(res["centroids"], g[f"{name}/centroids"])
    assert np.array_equal(res["assignment"], g[f"{name}/assignment"])
    assert np.array_equal(np.array(res["history"]), g[f"{name}/history"])


def test_kmeans_known_answers():
    # reference test_sampler.py:48-62, test_acceptance.py:184-185
    res = osamp.kmeans(np.array([0.0, 1.0, 10.0, 11.0]), 2, 0)
    assert res["loss"] == 1.0
    assert sorted(res["centroids"][:, 0].tolist()) == [0.5, 10.5]
    with pytest.raises(ValueError, match="out of range"):
        osamp.kmeans(np.array([[0.0], [1.0], [1.0]]), 3, 0)


@pytest.mark.parametrize("name", cases("knee", "points"))
def test_knee_matches_reference(name):
    g = npz("knee")
    res, curve = osamp.knee_scan(g[f"{name}/points"], int(g[f"{name}/seed"][0]))
    assert np.array_equal(np.array(curve, dtype=np.float64), g[f"{name}/scanned"])
    assert np.array_equal(res["centroids"], g[f"{name}/centroids"])
    assert np.array_equal(res["assignment"], g[f"{name}/assignment"])


@pytest.mark.parametrize("name", sorted(meta("adaptive")))
def test_adaptive_sample_matches_reference(name):
    g = npz("adaptive")
    md = meta("adaptive")[name]
    visited = {tuple(r) for r in g[f"{name}/visited"].tolist()}
    batch = osamp.adaptive_sample(g[f"{name}/idx"], visited, md["cards"], md["seed"])
    assert batch == [tuple(r) for r in g[f"{name}/batch"].tolist()]
    assert osamp.mode_vote(g[f"{name}/idx"], md["cards"]) == tuple(g[f"{name}/mode"].tolist())


def test_mode_and_round_known_answers():
    # reference test_sampler.py:110-136
    assert osamp.mode_vote([[1, 2], [1, 3], [2, 3]], [4, 4]) == (1, 3)
    assert osamp.mode_vote([[1, 0], [2, 0], [1, 1], [2, 1]], [4, 4]) == (1, 0)
    assert osamp.round_centroid(np.array([0.4, 2.6]), [4, 4]) == (0, 3)
    assert osamp.round_centroid(np.array([3.7]), [3]) == (2,)
    assert osamp.round_centroid(np.array([1.5]), [4]) == (2,)


# ---------------------------------------------------------------- SA
@pytest.mark.parametrize("name", sorted(meta("sa")))
def test_sa_matches_reference(name):
    g = npz("sa")
    md = meta("sa")[name]
    m = models()[md["model"]]
    idx, scores, steps = osa.run_sa_round(m["model"], m["values"], g[f"{name}/starts"], md["seed"],
                                          chains=md["chains"], steps=md["steps"],
                                          initial_temperature=md["initial_temperature"], cooling=md["cooling"])
    assert np.array_equal(idx, g[f"{name}/idx"])
    assert np.array_equal(scores, g[f"{name}/scores"])
    assert np.array_equal(steps, g[f"{name}/steps"])


# ---------------------------------------------------------------- RL
def _flat(p):
    return np.concatenate([p[k].ravel() for k in oagent.KEYS])


@pytest.mark.parametrize("name", sorted(meta("rl")))
def test_search_round_matches_reference(name):
    g = npz("rl")
    md = meta("rl")[name]
    m = models()[md["model"]]
    agent = oagent.new_agent(len(m["values"]), md["hyper"], md["seed"])
    assert np.array_equal(_flat(agent["params"]), g[f"{name}/params0"])
    for rd in range(md["rounds"]):
        idx, scores, steps = oagent.search_round(agent, m["model"], m["values"], g[f"{name}/r{rd}/starts"], md["hyper"])
        assert np.array_equal(idx, g[f"{name}/r{rd}/idx"])
        assert np.array_equal(scores, g[f"{name}/r{rd}/scores"])
        assert np.array_equal(steps, g[f"{name}/r{rd}/steps"])
        assert np.array_equal(_flat(agent["params"]), g[f"{name}/r{rd}/params"])
        assert np.array_equal(_flat(agent["m"]), g[f"{name}/r{rd}/adam_m"])
        assert np.array_equal(_flat(agent["v"]), g[f"{name}/r{rd}/adam_v"])


def test_gae_known_answers():
    # reference test_agent.py:45-61
    assert oagent.gae(np.array([1.0, 1.0]), np.array([0.0, 0.0]), 0.0, 0.9, 0.99) == pytest.approx([1.891, 1.0], abs=1e-9)
    rng = np.random.default_rng(2)
    r, v = rng.normal(size=6), rng.normal(size=6)
    nv = np.append(v[1:], 0.7)
    d = r + 0.9 * nv - v
    want = [sum((0.9 * 0.99) ** (k - t) * d[k] for k in range(t, 6)) for t in range(6)]
    assert oagent.gae(r, v, 0.7, 0.9, 0.99) == pytest.approx(want, abs=1e-12)


def test_ppo_clip_known_answers():
    # reference test_agent.py:146-169: clipped objective -1.3 / -0.5 / 0.7
    p = oagent.init_params(2, 4, 4, 0)
    rng = np.random.default_rng(0)
    p = {"w1": rng.uniform(-1, 1, (4, 2)), "b1": np.zeros(4), "w2p": rng.uniform(-1, 1, (4, 4)), "b2p": np.zeros(4),
         "w3p": rng.uniform(-1, 1, (6, 4)), "b3p": np.zeros(6), "w2v": rng.uniform(-1, 1, (4, 4)), "b2v": np.zeros(4),
         "w3v": rng.uniform(-1, 1, (1, 4)), "b3v": np.zeros(1)}
    X = np.array([[0.2, 0.8]])
    a = np.array([[2, 0]])
    logits, _, _ = oagent.forward(p, X)
    base = oagent.joint_log_prob(logits, a)
    args = dict(clip=0.3, value_coef=0.0, entropy_coef=0.0)
    rep, _ = oagent.loss_and_grads(p, X, a, base - math.log(2.0), np.array([1.0]), np.array([0.0]), **args)
    assert rep[0] == pytest.approx(-1.3)
    rep, _ = oagent.loss_and_grads(p, X, a, base + math.log(2.0), np.array([1.0]), np.array([0.0]), **args)
    assert rep[0] == pytest.approx(-0.5)
    rep, _ = oagent.loss_and_grads(p, X, a, base + math.log(2.0), np.array([-1.0]), np.array([0.0]), **args)
    assert rep[0] == pytest.approx(0.7)


def test_ppo_gradient_finite_differences():
    # reference test_agent.py:171-202: central differences, h=1e-5, rel err < 1e-4
    rng = np.random.default_rng(42)
    p = oagent.init_params(2, 4, 4, 42)
    B = 3
    X = rng.random((B, 2))
    a = rng.integers(0, 3, size=(B, 2))
    logits, _, _ = oagent.forward(p, X)
    old = oagent.joint_log_prob(logits, a) + rng.normal(0.0, 0.3, size=B)
    adv, ret = rng.normal(size=B), rng.normal(size=B)
    kw = dict(clip=0.3, value_coef=1.0, entropy_coef=0.1)
    _, grads = oagent.loss_and_grads(p, X, a, old, adv, ret, **kw)
    worst = 0.0
    for key in oagent.KEYS:
        for i in range(p[key].size):
            up = {k: v.copy() for k, v in p.items()}
            dn = {k: v.copy() for k, v in p.items()}
            up[key].flat[i] += 1e-5
            dn[key].flat[i] -= 1e-5
            fd = (oagent.loss_and_grads(up, X, a, old, adv, ret, **kw)[0][3]
                  - oagent.loss_and_grads(dn, X, a, old, adv, ret, **kw)[0][3]) / 2e-5
            an = grads[key].flat[i]
            worst = max(worst, abs(fd - an) / max(1e-6, abs(fd), abs(an)))
    assert worst < 1e-4


# ------------------------------------------------ wide spaces (knobs > 255 settings)
def _wide(kind):
    return sorted(meta("wide")[kind])


@pytest.mark.parametrize("name", ["alexnet2", "alexnet3", "wide8"])
def test_wide_predict_matches_reference(name):
    m = meta("wide")["models"][name]
    g = npz("wide")
    X = otrees.featurize_rows(m["values"], g[f"predict/{name}/idx"])
    assert np.array_equal(otrees.predict_features(m["model"], X), g[f"predict/{name}/scores"])


@pytest.mark.parametrize("name", ["alexnet3", "wide8"])
def test_wide_landscape_matches_reference(name):
    m = meta("wide")["models"][name]
    g = npz("wide")
    got = oland.synthetic_runtimes(m["landscape"], g[f"landscape/{name}/idx"])
    assert np.array_equal(got, g[f"landscape/{name}/runtime"])


@pytest.mark.parametrize("name", _wide("adaptive"))
def test_wide_adaptive_sample_matches_reference(name):
    g = npz("wide")
    md = meta("wide")["adaptive"][name]
    visited = {tuple(r) for r in g[f"adaptive/{name}/visited"].tolist()}
    batch = osamp.adaptive_sample(g[f"adaptive/{name}/idx"], visited, md["cards"], md["seed"])
    assert batch == [tuple(r) for r in g[f"adaptive/{name}/batch"].tolist()]
    assert osamp.mode_vote(g[f"adaptive/{name}/idx"], md["cards"]) == tuple(g[f"adaptive/{name}/mode"].tolist())


@pytest.mark.parametrize("name", _wide("sa"))
def test_wide_sa_matches_reference(name):
    g = npz("wide")
    md = meta("wide")["sa"][name]
    m = meta("wide")["models"][md["model"]]
    idx, scores, steps = osa.run_sa_round(m["model"], m["values"], g[f"sa/{name}/starts"], md["seed"],
                                          chains=md["chains"], steps=md["steps"],
                                          initial_temperature=md["initial_temperature"], cooling=md["cooling"])
    assert np.array_equal(idx, g[f"sa/{name}/idx"])
    assert np.array_equal(scores, g[f"sa/{name}/scores"])
    assert np.array_equal(steps, g[f"sa/{name}/steps"])


def test_wide_search_round_matches_reference():
    g = npz("wide")
    md = meta("wide")["rl"]["alexnet3"]
    m = meta("wide")["models"]["alexnet3"]
    agent = oagent.new_agent(len(m["values"]), md["hyper"], md["seed"])
    assert np.array_equal(_flat(agent["params"]), g["rl/alexnet3/params0"])
    idx, scores, steps = oagent.search_round(agent, m["model"], m["values"], g["rl/alexnet3/starts"], md["hyper"])
    assert np.array_equal(idx, g["rl/alexnet3/idx"])
    assert np.array_equal(scores, g["rl/alexnet3/scores"])
    assert np.array_equal(steps, g["rl/alexnet3/steps"])
    assert np.array_equal(_flat(agent["params"]), g["rl/alexnet3/params"])
