"""Parity of the B200 PPO search round (K1 rollout, K4 GAE, K5 PPO) with the reference.

* Rollout decisions are exact: for identical parameters and uniforms the
  trajectory (configs, scores, step indices) must be bit-identical (float64
  forward pass; measure-zero caveat for uniforms within ~1e-15 of a cdf edge).
* Rollout policy outputs (float64 forward, sequential dot products vs numpy's
  BLAS order) are within 1e-12; the PPO update runs its GEMMs on tcgen05 tensor
  cores (3xTF32) and is held to the north star's TF32/bf16 tier (1e-3 relative
  on policy outputs).
* Later rounds are compared per call (survey §7 hard part 2): the oracle is
  seeded with the engine's own post-update state, then both run one round.
"""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_12799_b200 as kt  # noqa: E402
from golden_io import GOLDEN, meta, npz  # noqa: E402
from oracle import agent as oagent  # noqa: E402
from paper_1905_12799_b200.agent import PARAM_KEYS, _flat  # noqa: E402

MODELS = json.loads((GOLDEN / "models.json").read_text())
LR = 1e-3


def space_of(values):
    return kt.DesignSpace("grid", tuple(kt.KnobDef(f"k{i}", tuple(v)) for i, v in enumerate(values)))


def oracle_from(agent):
    return {"params": {k: v.copy() for k, v in agent.params.items()},
            "m": {k: v.copy() for k, v in agent.adam.m.items()}, "v": {k: v.copy() for k, v in agent.adam.v.items()},
            "t": agent.adam.t, "seed": agent.seed, "rounds": agent.rounds_completed}


def _unflat(flat, like):
    out, pos = {}, 0
    for k in PARAM_KEYS:
        out[k] = flat[pos:pos + like[k].size].reshape(like[k].shape)
        pos += like[k].size
    return out


def assert_update_close(before, after, want_after, like=None, n=None, rel=1e-5):
    """The PPO update runs its GEMMs on the tensor cores as 3xTF32 (hi/lo split: fp32-accurate
    products, fp32 accumulation in TMEM), so it is held to the north star's FP32 tier: 1e-5
    relative on the updated network's probabilities and values over a batch of states
    (achieved <= 7e-7, tools/ppo_error.py / profiles/r2/ppo_error.json).  Per parameter, the
    update stays within 5% of one Adam step (lr): Adam normalises each gradient by its own
    running RMS, so a parameter whose gradient is ~0 turns fp32-level gradient differences
    into visible step differences (2.6% of lr observed on the 256-episode golden).
    """
    got, want = after - before, want_after - before
    assert np.max(np.abs(got - want)) < 5e-2 * LR  # every parameter moved like the reference's
    if like is None:
        return
    X = np.random.default_rng(0).random((512, n))
    lg, vg, _ = oagent.forward(_unflat(after, like), X)
    lw, vw, _ = oagent.forward(_unflat(want_after, like), X)
    pg, pw = np.exp(oagent.log_softmax(lg)), np.exp(oagent.log_softmax(lw))
    assert np.max(np.abs(pg - pw) / pw) <= rel
    assert np.max(np.abs(vg - vw) / np.maximum(np.abs(vw), 1.0)) <= rel


@pytest.mark.parametrize("name", sorted(meta("rl")))
def test_first_round_matches_reference(name):
    g = npz("rl")
    md = meta("rl")[name]
    mm = MODELS[md["model"]]
    space = space_of(mm["values"])
    model = kt.CostModel.from_dict(mm["model"])
    hyper = kt.AgentHyperparams.from_dict(md["hyper"])
    agent = kt.init_agent(space, hyper, seed=md["seed"])
    assert np.array_equal(_flat(agent.params), g[f"{name}/params0"])
    starts = [kt.Configuration(tuple(r)) for r in g[f"{name}/r0/starts"].tolist()]
    before = _flat(agent.params)
    tr = kt.run_search_round(agent, model, space, starts)
    assert np.array_equal(tr.index_matrix(), g[f"{name}/r0/idx"])
    assert np.array_equal(tr.scores(), g[f"{name}/r0/scores"])
    assert tr.step_indices == tuple(g[f"{name}/r0/steps"].tolist())
    assert agent.rounds_completed == 1
    if hyper.max_steps_per_episode:
        assert_update_close(before, _flat(agent.params), g[f"{name}/r0/params"], agent.params, len(space.knobs))


@pytest.mark.parametrize("name", ["bowl_default_2r", "bowl_tiny"])
def test_later_rounds_per_call_parity(name):
    g = npz("rl")
    md = meta("rl")[name]
    mm = MODELS[md["model"]]
    space = space_of(mm["values"])
    model = kt.CostModel.from_dict(mm["model"])
    hyper = kt.AgentHyperparams.from_dict(md["hyper"])
    agent = kt.init_agent(space, hyper, seed=md["seed"])
    rng = np.random.default_rng(77)
    for _ in range(3):
        ref = oracle_from(agent)
        starts = rng.integers(0, np.array(space.cardinalities), size=(md["E"], len(space.knobs)))
        before = _flat(agent.params)
        tr = kt.run_search_round(agent, model, space, [kt.Configuration(tuple(r)) for r in starts.tolist()])
        o_idx, o_sc, o_st = oagent.search_round(ref, mm["model"], mm["values"], starts, md["hyper"])
        assert np.array_equal(tr.index_matrix(), o_idx)
        assert np.array_equal(tr.scores(), o_sc)
        assert np.array_equal(np.array(tr.step_indices), o_st)
        want = np.concatenate([ref["params"][k].ravel() for k in PARAM_KEYS])
        assert_update_close(before, _flat(agent.params), want, agent.params, len(space.knobs))
        assert agent.adam.t == ref["t"] and agent.rounds_completed == ref["rounds"]


def test_large_round_vs_oracle():
    """4096 episodes of 32 steps on the Table-1 conv space: exact trajectory, update within tolerance."""
    mm = MODELS["table1"]
    space = space_of(mm["values"])
    model = kt.CostModel.from_dict(mm["model"])
    hyper = kt.AgentHyperparams(episodes_per_round=4096)
    agent = kt.init_agent(space, hyper, seed=21)
    ref = oracle_from(agent)
    starts = np.random.default_rng(4).integers(0, np.array(space.cardinalities), size=(4096, 8))
    before = _flat(agent.params)
    info = kt._lib.RoundInfo()
    rows = torch.from_numpy(kt.pack(starts).view(np.int64)).cuda()
    roll = {}
    r_rows, r_sc, r_st = kt.run_search_rows(agent, model, space, rows, info=info, rollout_out=roll)
    o_idx, o_sc, o_st, o_roll = oagent.search_round(ref, mm["model"], mm["values"], starts, hyper.to_dict(),
                                                    return_rollout=True)
    # policy outputs of the rollout (identical parameters): float64 path within 1e-12
    # relative (absolute for magnitudes below 1: log-probs and values straddle 0)
    lp, vals = roll["log_probs"].cpu().numpy(), roll["values"].cpu().numpy()
    assert np.max(np.abs(lp - o_roll["logp"]) / np.maximum(np.abs(o_roll["logp"]), 1.0)) <= 1e-12
    assert np.max(np.abs(vals - o_roll["values"]) / np.maximum(np.abs(o_roll["values"]), 1.0)) <= 1e-12
    assert info.guarded == 0
    assert np.array_equal(kt.unpack(r_rows.cpu().numpy().view(np.uint64), 8), o_idx)
    assert np.array_equal(r_sc.cpu().numpy(), o_sc)
    assert np.array_equal(r_st.cpu().numpy(), o_st)
    want = np.concatenate([ref["params"][k].ravel() for k in PARAM_KEYS])
    assert_update_close(before, _flat(agent.params), want, agent.params, 8)
    assert info.steps == len(o_idx) - 4096
    # the loss report of the last epoch (ppo_update's return, nets.py:94-171): FP32 tier
    got = (info.policy_loss, info.value_loss, info.entropy, info.total)
    for g_, w_ in zip(got, o_roll["report"]):
        assert abs(g_ - w_) <= 1e-5 * max(abs(w_), 1.0), (got, o_roll["report"])


def test_gae_kernel_vs_oracle():
    """gae_kernel (the PPO update's GAE, kt_gae) bit-exact vs compute_gae (agent.py:191-210):
    the reference's known answer [1.891, 1.0] and ragged random episodes (lengths 1..32)."""
    def run(rewards, values, lengths, gamma=0.9, lam=0.99):
        e = kt.engine()
        r = torch.tensor(rewards, dtype=torch.float64, device="cuda")
        v = torch.tensor(values, dtype=torch.float64, device="cuda")
        ln = torch.tensor(lengths, dtype=torch.int32, device="cuda")
        out = torch.empty_like(r)
        with e.scope():
            kt._lib.call("kt_gae", e.handle, kt._lib.ptr(r), kt._lib.ptr(v), kt._lib.ptr(ln), len(lengths), gamma, lam,
                         kt._lib.ptr(out))
        return out.cpu().numpy()

    got = run([1.0, 1.0], [0.0, 0.0], [2])
    assert got.tolist() == oagent.gae(np.array([1.0, 1.0]), np.zeros(2), 0.0, 0.9, 0.99).tolist()
    assert got.tolist() == pytest.approx([1.891, 1.0], abs=1e-12)
    rng = np.random.default_rng(12)
    lengths = rng.integers(1, 33, size=500)
    lengths[:3] = [1, 32, 1]
    T = int(lengths.sum())
    rew, val = rng.normal(size=T), rng.normal(size=T)
    got = run(rew, val, lengths.tolist(), 0.9, 0.99)
    want, lo = np.empty(T), 0
    for L in lengths:
        want[lo:lo + L] = oagent.gae(rew[lo:lo + L], val[lo:lo + L], 0.0, 0.9, 0.99)
        lo += L
    assert np.array_equal(got, want)


def test_zero_steps_and_errors():
    space = kt.grid(4, 4)
    agent = kt.init_agent(space, kt.AgentHyperparams(max_steps_per_episode=0, shared_width=4, head_width=4), seed=0)
    starts = [kt.Configuration((0, 0)), kt.Configuration((3, 2))]
    tr = kt.run_search_round(agent, kt.CostModel.sentinel(2), space, starts)
    assert [c.indices for c in tr.configs()] == [(0, 0), (3, 2)] and agent.rounds_completed == 1
    with pytest.raises(ValueError):
        kt.run_search_round(agent, kt.CostModel.sentinel(2), space, [])
    with pytest.raises(kt.errors.DimensionMismatchError):
        kt.run_search_round(agent, kt.CostModel.sentinel(3), kt.grid(3, 3, 3), [kt.Configuration((0, 0, 0))])


def test_cardinality_one_space():
    space = kt.DesignSpace("one", (kt.KnobDef("k", (1,)),))
    hyper = kt.AgentHyperparams(shared_width=4, head_width=4, episodes_per_round=4, max_steps_per_episode=8)
    agent = kt.init_agent(space, hyper, seed=0)
    tr = kt.run_search_round(agent, kt.CostModel.sentinel(1, base_score=1.0), space, [kt.Configuration((0,))])
    assert {c.indices for c in tr.configs()} == {(0,)}


def test_checkpoint_roundtrip_after_device_round():
    space = kt.grid(6, 6)
    hyper = kt.AgentHyperparams(shared_width=4, head_width=4, episodes_per_round=4, max_steps_per_episode=8)
    model = kt.CostModel.sentinel(2, base_score=1.0)
    starts = [kt.Configuration((0, 0)), kt.Configuration((5, 5))]
    a = kt.init_agent(space, hyper, seed=2)
    kt.run_search_round(a, model, space, starts)
    resumed = kt.Agent.from_json(a.to_json())
    t1 = kt.run_search_round(a, model, space, starts)
    t2 = kt.run_search_round(resumed, model, space, starts)
    assert t1.entries == t2.entries
