"""Oracle: actor-critic MLP, PPO update and lockstep search round (TEST INFRASTRUCTURE ONLY).

Restates, in float64 numpy:

* ``init_params``        <- nets.py:29-48 + agent.py:179-188 (Xavier-uniform, biases 0)
* ``forward``            <- nets.py:51-60  (tanh trunk -> policy logits (B,n,3) + value)
* ``log_softmax``        <- nets.py:63-65
* ``loss_and_grads``     <- nets.py:94-171 (clipped PPO + value MSE - entropy, analytic grads)
* ``adam_step``          <- nets.py:189-200
* ``gae``                <- agent.py:191-210
* ``ppo_update``         <- agent.py:218-258
* ``sample_actions``     <- agent.py:261-264 (inverse CDF with host uniforms)
* ``search_round``       <- agent.py:267-366 (lockstep episodes, one surrogate query, PPO)

The agent is a plain dict: ``{"params": {...}, "m": {...}, "v": {...}, "t": int,
"seed": int, "rounds": int}``.  Matrix products use the same operand shapes and
orientation as the reference so OpenBLAS rounds identically on the same host.
"""

from __future__ import annotations

import numpy as np

from .trees import feature_table, predict_features

KEYS = ("w1", "b1", "w2p", "b2p", "w3p", "b3p", "w2v", "b2v", "w3v", "b3v")
BETA1, BETA2, EPS = 0.9, 0.999, 1e-8
REWARD_STD_FLOOR = 1e-8

DEFAULT_HYPER = dict(adam_step_size=1e-3, discount=0.9, gae_parameter=0.99, epochs=3, clip=0.3,
                     value_coef=1.0, entropy_coef=0.1, episodes_per_round=64,
                     max_steps_per_episode=32, shared_width=128, head_width=64)


def init_params(n: int, h: int, g: int, seed: int) -> dict:
    rng = np.random.default_rng(np.random.SeedSequence(int(seed) & (2**64 - 1)))

    def xavier(fan_out, fan_in):
        a = np.sqrt(6.0 / (fan_in + fan_out))
        return rng.uniform(-a, a, size=(fan_out, fan_in))

    w1 = xavier(h, n)
    w2p = xavier(g, h)
    w3p = xavier(3 * n, g)
    w2v = xavier(g, h)
    w3v = xavier(1, g)
    return {"w1": w1, "b1": np.zeros(h), "w2p": w2p, "b2p": np.zeros(g), "w3p": w3p,
            "b3p": np.zeros(3 * n), "w2v": w2v, "b2v": np.zeros(g), "w3v": w3v, "b3v": np.zeros(1)}


def new_agent(n: int, hyper: dict, seed: int) -> dict:
    p = init_params(n, hyper["shared_width"], hyper["head_width"], seed)
    return {"params": p, "m": {k: np.zeros_like(v) for k, v in p.items()},
            "v": {k: np.zeros_like(v) for k, v in p.items()}, "t": 0, "seed": int(seed), "rounds": 0}


def forward(p: dict, X: np.ndarray):
    B = X.shape[0]
    h1 = np.tanh(X @ p["w1"].T + p["b1"])
    hp = np.tanh(h1 @ p["w2p"].T + p["b2p"])
    logits = (hp @ p["w3p"].T + p["b3p"]).reshape(B, -1, 3)
    hv = np.tanh(h1 @ p["w2v"].T + p["b2v"])
    values = (hv @ p["w3v"].T + p["b3v"])[:, 0]
    return logits, values, (X, h1, hp, hv)


def log_softmax(z: np.ndarray) -> np.ndarray:
    s = z - z.max(axis=-1, keepdims=True)
    return s - np.log(np.exp(s).sum(axis=-1, keepdims=True))


def joint_log_prob(logits: np.ndarray, actions: np.ndarray) -> np.ndarray:
    lp = log_softmax(logits)
    B, n, _ = logits.shape
    return lp[np.arange(B)[:, None], np.arange(n)[None, :], actions].sum(axis=1)


def loss_and_grads(p, X, actions, old_logp, adv, returns, clip, value_coef, entropy_coef):
    B = X.shape[0]
    logits, values, (X, h1, hp, hv) = forward(p, X)
    lp = log_softmax(logits)
    probs = np.exp(lp)
    new_logp = joint_log_prob(logits, actions)
    ratio = np.exp(new_logp - old_logp)
    raw = ratio * adv
    clipped = np.clip(ratio, 1.0 - clip, 1.0 + clip) * adv
    policy_loss = -float(np.minimum(raw, clipped).mean())
    knob_entropy = -(probs * lp).sum(axis=-1)
    entropy = float(knob_entropy.sum(axis=-1).mean())
    err = values - returns
    value_loss = float(np.mean(err * err))
    total = policy_loss + value_coef * value_loss - entropy_coef * entropy

    n = logits.shape[1]
    coeff = np.where(raw <= clipped, adv * ratio, 0.0) / B
    onehot = np.zeros_like(logits)
    onehot[np.arange(B)[:, None], np.arange(n)[None, :], actions] = 1.0
    d_logits = -coeff[:, None, None] * (onehot - probs)
    d_logits += (entropy_coef / B) * probs * (lp + knob_entropy[:, :, None])
    d_values = value_coef * 2.0 * err / B
    dz = d_logits.reshape(B, 3 * n)
    dv = d_values[:, None]

    gr = {}
    gr["w3p"] = dz.T @ hp
    gr["b3p"] = dz.sum(axis=0)
    d2p = (dz @ p["w3p"]) * (1.0 - hp * hp)
    gr["w2p"] = d2p.T @ h1
    gr["b2p"] = d2p.sum(axis=0)
    gr["w3v"] = dv.T @ hv
    gr["b3v"] = dv.sum(axis=0)
    d2v = (dv @ p["w3v"]) * (1.0 - hv * hv)
    gr["w2v"] = d2v.T @ h1
    gr["b2v"] = d2v.sum(axis=0)
    d1 = (d2p @ p["w2p"] + d2v @ p["w2v"]) * (1.0 - h1 * h1)
    gr["w1"] = d1.T @ X
    gr["b1"] = d1.sum(axis=0)
    return (policy_loss, value_loss, entropy, total), gr


def adam_step(agent: dict, grads: dict, lr: float) -> None:
    agent["t"] += 1
    c1 = 1.0 - BETA1 ** agent["t"]
    c2 = 1.0 - BETA2 ** agent["t"]
    for k in agent["params"]:
        g = grads[k]
        agent["m"][k] = BETA1 * agent["m"][k] + (1.0 - BETA1) * g
        agent["v"][k] = BETA2 * agent["v"][k] + (1.0 - BETA2) * (g * g)
        agent["params"][k] -= lr * (agent["m"][k] / c1) / (np.sqrt(agent["v"][k] / c2) + EPS)


def gae(rewards, values, terminal, discount, lam):
    rewards = np.asarray(rewards, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    delta = rewards + discount * np.append(values[1:], terminal) - values
    out = np.empty_like(delta)
    run = 0.0
    for t in range(delta.shape[0] - 1, -1, -1):
        run = delta[t] + discount * lam * run
        out[t] = run
    return out


def ppo_update(agent, states, actions, logp, rewards, values, bounds, hyper):
    adv = np.empty(states.shape[0])
    lo = 0
    for hi in bounds:
        adv[lo:hi] = gae(rewards[lo:hi], values[lo:hi], 0.0, hyper["discount"], hyper["gae_parameter"])
        lo = hi
    sd = float(adv.std())
    if sd < REWARD_STD_FLOOR:
        adv = np.zeros_like(adv)
        returns = values.copy()
    else:
        returns = adv + values
        adv = (adv - adv.mean()) / sd
    report = (0.0, 0.0, 0.0, 0.0)
    for _ in range(hyper["epochs"]):
        report, grads = loss_and_grads(agent["params"], states, actions, logp, adv, returns,
                                       hyper["clip"], hyper["value_coef"], hyper["entropy_coef"])
        adam_step(agent, grads, hyper["adam_step_size"])
    return report


def sample_actions(probs: np.ndarray, u: np.ndarray) -> np.ndarray:
    cdf = np.cumsum(probs, axis=-1)
    return (u[..., None] > cdf[..., :2]).sum(axis=-1)


def episode_uniforms(seed: int, round_index: int, episode: int, steps: int, n: int) -> np.ndarray:
    """The (steps, n) uniforms episode ``episode`` would draw (agent.py:292-296, :313)."""
    g = np.random.default_rng(np.random.SeedSequence(int(seed) & (2**64 - 1), spawn_key=(round_index, episode)))
    return g.random((steps, n))


def search_round(agent: dict, model: dict, knob_values, starts, hyper: dict, return_rollout: bool = False):
    """Returns (entries_idx (N,n), scores (N,), step_indices (N,)); mutates ``agent``."""
    cards = np.array([len(v) for v in knob_values], dtype=np.int64)
    n = cards.size
    starts = np.asarray(starts, dtype=np.int64).reshape(-1, n)
    E = starts.shape[0]
    table, _ = feature_table(knob_values)
    knob_axis = np.arange(n)
    S = hyper["max_steps_per_episode"]
    if S == 0:
        scores = predict_features(model, table[knob_axis[None, :], starts])
        agent["rounds"] += 1
        return starts.copy(), scores, np.zeros(E, dtype=np.int64)

    r = agent["rounds"]
    U = [episode_uniforms(agent["seed"], r, e, S, n) for e in range(E)]
    denom = np.maximum(1, cards - 1).astype(np.float64)
    cur = starts.copy()
    path = [[cur[e].copy()] for e in range(E)]
    st = [[] for _ in range(E)]
    ac = [[] for _ in range(E)]
    lpb = [[] for _ in range(E)]
    vb = [[] for _ in range(E)]
    live = list(range(E))
    for step in range(S):
        if not live:
            break
        X = cur[live] / denom[None, :]
        logits, values, _ = forward(agent["params"], X)
        probs = np.exp(log_softmax(logits))
        u = np.stack([U[e][step] for e in live])
        a = sample_actions(probs, u)
        lp = joint_log_prob(logits, a)
        nxt_live = []
        for row, e in enumerate(live):
            moved = np.minimum(np.maximum(cur[e] + (a[row] - 1), 0), cards - 1)
            st[e].append(X[row])
            ac[e].append(a[row])
            lpb[e].append(float(lp[row]))
            vb[e].append(float(values[row]))
            path[e].append(moved)
            cur[e] = moved
            if (a[row] != 1).any():
                nxt_live.append(e)
        live = nxt_live

    flat = np.array([c for ep in path for c in ep], dtype=np.int64)
    scores = predict_features(model, table[knob_axis[None, :], flat])
    steps_idx = np.array([s for ep in path for s in range(len(ep))], dtype=np.int64)
    rewards = []
    pos = 0
    for ep in path:
        rewards.append(np.asarray(scores[pos + 1: pos + len(ep)], dtype=np.float64))
        pos += len(ep)
    allr = np.concatenate(rewards)
    mu, sd = float(allr.mean()), float(allr.std())
    if sd < REWARD_STD_FLOOR:
        normed = [np.zeros_like(x) for x in rewards]
    else:
        normed = [(x - mu) / sd for x in rewards]
    bounds = list(np.cumsum([len(s) for s in st]))
    rollout = dict(
        states=np.concatenate([np.stack(s) for s in st]),
        actions=np.concatenate([np.stack(x) for x in ac]),
        logp=np.array([x for ep in lpb for x in ep], dtype=np.float64),
        rewards=np.concatenate(normed),
        values=np.array([x for ep in vb for x in ep], dtype=np.float64),
        bounds=bounds,
    )
    # the loss report of the last epoch (policy, value, entropy, total), as ppo_update returns it
    rollout["report"] = ppo_update(agent, rollout["states"], rollout["actions"], rollout["logp"], rollout["rewards"],
                                   rollout["values"], rollout["bounds"], hyper)
    agent["rounds"] += 1
    if return_rollout:
        return flat, scores, steps_idx, rollout
    return flat, scores, steps_idx
