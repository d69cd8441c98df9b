"""PPO search agents on the B200 (K1 rollout, K4 GAE, K5 PPO) — drop-in for knobtuner/agent.py.

``run_search_round(agent, model, space, starts)`` keeps the reference's
signature, validation, RNG streams, in-place mutation of the agent (params,
Adam state, rounds_completed) and episode-major trajectory (agent.py:267-366).
The whole round runs in libknobtuner_b200 (csrc/rollout.cu, csrc/ppo.cu):
rollout of all episodes in one kernel, surrogate scoring of every visited
configuration, reward/advantage statistics in numpy's float64 order, and the
PPO epochs with float64 master weights and Adam moments.

Agents may be the reference's ``Agent`` objects or this module's mirror;
their float64 host parameters are synchronised after every round so
checkpoints (``to_json``) keep working.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field, fields

import numpy as np

from . import _lib, errors
from . import space as sp
from .cost_model import _check_model, device_forest, predict
from .sa import seed_words
from .trajectory import Trajectory

PARAM_KEYS = ("w1", "b1", "w2p", "b2p", "w3p", "b3p", "w2v", "b2v", "w3v", "b3v")
CHECKPOINT_VERSION = 1


@dataclass(frozen=True)
class AgentHyperparams:
    """Mirror of agent.py:30-71 (Table-2 defaults, same validation messages)."""

    adam_step_size: float = 1e-3
    discount: float = 0.9
    gae_parameter: float = 0.99
    epochs: int = 3
    clip: float = 0.3
    value_coef: float = 1.0
    entropy_coef: float = 0.1
    episodes_per_round: int = 64
    max_steps_per_episode: int = 32
    shared_width: int = 128
    head_width: int = 64

    def __post_init__(self) -> None:
        for f in fields(self):
            value = getattr(self, f.name)
            if not np.isfinite(value):
                raise ValueError(f"{f.name} must be finite, got {value}")
        if not 0.0 < self.discount <= 1.0:
            raise ValueError(f"discount must be in (0, 1], got {self.discount}")
        if not 0.0 < self.gae_parameter <= 1.0:
            raise ValueError(f"gae_parameter must be in (0, 1], got {self.gae_parameter}")
        if self.clip <= 0.0:
            raise ValueError(f"clip must be > 0, got {self.clip}")
        if self.adam_step_size <= 0.0:
            raise ValueError(f"adam_step_size must be > 0, got {self.adam_step_size}")
        if self.epochs < 1:
            raise ValueError(f"epochs must be >= 1, got {self.epochs}")
        if self.episodes_per_round < 1:
            raise ValueError(f"episodes_per_round must be >= 1, got {self.episodes_per_round}")
        if self.max_steps_per_episode < 0:
            raise ValueError(f"max_steps_per_episode must be >= 0, got {self.max_steps_per_episode}")
        if self.shared_width < 1 or self.head_width < 1:
            raise ValueError("network widths must be >= 1")

    def to_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    @classmethod
    def from_dict(cls, obj: dict) -> "AgentHyperparams":
        return cls(**obj)


@dataclass
class AdamState:
    m: dict = field(default_factory=dict)
    v: dict = field(default_factory=dict)
    t: int = 0


@dataclass
class Agent:
    space_knobs: int
    hyper: AgentHyperparams
    seed: int
    params: dict
    adam: AdamState
    rounds_completed: int = 0

    def to_json(self) -> str:
        return json.dumps({
            "version": CHECKPOINT_VERSION, "space_knobs": self.space_knobs, "hyper": self.hyper.to_dict(),
            "seed": self.seed, "rounds_completed": self.rounds_completed,
            "params": {k: v.tolist() for k, v in self.params.items()},
            "adam_m": {k: v.tolist() for k, v in self.adam.m.items()},
            "adam_v": {k: v.tolist() for k, v in self.adam.v.items()}, "adam_t": self.adam.t,
        }, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "Agent":
        obj = json.loads(text)
        if obj.get("version") != CHECKPOINT_VERSION:
            raise ValueError(f"unsupported checkpoint version {obj.get('version')}")
        arr = lambda d: {k: np.array(v, dtype=np.float64) for k, v in d.items()}
        return cls(space_knobs=int(obj["space_knobs"]), hyper=AgentHyperparams.from_dict(obj["hyper"]),
                   seed=int(obj["seed"]), params=arr(obj["params"]),
                   adam=AdamState(m=arr(obj["adam_m"]), v=arr(obj["adam_v"]), t=int(obj["adam_t"])),
                   rounds_completed=int(obj["rounds_completed"]))


def init_params(n_knobs: int, shared_width: int, head_width: int, rng: np.random.Generator) -> dict:
    """Xavier-uniform weights drawn in PARAM_KEYS order, zero biases (nets.py:29-48)."""
    if n_knobs < 1 or shared_width < 1 or head_width < 1:
        raise ValueError("network sizes must be positive")

    def xavier(fan_out: int, fan_in: int) -> np.ndarray:
        a = np.sqrt(6.0 / (fan_in + fan_out))
        return rng.uniform(-a, a, size=(fan_out, fan_in))

    w1 = xavier(shared_width, n_knobs)
    w2p = xavier(head_width, shared_width)
    w3p = xavier(3 * n_knobs, head_width)
    w2v = xavier(head_width, shared_width)
    w3v = xavier(1, head_width)
    return {"w1": w1, "b1": np.zeros(shared_width), "w2p": w2p, "b2p": np.zeros(head_width), "w3p": w3p,
            "b3p": np.zeros(3 * n_knobs), "w2v": w2v, "b2v": np.zeros(head_width), "w3v": w3v, "b3v": np.zeros(1)}


def init_agent(space, hyper: AgentHyperparams = AgentHyperparams(), seed: int = 0) -> Agent:
    rng = np.random.default_rng(np.random.SeedSequence(seed & (2**64 - 1)))
    params = init_params(len(space.knobs), hyper.shared_width, hyper.head_width, rng)
    return Agent(space_knobs=len(space.knobs), hyper=hyper, seed=seed, params=params,
                 adam=AdamState(m={k: np.zeros_like(v) for k, v in params.items()},
                                v={k: np.zeros_like(v) for k, v in params.items()}))


def _flat(d: dict) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate([np.asarray(d[k], dtype=np.float64).ravel() for k in PARAM_KEYS]))


def _unflat_into(flat: np.ndarray, d: dict) -> None:
    pos = 0
    for k in PARAM_KEYS:
        arr = d[k]
        size = arr.size
        arr[...] = flat[pos:pos + size].reshape(arr.shape)
        pos += size


class _DeviceAgent:
    """kt_agent handle plus the host snapshot it was last synchronised with."""

    def __init__(self, agent, engine: _lib.Engine):
        h, g = agent.hyper.shared_width, agent.hyper.head_width
        p, m, v = _flat(agent.params), _flat(agent.adam.m), _flat(agent.adam.v)
        handle = _lib.P()
        _lib.call("kt_agent_create", engine.handle, int(agent.space_knobs), int(h), int(g),
                  _lib.as_ptr(p, _lib.C.c_double), _lib.as_ptr(m, _lib.C.c_double), _lib.as_ptr(v, _lib.C.c_double),
                  int(agent.adam.t), _lib.C.byref(handle))
        self.handle = handle
        self.device = engine.device
        self.snapshot = (p, m, v, int(agent.adam.t))

    def matches(self, agent) -> bool:
        p, m, v, t = self.snapshot
        return (t == int(agent.adam.t) and np.array_equal(p, _flat(agent.params))
                and np.array_equal(m, _flat(agent.adam.m)) and np.array_equal(v, _flat(agent.adam.v)))

    def pull_into(self, agent, engine: _lib.Engine) -> None:
        size = self.snapshot[0].size
        p, m, v = (np.empty(size, dtype=np.float64) for _ in range(3))
        t = _lib.C.c_int64(0)
        _lib.call("kt_agent_get_state", engine.handle, self.handle, _lib.as_ptr(p, _lib.C.c_double),
                  _lib.as_ptr(m, _lib.C.c_double), _lib.as_ptr(v, _lib.C.c_double), _lib.C.byref(t))
        _unflat_into(p, agent.params)
        _unflat_into(m, agent.adam.m)
        _unflat_into(v, agent.adam.v)
        agent.adam.t = int(t.value)
        self.snapshot = (p, m, v, int(t.value))

    def __del__(self):
        try:
            _lib.load().kt_agent_destroy(self.handle)
        except Exception:
            pass


def _device_agent(agent, engine: _lib.Engine) -> _DeviceAgent:
    d = getattr(agent, "__dict__", {}).get("_b200_agent")
    if d is None or d.device != engine.device or not d.matches(agent):
        d = _DeviceAgent(agent, engine)
        try:
            object.__setattr__(agent, "_b200_agent", d)
        except (AttributeError, TypeError):
            pass
    return d


RoundInfo = _lib.RoundInfo
PPOHyper = _lib.PPOHyper


def run_search_rows(agent, model, space, start_rows, engine=None, info: RoundInfo | None = None,
                    rollout_out: dict | None = None, all_reduce=None, episode_offset: int = 0, collective=None):
    """Array path: CUDA int64 start rows -> (rows, scores, step indices) CUDA tensors; mutates ``agent``.

    ``rollout_out`` (optional dict) receives the rollout's per-step log-probs and
    values (Rollout.log_probs / values, agent.py:351-363) as CUDA float64 tensors.

    Sharded rounds (shard.run_search_rows_sharded): ``start_rows`` are the global
    episodes [episode_offset, episode_offset + E) and ``all_reduce(t)`` sums a CUDA
    float64 tensor in place over the ranks (reward / advantage statistics, batch
    size, per-epoch gradients, loss report).
    """
    import torch

    engine = engine or _lib.engine()
    hyper = agent.hyper
    _check_model(model, space)
    cards = sp.check_engine_space(space)
    f = device_forest(model, space, engine)
    if f.neg_prefix.any():
        raise ValueError("featurize requires non-negative knob values")
    dev_agent = _device_agent(agent, engine)
    E = int(start_rows.numel())
    S = int(hyper.max_steps_per_episode)
    cap = E * (S + 1)
    hp = PPOHyper(float(hyper.adam_step_size), float(hyper.discount), float(hyper.gae_parameter), float(hyper.clip),
                  float(hyper.value_coef), float(hyper.entropy_coef), int(hyper.epochs), S)
    words = seed_words(agent.seed)
    total = _lib.C.c_int64(0)
    info = info if info is not None else RoundInfo()
    with engine.scope():
        rows = torch.empty(cap, dtype=torch.int64, device=start_rows.device)
        scores = torch.empty(cap, dtype=torch.float64, device=start_rows.device)
        steps = torch.empty(cap, dtype=torch.int32, device=start_rows.device)
        lp = vals = None
        if rollout_out is not None:
            lp = torch.empty(E * S, dtype=torch.float64, device=start_rows.device)
            vals = torch.empty(E * S, dtype=torch.float64, device=start_rows.device)
        coll = collective  # a ready kt_collective (e.g. shard.NativeComm: NCCL inside the library)
        if coll is None and all_reduce is not None:
            errors_seen = []

            def _cb(user, ptr, count):
                try:
                    all_reduce(_lib.device_tensor(ptr, count, engine.device))
                    return 0
                except Exception as ex:  # surfaced as an engine error
                    errors_seen.append(ex)
                    return 1

            cb = _lib.ALL_REDUCE_F64(_cb)
            coll = _lib.Collective(cb, None, int(episode_offset))
        _lib.call("kt_search_round_ex", engine.handle, dev_agent.handle, f.handle, _lib.ptr(start_rows), E,
                  _lib.as_ptr(cards, _lib.C.c_int32), int(cards.size), _lib.as_ptr(words, _lib.C.c_uint32),
                  int(words.size), int(agent.rounds_completed), _lib.C.byref(hp), _lib.ptr(rows), _lib.ptr(scores),
                  _lib.ptr(steps), _lib.C.byref(total), _lib.C.byref(info),
                  _lib.ptr(lp) if lp is not None else None, _lib.ptr(vals) if vals is not None else None,
                  _lib.C.byref(coll) if coll is not None else None)
        if rollout_out is not None:
            rollout_out["log_probs"] = lp[: info.steps]
            rollout_out["values"] = vals[: info.steps]
    dev_agent.pull_into(agent, engine)
    agent.rounds_completed += 1
    n = int(total.value)
    return rows[:n], scores[:n], steps[:n]


def run_search_round(agent, model, space, starts) -> Trajectory:
    """One search round: episodes from each start, one PPO update, trajectory out (agent.py:267-366)."""
    import torch

    if not starts:
        raise ValueError("run_search_round needs at least one start configuration")
    if len(space.knobs) != agent.space_knobs:
        raise errors.DimensionMismatchError(
            f"agent built for {agent.space_knobs} knobs, space has {len(space.knobs)}")
    idx = sp.index_matrix(space, starts)  # validate_config per start (agent.py:278-279)
    cls = type(starts[0])
    if agent.hyper.max_steps_per_episode == 0:
        scores = predict(model, space, starts)
        agent.rounds_completed += 1
        cards = sp.cardinalities(space)
        return Trajectory(sp.pack(idx, cards), scores, np.zeros(len(starts), dtype=np.int64),
                          n_knobs=len(space.knobs), config_cls=cls, cards=cards)
    engine = _lib.engine()
    with engine.scope():
        start_rows = torch.from_numpy(sp.pack(idx, sp.cardinalities(space)).view(np.int64)).to(f"cuda:{engine.device}")
    rows, scores, steps = run_search_rows(agent, model, space, start_rows, engine=engine)
    return Trajectory(rows, scores, steps, n_knobs=len(space.knobs), config_cls=cls, cards=sp.cardinalities(space))
