"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container, where the read-only reference is importable:

    python tests/golden/make_golden.py            # writes tests/golden/*.npz|json, data/models/*.json

The outputs are committed; the GPU box never reads /root/reference.  Every
fixture records inputs plus the reference's outputs, so the oracle
(``oracle/``) and the CUDA path can both be checked against the reference
itself.  Sizes are kept small (the whole directory stays a few MB).
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_PKG = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(ROOT))

from knobtuner import nets  # noqa: E402
from knobtuner.agent import AgentHyperparams, Trajectory, init_agent, run_search_round  # noqa: E402
from knobtuner.backends import SyntheticLandscape, gen_landscape, landscape_to_dict, load_landscape, synthetic_runtime  # noqa: E402
from knobtuner.cost_model import BoostParams, CostModel, TrainingSet, featurize_batch, fit, predict  # noqa: E402
from knobtuner.sa import SAParams, run_sa_round  # noqa: E402
from knobtuner.sampler import VisitedSet, adaptive_sample, kmeans, knee_scan, mode_config  # noqa: E402
from knobtuner.space import Configuration, DesignSpace, KnobDef, enumerate_space, load_space, random_config, space_from_dict  # noqa: E402

from paper_1905_12799_b200.workloads import RESNET18_S2  # noqa: E402


def grid(*cards):
    return DesignSpace(name="grid", knobs=tuple(KnobDef(f"k{i}", tuple(range(c))) for i, c in enumerate(cards)))


def values_of(space):
    return [list(k.values) for k in space.knobs]


def idx_of(configs):
    return np.array([c.indices for c in configs], dtype=np.int64)


def bowl_model(space, center):
    configs = list(enumerate_space(space))
    X = featurize_batch(space, configs)
    d2 = np.array([sum((i - c) ** 2 for i, c in zip(cfg.indices, center)) for cfg in configs], dtype=np.float64)
    return fit(TrainingSet(features=X, targets=3.0 - 0.01 * d2), BoostParams(rounds=30, depth=4))


def landscape_model(space, land, n_train, seed, params=BoostParams()):
    rng = np.random.default_rng(seed)
    train = [random_config(space, rng) for _ in range(n_train)]
    X = featurize_batch(space, train)
    y = np.array([1.0 / synthetic_runtime(land, c) for c in train])
    return fit(TrainingSet(features=X, targets=y), params)


def spaces():
    bench = load_space(REF_PKG / "spaces" / "bench_grid4d.json")
    table1 = load_space(REF_PKG / "spaces" / "conv_gpu_table1.json")
    s2 = space_from_dict(RESNET18_S2.space_dict())
    return bench, table1, s2


def make_models(out_models: dict):
    bench, table1, s2 = spaces()
    g10 = grid(10, 10, 10)
    models = {}
    models["bowl_g10"] = (g10, bowl_model(g10, (7, 2, 5)))
    land_b = load_landscape(REF_PKG / "landscapes" / "bench_grid4d_s0.json", bench)
    models["bench_s0"] = (bench, landscape_model(bench, land_b, 200, 2000))
    land_t1 = gen_landscape(table1, seed=1)
    models["table1"] = (table1, landscape_model(table1, land_t1, 500, 11))
    land_s2 = gen_landscape(s2, seed=1)
    models["s2_resnet18"] = (s2, landscape_model(s2, land_s2, 500, 12))
    models["s2_deep6"] = (s2, landscape_model(s2, land_s2, 300, 13, BoostParams(rounds=8, depth=6)))
    models["table1_stumps"] = (table1, landscape_model(table1, land_t1, 200, 14, BoostParams(rounds=20, depth=1)))
    models["sentinel3"] = (g10, CostModel.sentinel(3, base_score=0.25))
    for name, (space, model) in models.items():
        out_models[name] = {"values": values_of(space), "model": json.loads(model.to_json()), "space": space.name}
    return models, {"table1": land_t1, "s2": land_s2, "bench_s0": land_b}


def gen_predict(models, rng):
    cases = {}
    for name, (space, model) in models.items():
        cards = np.array(space.cardinalities)
        idx = rng.integers(0, cards, size=(3000, len(cards)))
        idx = np.vstack([idx, np.zeros(len(cards), dtype=np.int64), cards - 1])
        configs = [Configuration(tuple(r)) for r in idx.tolist()]
        cases[f"{name}/idx"] = idx
        cases[f"{name}/scores"] = predict(model, space, configs)
    return cases


def gen_landscapes(lands, rng):
    bench, table1, s2 = spaces()
    out_json = {}
    arrays = {}
    items = []
    for s in range(5):
        items.append((f"bench_s{s}", bench, load_landscape(REF_PKG / "landscapes" / f"bench_grid4d_s{s}.json", bench)))
    items.append(("table1_gen1", table1, lands["table1"]))
    items.append(("s2_gen1", s2, lands["s2"]))
    g = grid(10, 10)
    items.append(("neg_seed_noisy", g, SyntheticLandscape(seed=-3, space=g, centers=((5, 5), (1, 8)), depths=(0.5, 0.3), radii=(2.0, 1.5), noise_rel=0.3)))
    items.append(("big_seed", g, SyntheticLandscape(seed=2**40 + 7, space=g, centers=((2, 2),), depths=(0.9,), radii=(3.0,), base_runtime=2.5, noise_rel=0.05)))
    items.append(("noiseless", g, SyntheticLandscape(seed=1, space=g, centers=((0, 0),), depths=(0.9,), radii=(0.5,))))
    for name, space, land in items:
        cards = np.array(space.cardinalities)
        n_rows = 1500 if space.name != "grid" else 100
        idx = rng.integers(0, cards, size=(n_rows, len(cards)))
        idx = np.vstack([idx] + [np.array(c, dtype=np.int64)[None, :] for c in land.centers])
        rt = np.array([synthetic_runtime(land, Configuration(tuple(r))) for r in idx.tolist()])
        arrays[f"{name}/idx"] = idx
        arrays[f"{name}/runtime"] = rt
        out_json[name] = {"values": values_of(space), "landscape": landscape_to_dict(land)}
    return arrays, out_json


def clustered_points(cards, centers, per_center, seed):
    rng = np.random.default_rng(seed)
    out = []
    for center in centers:
        out.append(tuple(center))
        for _ in range(per_center - 1):
            p = list(center)
            if rng.random() < 0.4:
                d = int(rng.integers(0, len(center)))
                p[d] = min(max(p[d] + (1 if rng.random() < 0.5 else -1), 0), cards[d] - 1)
            out.append(tuple(p))
    return np.array(out, dtype=np.int64)


CENTERS10 = [(3, 3, 3), (3, 3, 27), (3, 27, 3), (3, 27, 27), (27, 3, 3), (27, 3, 27), (27, 27, 3), (27, 27, 27), (15, 15, 15), (3, 15, 15)]


def kmeans_cases(rng):
    cases = []
    cases.append(("quad1d", np.array([0.0, 1.0, 10.0, 11.0])[:, None], 2, 0))
    cases.append(("dup4", np.array([[0, 0], [3, 1], [7, 7], [0, 0]], dtype=np.float64), 3, 1))
    cases.append(("k1", rng.integers(0, 10, size=(20, 3)).astype(np.float64), 1, 2))
    cases.append(("r60", rng.integers(0, 20, size=(60, 2)).astype(np.float64), 5, 3))
    cases.append(("r90", rng.integers(0, 30, size=(90, 2)).astype(np.float64), 6, 4))
    cl = clustered_points((31, 31, 31), CENTERS10, 20, 0).astype(np.float64)
    for k, s in ((8, 0), (10, 5), (14, 9)):
        cases.append((f"clustered_k{k}", cl, k, s))
    for s in range(12):
        m = int(rng.integers(9, 200))
        pts = rng.integers(0, int(rng.integers(2, 12)), size=(m, int(rng.integers(1, 9)))).astype(np.float64)
        nd = len({tuple(r) for r in pts})
        if nd < 1:
            continue
        k = int(rng.integers(1, min(nd, 20) + 1))
        cases.append((f"rand{s}", pts, k, 100 + s))
    s2 = np.array([len(v) for v in (RESNET18_S2.space_dict()["knobs"][i]["values"] for i in range(8))])
    lat = np.unique(rng.integers(0, s2, size=(3000, 8)), axis=0)
    lat = lat[rng.permutation(lat.shape[0])].astype(np.float64)
    cases.append(("s2_k8", lat, 8, 7))
    cases.append(("s2_k9", lat, 9, 7))
    t1 = np.array([7, 5, 5, 7, 2, 2, 5, 2])
    lat1 = np.unique(rng.integers(0, t1, size=(1500, 8)), axis=0)
    lat1 = lat1[rng.permutation(lat1.shape[0])].astype(np.float64)
    cases.append(("t1_k12", lat1, 12, 3))
    # a small, spread lattice where empty clusters are frequent
    cases.append(("line_k9", np.array([[i] for i in (0, 0, 1, 2, 3, 50, 51, 52, 100, 101, 150, 200)], dtype=np.float64), 9, 4))
    return cases


def gen_kmeans(rng):
    arrays = {}
    names = []
    for name, pts, k, seed in kmeans_cases(rng):
        res = kmeans(pts, k=k, seed=seed)
        arrays[f"{name}/points"] = pts
        arrays[f"{name}/meta"] = np.array([k, seed], dtype=np.int64)
        arrays[f"{name}/centroids"] = res.centroids
        arrays[f"{name}/assignment"] = res.assignment
        arrays[f"{name}/history"] = np.array(res.loss_history)
        names.append(name)
    return arrays, names


def gen_knee(rng):
    arrays = {}
    names = []
    cases = []
    for s in (7, 9):
        cases.append((f"clustered_s{s}", np.array(sorted({tuple(r) for r in clustered_points((31, 31, 31), CENTERS10, 20, s).tolist()}), dtype=np.float64), s))
    cases.append(("u150x3", rng.integers(0, 40, size=(150, 3)).astype(np.float64), 21))
    s2 = np.array([84, 80, 80, 7, 2, 2, 3, 2])
    lat = np.unique(rng.integers(0, s2, size=(4000, 8)), axis=0)
    lat = lat[rng.permutation(lat.shape[0])].astype(np.float64)
    cases.append(("s2_4000", lat, 123))
    for name, pts, seed in cases:
        res, scanned = knee_scan(pts, seed=seed)
        arrays[f"{name}/points"] = pts
        arrays[f"{name}/seed"] = np.array([seed], dtype=np.int64)
        arrays[f"{name}/scanned"] = np.array(scanned, dtype=np.float64)
        arrays[f"{name}/centroids"] = res.centroids
        arrays[f"{name}/assignment"] = res.assignment
        names.append(name)
    return arrays, names


def traj_of(idx):
    return Trajectory(entries=tuple((Configuration(tuple(r)), 0.0) for r in idx.tolist()))


def gen_adaptive(rng, models):
    arrays = {}
    meta = {}
    cases = []
    g31 = grid(31, 31, 31)
    for s in (0, 5):
        cases.append((f"clustered_s{s}", g31, clustered_points((31, 31, 31), CENTERS10, 20, s), [], s))
    g44 = grid(4, 4)
    cases.append(("collapse", g44, np.array([[2, 3]] * 40), [], 1))
    g66 = grid(6, 6)
    cases.append(("small", g66, np.array([[i, i] for i in range(5)] * 3), [(0, 0)], 2))
    g12 = grid(12, 12)
    allp = np.array([[i, j] for i in range(12) for j in range(12)])
    cases.append(("all_visited", g12, allp, [tuple(r) for r in allp.tolist()], 3))
    g9 = grid(9, 9, 9)
    for s in range(6):
        r = np.random.default_rng(s)
        pts = r.integers(0, 9, size=(int(r.integers(1, 120)), 3))
        vis = [tuple(r.integers(0, 9, size=3).tolist()) for _ in range(20)]
        cases.append((f"prop{s}", g9, pts, vis, s))
    _, table1, s2 = spaces()
    c1 = np.array(table1.cardinalities)
    pts = rng.integers(0, c1, size=(3000, 8))
    vis = [tuple(r) for r in pts[rng.integers(0, 3000, size=200)].tolist()]
    cases.append(("table1_uniform", table1, pts, vis, 77))
    c2 = np.array(s2.cardinalities)
    cases.append(("s2_uniform", s2, rng.integers(0, c2, size=(5000, 8)), [], 99))
    # a real RL round on table1
    space, model = models["table1"]
    agent = init_agent(space, AgentHyperparams(episodes_per_round=64), seed=3)
    st_rng = np.random.default_rng(5)
    starts = [random_config(space, st_rng) for _ in range(64)]
    tr = run_search_round(agent, model, space, starts)
    idx = idx_of(tr.configs())
    cases.append(("table1_rl_round", table1, idx, [tuple(r) for r in idx_of(starts).tolist()], 1234))
    # visited centroids replaced by mode
    cl = clustered_points((31, 31, 31), CENTERS10, 20, 5)
    probe = adaptive_sample(traj_of(cl), VisitedSet(), g31, seed=6)
    mode = mode_config(traj_of(cl), g31)
    cases.append(("mode_replace", g31, cl, [c.indices for c in probe if c != mode], 6))
    for name, space, pts, vis, seed in cases:
        batch = adaptive_sample(traj_of(np.asarray(pts)), VisitedSet([Configuration(v) for v in vis]), space, seed=seed)
        arrays[f"{name}/idx"] = np.asarray(pts, dtype=np.int64)
        arrays[f"{name}/visited"] = np.array(vis, dtype=np.int64).reshape(-1, space.n_knobs)
        arrays[f"{name}/batch"] = idx_of(batch).reshape(-1, space.n_knobs)
        arrays[f"{name}/mode"] = np.array(mode_config(traj_of(np.asarray(pts)), space).indices, dtype=np.int64)
        meta[name] = {"cards": list(space.cardinalities), "seed": seed}
    return arrays, meta


def gen_sa(models):
    arrays = {}
    meta = {}
    g10, bowl = models["bowl_g10"]
    table1, m1 = models["table1"]
    s2, m2 = models["s2_resnet18"]
    cases = []
    r = np.random.default_rng(17)
    cases.append(("bowl_4x500", "bowl_g10", SAParams(chains=4, steps_per_round=500), [random_config(g10, r) for _ in range(4)], 17))
    cases.append(("bowl_hot", "bowl_g10", SAParams(chains=2, steps_per_round=300, initial_temperature=1e12, cooling=1.0), [Configuration((0, 0, 0)), Configuration((9, 9, 9))], 0))
    cases.append(("bowl_cold", "bowl_g10", SAParams(chains=1, steps_per_round=300, initial_temperature=1e-12, cooling=1.0), [Configuration((0, 0, 0))], 3))
    cases.append(("bowl_pad", "bowl_g10", SAParams(chains=8, steps_per_round=20), [Configuration((0, 0, 0))], 5))
    r = np.random.default_rng(23)
    cases.append(("table1_64x128", "table1", SAParams(), [random_config(table1, r) for _ in range(64)], 2**63 + 5))
    r = np.random.default_rng(29)
    cases.append(("s2_256x64", "s2_resnet18", SAParams(chains=256, steps_per_round=64), [random_config(s2, r) for _ in range(256)], 31))
    for name, model_name, params, starts, seed in cases:
        space, model = models[model_name]
        tr = run_sa_round(params, model, space, starts, seed)
        arrays[f"{name}/starts"] = idx_of(starts)
        arrays[f"{name}/idx"] = idx_of(tr.configs())
        arrays[f"{name}/scores"] = tr.scores()
        arrays[f"{name}/steps"] = np.array(tr.step_indices, dtype=np.int64)
        meta[name] = {"model": model_name, "chains": params.chains, "steps": params.steps_per_round,
                      "initial_temperature": params.initial_temperature, "cooling": params.cooling, "seed": seed}
    return arrays, meta


def gen_rl(models):
    arrays = {}
    meta = {}
    cases = []
    g10, bowl = models["bowl_g10"]
    cases.append(("bowl_default_2r", "bowl_g10", AgentHyperparams(), 0, 2, 64, 123))
    cases.append(("bowl_tiny", "bowl_g10", AgentHyperparams(shared_width=4, head_width=4, episodes_per_round=4, max_steps_per_episode=8), 11, 2, 4, 5))
    cases.append(("table1_256", "table1", AgentHyperparams(episodes_per_round=256), 3, 1, 256, 9))
    cases.append(("zero_steps", "bowl_g10", AgentHyperparams(max_steps_per_episode=0), 1, 1, 8, 4))
    for name, model_name, hyper, seed, rounds, E, start_seed in cases:
        space, model = models[model_name]
        agent = init_agent(space, hyper, seed=seed)
        st_rng = np.random.default_rng(start_seed)
        arrays[f"{name}/params0"] = nets.flatten_params(agent.params)
        for rd in range(rounds):
            starts = [random_config(space, st_rng) for _ in range(E)]
            tr = run_search_round(agent, model, space, starts)
            arrays[f"{name}/r{rd}/starts"] = idx_of(starts)
            arrays[f"{name}/r{rd}/idx"] = idx_of(tr.configs())
            arrays[f"{name}/r{rd}/scores"] = tr.scores()
            arrays[f"{name}/r{rd}/steps"] = np.array(tr.step_indices, dtype=np.int64)
            arrays[f"{name}/r{rd}/params"] = nets.flatten_params(agent.params)
            arrays[f"{name}/r{rd}/adam_m"] = nets.flatten_params(agent.adam.m)
            arrays[f"{name}/r{rd}/adam_v"] = nets.flatten_params(agent.adam.v)
        meta[name] = {"model": model_name, "hyper": hyper.to_dict(), "seed": seed, "rounds": rounds, "E": E}
    return arrays, meta


def make_task_models():
    """Surrogates for the ResNet-18 conv tasks used by the RL bench mode (data/models/)."""
    from paper_1905_12799_b200.workloads import RESNET18_TASKS

    out = ROOT / "data" / "models"
    for i, task in enumerate(RESNET18_TASKS[:5]):
        space = space_from_dict(task.space_dict())
        land = gen_landscape(space, seed=100 + i)
        model = landscape_model(space, land, 500, 200 + i)
        doc = {"values": values_of(space), "model": json.loads(model.to_json()), "space": space.name,
               "landscape": landscape_to_dict(land)}
        (out / f"resnet18_task{i}.json").write_text(json.dumps(doc, sort_keys=True))


def make_alexnet_models():
    """Surrogates + landscapes for AlexNet's 5 conv tasks (configs[1]; bit-field rows)."""
    from paper_1905_12799_b200.workloads import ALEXNET_TASKS

    out = ROOT / "data" / "models"
    models = {}
    for i, task in enumerate(ALEXNET_TASKS):
        space = space_from_dict(task.space_dict())
        land = gen_landscape(space, seed=300 + i)
        model = landscape_model(space, land, 500, 400 + i)
        doc = {"values": values_of(space), "model": json.loads(model.to_json()), "space": space.name,
               "landscape": landscape_to_dict(land)}
        (out / f"alexnet_task{i}.json").write_text(json.dumps(doc, sort_keys=True))
        models[f"alexnet{i}"] = (space, model, land)
    return models


def gen_wide():
    """Golden vectors on spaces whose knobs exceed 255 settings (AlexNet conv3/conv4,
    plus a synthetic 8-knob space near the 63-bit row limit): every path once."""
    rng = np.random.default_rng(480)
    alex = make_alexnet_models()
    arrays, meta = {}, {"models": {}, "adaptive": {}, "sa": {}, "rl": {}}
    wide8 = space_from_dict({"name": "wide8", "knobs": [{"name": f"k{i}", "values": list(range(c))}
                                                        for i, c in enumerate((300, 257, 1000, 9, 2, 3, 70, 5))]})
    land_w8 = gen_landscape(wide8, seed=5)
    models = {"alexnet2": alex["alexnet2"][:2], "alexnet3": alex["alexnet3"][:2],
              "wide8": (wide8, landscape_model(wide8, land_w8, 400, 6))}
    for name, (space, model) in models.items():
        meta["models"][name] = {"values": values_of(space), "model": json.loads(model.to_json()), "space": space.name}
        cards = np.array(space.cardinalities)
        idx = rng.integers(0, cards, size=(3000, len(cards)))
        idx = np.vstack([idx, np.zeros(len(cards), dtype=np.int64), cards - 1])
        arrays[f"predict/{name}/idx"] = idx
        arrays[f"predict/{name}/scores"] = predict(model, space, [Configuration(tuple(r)) for r in idx.tolist()])
    for name, space, land in (("alexnet3", alex["alexnet3"][0], alex["alexnet3"][2]), ("wide8", wide8, land_w8)):
        cards = np.array(space.cardinalities)
        idx = rng.integers(0, cards, size=(1500, len(cards)))
        idx = np.vstack([idx] + [np.array(c, dtype=np.int64)[None, :] for c in land.centers])
        arrays[f"landscape/{name}/idx"] = idx
        arrays[f"landscape/{name}/runtime"] = np.array([synthetic_runtime(land, Configuration(tuple(r)))
                                                        for r in idx.tolist()])
        meta["models"][name]["landscape"] = landscape_to_dict(land)
    # adaptive sampling (dedup, knee k-means, mode vote, batch) on wide points
    a3, m3 = models["alexnet3"]
    agent = init_agent(a3, AgentHyperparams(episodes_per_round=128), seed=8)
    st = np.random.default_rng(9)
    starts = [random_config(a3, st) for _ in range(128)]
    tr = run_search_round(agent, m3, a3, starts)
    cases = [("alexnet3_rl_round", a3, idx_of(tr.configs()), [tuple(r) for r in idx_of(starts).tolist()], 4242),
             ("alexnet3_uniform", a3, rng.integers(0, np.array(a3.cardinalities), size=(4000, 8)), [], 7),
             ("wide8_uniform", wide8, rng.integers(0, np.array(wide8.cardinalities), size=(3000, 8)), [], 8)]
    for name, space, pts, vis, seed in cases:
        batch = adaptive_sample(traj_of(np.asarray(pts)), VisitedSet([Configuration(v) for v in vis]), space, seed=seed)
        arrays[f"adaptive/{name}/idx"] = np.asarray(pts, dtype=np.int64)
        arrays[f"adaptive/{name}/visited"] = np.array(vis, dtype=np.int64).reshape(-1, space.n_knobs)
        arrays[f"adaptive/{name}/batch"] = idx_of(batch).reshape(-1, space.n_knobs)
        arrays[f"adaptive/{name}/mode"] = np.array(mode_config(traj_of(np.asarray(pts)), space).indices, dtype=np.int64)
        meta["adaptive"][name] = {"cards": list(space.cardinalities), "seed": seed, "model": space.name}
    # SA chains (default params) on the wide surrogate
    for name, mname, params, n_starts, seed in (("alexnet3_64x128", "alexnet3", SAParams(), 64, 77),
                                                ("wide8_32x64", "wide8", SAParams(chains=32, steps_per_round=64), 20, 5)):
        space, model = models[mname]
        r = np.random.default_rng(seed)
        starts = [random_config(space, r) for _ in range(n_starts)]
        tr = run_sa_round(params, model, space, starts, seed)
        arrays[f"sa/{name}/starts"] = idx_of(starts)
        arrays[f"sa/{name}/idx"] = idx_of(tr.configs())
        arrays[f"sa/{name}/scores"] = tr.scores()
        arrays[f"sa/{name}/steps"] = np.array(tr.step_indices, dtype=np.int64)
        meta["sa"][name] = {"model": mname, "chains": params.chains, "steps": params.steps_per_round,
                            "initial_temperature": params.initial_temperature, "cooling": params.cooling, "seed": seed}
    # one PPO search round (trajectory bit-exact, update at the TF32 tier)
    hyper = AgentHyperparams(episodes_per_round=256)
    agent = init_agent(a3, hyper, seed=12)
    st = np.random.default_rng(13)
    starts = [random_config(a3, st) for _ in range(256)]
    arrays["rl/alexnet3/params0"] = nets.flatten_params(agent.params)
    tr = run_search_round(agent, m3, a3, starts)
    arrays["rl/alexnet3/starts"] = idx_of(starts)
    arrays["rl/alexnet3/idx"] = idx_of(tr.configs())
    arrays["rl/alexnet3/scores"] = tr.scores()
    arrays["rl/alexnet3/steps"] = np.array(tr.step_indices, dtype=np.int64)
    arrays["rl/alexnet3/params"] = nets.flatten_params(agent.params)
    meta["rl"]["alexnet3"] = {"model": "alexnet3", "hyper": hyper.to_dict(), "seed": 12}
    np.savez_compressed(HERE / "wide.npz", **arrays)
    (HERE / "wide.json").write_text(json.dumps(meta, sort_keys=True))


def main():
    make_task_models()
    rng = np.random.default_rng(20261017)
    out_models: dict = {}
    models, lands = make_models(out_models)
    (HERE / "models.json").write_text(json.dumps(out_models, sort_keys=True))
    # the bench reads the S2 surrogate from data/ (not from tests/)
    (ROOT / "data" / "models").mkdir(parents=True, exist_ok=True)
    (ROOT / "data" / "models" / "s2_resnet18.json").write_text(json.dumps(out_models["s2_resnet18"], sort_keys=True))
    np.savez_compressed(HERE / "predict.npz", **gen_predict(models, rng))
    arrays, land_json = gen_landscapes(lands, rng)
    np.savez_compressed(HERE / "landscape.npz", **arrays)
    (HERE / "landscapes.json").write_text(json.dumps(land_json, sort_keys=True))
    arrays, names = gen_kmeans(rng)
    np.savez_compressed(HERE / "kmeans.npz", **arrays)
    arrays, names = gen_knee(rng)
    np.savez_compressed(HERE / "knee.npz", **arrays)
    arrays, meta = gen_adaptive(rng, models)
    np.savez_compressed(HERE / "adaptive.npz", **arrays)
    (HERE / "adaptive.json").write_text(json.dumps(meta, sort_keys=True))
    arrays, meta = gen_sa(models)
    np.savez_compressed(HERE / "sa.npz", **arrays)
    (HERE / "sa.json").write_text(json.dumps(meta, sort_keys=True))
    arrays, meta = gen_rl(models)
    np.savez_compressed(HERE / "rl.npz", **arrays)
    (HERE / "rl.json").write_text(json.dumps(meta, sort_keys=True))
    gen_wide()
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    import sys

    if sys.argv[1:] == ["wide"]:  # only the bit-field-layout fixtures (leaves the others untouched)
        gen_wide()
    else:
        main()
